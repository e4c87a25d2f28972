# tcgen05 epilogue: dynamic chunk tickets per TMEM lane quarter (LINR_TC_DYN)
O=gpurun_out/r02dyn; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_union.py -q -x --timeout 600 -k "batched or tensor or fullsize or certification or union" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 256 --steps 100; LINR_TC_DYN=0 B --batch 256 --steps 100
B --batch 64 --steps 100; LINR_TC_DYN=0 B --batch 64 --steps 100
B --items 6250000 --vectors 8 --batch 32 --steps 100; LINR_TC_DYN=0 B --items 6250000 --vectors 8 --batch 32 --steps 100
B --dtype i8 --dim 64 --items 125000000 --batch 256 --steps 10 --warmup 3; LINR_TC_DYN=0 B --dtype i8 --dim 64 --items 125000000 --batch 256 --steps 10 --warmup 3
