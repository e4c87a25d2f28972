O=gpurun_out/r02ref; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_union.py -q -x --timeout 600 -k "batched or tensor or fullsize or certification or finalize or union or refine" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED\|assert" $O/pytest.log
python scripts/tc_diag.py 125000000 64 i8 > $O/diag.txt 2>&1; cat $O/diag.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --dtype i8 --dim 64 --items 125000000 --batch 256 --steps 10 --warmup 3
LINR_TC_REFINE=0 B --dtype i8 --dim 64 --items 125000000 --batch 256 --steps 10 --warmup 3
B --dtype i8 --dim 128 --items 100000000 --batch 256 --steps 10 --warmup 3
LINR_TC_REFINE=0 B --dtype i8 --dim 128 --items 100000000 --batch 256 --steps 10 --warmup 3
B --items 50000000 --vectors 8 --batch 32 --steps 20
B --batch 256 --steps 100
