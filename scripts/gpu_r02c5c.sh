O=gpurun_out/r02c5c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_union.py tests/test_gpu_fullsize.py -q -x --timeout 600 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --items 6250000 --vectors 8 --batch 1 --steps 500
B --items 50000000 --vectors 8 --batch 1 --steps 100
B --vectors 2 --batch 1 --steps 500
B --dtype i8 --dim 64 --items 125000000 --vectors 4 --steps 100
B --steps 1000
