# check: GR=16 one-tile loop restored (c2 HIGH), finalize cap, TC_MIN 9; then the sanitizer pass
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --steps 1000
B --preset LOW --steps 1000
B --batch 9 --steps 200
B --batch 256 --steps 100
B --dtype i8 --dim 128 --items 100000000 --batch 256 --steps 10 --warmup 3
