O=gpurun_out/r02g16; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_union.py tests/test_gpu_parity.py -q -x --timeout 600 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED\|assert" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 16 --steps 200; B --batch 16 --preset LOW --steps 200; B --batch 12 --steps 200; B --batch 12 --preset LOW --steps 200
B --batch 8 --steps 300; B --batch 8 --preset LOW --steps 300; B --batch 256 --steps 50; B --steps 2000
