O=gpurun_out/r02e2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "host or nccl or pipelined or concurrent" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 256 --steps 100
B --batch 16 --steps 200
B --batch 8 --steps 300
B --steps 2000
