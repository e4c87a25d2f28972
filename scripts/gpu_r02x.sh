# union dispatch rule (V = 1, 3 <= B <= 8): full GPU suite + small-batch bench lines
O=gpurun_out/r02x; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log; grep -m5 "Error\|FAILED" $O/pytest_gpu.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --steps 1000
for b in 2 3 4 8; do B --batch $b --steps 300; done
B --batch 8 --preset ALL --steps 100
B --batch 8 --preset LOW --steps 300
B --batch 4 --vectors 2 --steps 200
