# final state check: full GPU suite, smoke, default bench, reference arm
O=gpurun_out/r02final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log; grep -m5 "FAILED\|Error" $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -1 $O/bench_default.json | python scripts/fmt_line.py
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>&1; tail -c 300 $O/bench_ref.json
