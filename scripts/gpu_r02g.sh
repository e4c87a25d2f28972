# round-2 re-entry check: full GPU suite + default bench line + smoke
mkdir -p gpurun_out/r02g
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02g/pytest_gpu.log 2>&1; tail -3 gpurun_out/r02g/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g/smoke.log 2>&1; tail -1 gpurun_out/r02g/smoke.log
timeout 600 python bench.py > gpurun_out/r02g/bench_default.json 2>gpurun_out/r02g/bench.err; tail -c 1500 gpurun_out/r02g/bench_default.json
