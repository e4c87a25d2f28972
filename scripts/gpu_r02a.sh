# usage: bash scripts/gpu_r02a.sh -- round-2 state check: GPU tests + default bench
mkdir -p gpurun_out/r02a
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r02a/pytest_gpu.log 2>&1; tail -3 gpurun_out/r02a/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/r02a/bench_default.json 2> gpurun_out/r02a/bench_default.err; tail -1 gpurun_out/r02a/bench_default.json | python scripts/fmt_bench.py
run() { timeout 200 python bench.py --no-cpu-baseline --steps 100 "$@" 2>/dev/null | tail -1 | tee -a gpurun_out/r02a/sweep.jsonl | python scripts/fmt_bench.py; }
run --batch 256 --steps 30; run --preset LOW; run --dtype i8 --dim 64 --items 125000000
