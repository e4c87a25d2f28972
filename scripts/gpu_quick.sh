# usage: bash scripts/gpu_quick.sh -- GPU parity tests + default bench (+ old-kernel A/B)
mkdir -p gpurun_out
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 200 2>gpurun_out/bench.err | tail -1 | python scripts/fmt_bench.py 2>/dev/null || tail -3 gpurun_out/bench.err
LINR_NO_WS=1 timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1 | python scripts/fmt_bench.py
for pre in ALL LOW; do timeout 300 python bench.py --no-cpu-baseline --steps 200 --preset $pre 2>/dev/null | tail -1 | python scripts/fmt_bench.py; done
