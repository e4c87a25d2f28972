# usage: bash scripts/gpu_ws.sh -- ring-scan parity tests + A/B vs the per-warp kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 300 2>&1 | tail -3
for pre in HIGH ALL LOW; do
  echo "RING $pre: $(timeout 300 python bench.py --no-cpu-baseline --steps 200 --preset $pre 2>&1 | tail -1 | python scripts/fmt_bench.py)"
done
for kb in 64 256; do
  echo "RING ${kb}KB HIGH: $(LINR_WS_RING_KB=$kb timeout 300 python bench.py --no-cpu-baseline --steps 200 2>&1 | tail -1 | python scripts/fmt_bench.py)"
done
