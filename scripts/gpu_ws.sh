# usage: bash scripts/gpu_ws.sh -- ring-scan parity tests + bench presets + phase timers (bounded)
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 60 2>&1 | tail -3
for cm in 32768 4096 2048; do
for pre in HIGH ALL LOW; do
  echo "CMAX=$cm $pre: $(LINR_WS_CMAX=$cm timeout 60 python bench.py --no-cpu-baseline --steps 200 --preset $pre 2>&1 | tail -1 | python scripts/fmt_bench.py)"
done
done
echo "FUSED HIGH: $(LINR_FUSE_MERGE=1 timeout 60 python bench.py --no-cpu-baseline --steps 200 2>&1 | tail -1 | python scripts/fmt_bench.py)"
for cm in 32768 2048; do echo "== HIGH CMAX=$cm"; LINR_WS_CMAX=$cm timeout 60 python scripts/phase_timers.py --preset HIGH; done
