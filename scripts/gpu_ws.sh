# usage: bash scripts/gpu_ws.sh -- parity tests + bench presets + phase timers (bounded)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q --timeout 60 2>&1 | tail -3
for pre in HIGH ALL LOW; do
  echo "$pre: $(timeout 60 python bench.py --no-cpu-baseline --steps 200 --preset $pre 2>&1 | tail -1 | python scripts/fmt_bench.py)"
done
echo "OLD HIGH: $(LINR_NO_WS=1 timeout 60 python bench.py --no-cpu-baseline --steps 200 2>&1 | tail -1 | python scripts/fmt_bench.py)"
for pre in HIGH; do echo "== $pre"; timeout 60 python scripts/phase_timers.py --preset $pre; done
