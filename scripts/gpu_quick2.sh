# usage: bash scripts/gpu_quick2.sh -- headline bench lines + phase timers (bounded)
run() { echo "$*: $(timeout 120 python bench.py --no-cpu-baseline --steps 200 "$@" 2>&1 | tail -1 | python scripts/fmt_bench.py)"; }
run
run --dtype i8 --dim 64 --items 125000000
run --preset ALL
timeout 60 python scripts/phase_timers.py --preset HIGH
