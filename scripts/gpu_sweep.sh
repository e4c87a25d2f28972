# usage: bash scripts/gpu_sweep.sh -- GEMV-path bench lines across dtype (bounded)
mkdir -p gpurun_out/sweep
run() { echo "$*: $(timeout 120 python bench.py --no-cpu-baseline --steps 50 --warmup 3 "$@" 2>&1 | tail -1 | tee -a gpurun_out/sweep/lines.jsonl | python scripts/fmt_bench.py)"; }
timeout 300 python -m pytest tests -m gpu -x -q --timeout 60 2>&1 | tail -2
run
run --dtype i8 --dim 128 --items 12500000
run --dtype i8 --dim 64 --items 125000000
run --dtype bf16 --dim 64 --items 50000000
run --preset LOW
run --preset ALL
run --dtype i8 --dim 128 --items 12500000 --preset ALL
