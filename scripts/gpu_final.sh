# usage: bash scripts/gpu_final.sh <tag> -- full GPU evidence: tests, smoke, bench lines, sweep, launch list, ncu captures
TAG=${1:-r01c}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/$TAG/pytest_gpu.log 2>&1; tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; tail -1 gpurun_out/$TAG/smoke.log
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err; tail -1 gpurun_out/$TAG/bench_default.json | python scripts/fmt_bench.py
run() { timeout 200 python bench.py --no-cpu-baseline --steps 100 "$@" 2>/dev/null | tail -1 | tee -a gpurun_out/$TAG/sweep.jsonl | python scripts/fmt_bench.py; }
run --preset ALL; run --preset LOW; run --batch 8; run --batch 16 --steps 50; run --batch 256 --steps 30
run --dtype i8 --dim 128 --items 12500000; run --dtype i8 --dim 64 --items 125000000; run --dtype bf16 --dim 64 --items 50000000
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --pipeline 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o gpurun_out/$TAG/scan_ws_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o gpurun_out/$TAG/scan_ws_c4_i8_high python scripts/prof_search.py --iters 5 --dtype i8 --dim 64 --items 125000000 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_kernel -s 3 -c 1 -o gpurun_out/$TAG/merge_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
ls gpurun_out/$TAG
