# usage: bash scripts/gpu_check.sh <tag> -- GPU tests, smoke, bench lines, launch list, ncu --set full of the scan (outputs in gpurun_out/)
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/$TAG/pytest_gpu.log 2>&1; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; tail -2 gpurun_out/$TAG/smoke.log
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err; tail -1 gpurun_out/$TAG/bench_default.json
for bsz in 16 256; do timeout 300 python bench.py --no-cpu-baseline --batch $bsz --steps 50 --warmup 3 2>/dev/null | tail -1 > gpurun_out/$TAG/bench_b$bsz.json; cat gpurun_out/$TAG/bench_b$bsz.json; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_ref.json 2>&1; tail -1 gpurun_out/$TAG/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --pipeline 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o gpurun_out/$TAG/scan_ws_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_kernel -s 3 -c 1 -o gpurun_out/$TAG/merge_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
ls -la gpurun_out/$TAG
