# usage: bash scripts/gpu_check.sh  -- GPU tests, smoke, bench lines, launch list (outputs in gpurun_out/)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
for bsz in 16 256; do timeout 300 python bench.py --no-cpu-baseline --batch $bsz --steps 50 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_b$bsz.json; cat gpurun_out/bench_b$bsz.json; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_list.py gpurun_out/launches.csv | sort | uniq -c | sort -rn | head -20
