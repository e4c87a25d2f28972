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
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o /tmp/${TAG}_scan_ws_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o /tmp/${TAG}_scan_ws_c4_i8_high python scripts/prof_search.py --iters 5 --dtype i8 --dim 64 --items 125000000 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_kernel -s 3 -c 1 -o /tmp/${TAG}_merge_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
python scripts/ncu_summary.py $TAG --launches gpurun_out/$TAG/launches.csv --rep /tmp/${TAG}_scan_ws_c2_high.ncu-rep /tmp/${TAG}_merge_c2_high.ncu-rep --workload "c2: 10M items/GPU d=128 bf16, 64-bit attribute bitmask pre-filter (HIGH), B=1, K=1000"
python scripts/ncu_summary.py $TAG --rep /tmp/${TAG}_scan_ws_c4_i8_high.ncu-rep --workload "shard: 125M items/GPU d=64 i8, 64-bit attribute bitmask pre-filter (HIGH), B=1, K=1000"
cp profiles/${TAG}_* profiles/scan_traffic.json gpurun_out/$TAG/
for r in c2_high c4_i8_high; do ncu -i /tmp/${TAG}_scan_ws_$r.ncu-rep --page source --csv --print-source sass > /tmp/$r.src.csv 2>/dev/null; python scripts/sass_hot.py /tmp/$r.src.csv 40 > gpurun_out/$TAG/scan_ws_${r}_hot.txt 2>&1; done
ls -la gpurun_out/$TAG
