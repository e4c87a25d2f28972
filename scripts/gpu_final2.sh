# usage: bash scripts/gpu_final2.sh <tag> -- round-2 evidence: tests, smoke, default bench + reference arm,
# the measurement matrix, launch list, ncu captures (summaries into gpurun_out/<tag>)
TAG=${1:-r02z}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -1 $O/bench_default.json | python scripts/fmt_line.py
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2>&1; tail -c 400 $O/bench_ref.json
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/sweep.err | tail -1 | tee -a $O/sweep.jsonl | python scripts/fmt_line.py || tail -3 $O/sweep.err; }
B --preset ALL --steps 300; B --preset LOW --steps 2000; B --preset HIGH4 --steps 1000
B --batch 3 --steps 300; B --batch 4 --steps 300; B --batch 8 --steps 300; B --batch 8 --preset ALL --steps 100; B --batch 8 --preset LOW --steps 300
LINR_TC_MIN=2 B --batch 4 --steps 300; LINR_TC_MIN=2 B --batch 8 --steps 300; LINR_UNION=0 B --batch 8 --steps 300; LINR_UNION=0 B --batch 8 --preset ALL --steps 100
B --batch 12 --steps 200; B --batch 16 --steps 200; B --batch 64 --steps 100; B --batch 256 --steps 100
B --dtype f16 --batch 256 --steps 100
B --dtype i8 --dim 128 --items 12500000 --steps 1000
B --dtype i8 --dim 128 --items 100000000 --steps 200
B --dtype i8 --dim 64 --items 125000000 --steps 300
B --dtype i8 --dim 64 --items 125000000 --preset LOW --steps 300
B --dtype i8 --dim 64 --items 1000000000 --steps 20 --warmup 3
B --dtype i8 --dim 64 --items 1000000000 --preset LOW --steps 20 --warmup 3
B --dtype i8 --dim 128 --items 100000000 --batch 256 --steps 10 --warmup 3
B --dtype bf16 --dim 64 --items 50000000 --steps 300
B --items 6250000 --vectors 8 --batch 1 --steps 500
B --items 6250000 --vectors 8 --batch 32 --steps 100
B --items 50000000 --vectors 8 --batch 1 --steps 100
B --items 50000000 --vectors 8 --batch 32 --steps 20
for r in 0 300 600 100000; do B --dtype i8 --dim 64 --items 125000000 --update-rate $r --steps 2000; done
B --update-rate 100000 --steps 10000
B --path codes --dtype f16 --dim 64 --items 1000000000 --preset ALL --code-bits 64 --steps 20 --warmup 3
B --path v3 --dtype bf16 --dim 128 --items 10000000 --preset HIGH --code-bits 512 --keep 0.01 --steps 200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --pipeline 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o /tmp/${TAG}_scan_ws_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o /tmp/${TAG}_scan_ws_c4_i8_high python scripts/prof_search.py --iters 5 --dtype i8 --dim 64 --items 125000000 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_kernel -s 3 -c 1 -o /tmp/${TAG}_merge_c2_high python scripts/prof_search.py --iters 5 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o /tmp/${TAG}_tc_b256 python bench.py --no-cpu-baseline --batch 256 --steps 2 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py $TAG --launches $O/launches.csv --rep /tmp/${TAG}_scan_ws_c2_high.ncu-rep --workload "c2: 10M items/GPU d=128 bf16, 64-bit attribute bitmask pre-filter (HIGH), B=1, K=1000"
python scripts/ncu_summary.py $TAG --rep /tmp/${TAG}_merge_c2_high.ncu-rep
python scripts/ncu_summary.py $TAG --rep /tmp/${TAG}_tc_b256.ncu-rep --workload "c2: 10M items/GPU d=128 bf16, 64-bit attribute bitmask pre-filter (HIGH), B=256, K=1000"
python scripts/ncu_summary.py $TAG --rep /tmp/${TAG}_scan_ws_c4_i8_high.ncu-rep --workload "shard: 125M items/GPU d=64 i8, 64-bit attribute bitmask pre-filter (HIGH), B=1, K=1000"
cp profiles/${TAG}_* profiles/scan_traffic.json $O/
for r in scan_ws_c2_high scan_ws_c4_i8_high tc_b256 merge_c2_high; do ncu -i /tmp/${TAG}_$r.ncu-rep --page source --csv --print-source sass > /tmp/$r.src.csv 2>/dev/null; python scripts/sass_hot.py /tmp/$r.src.csv 40 > $O/${r}_hot.txt 2>&1; done
ls -la $O
