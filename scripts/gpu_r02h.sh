# measurement matrix + version-tag test + short-row gather / L2 fetch experiment + tc-min sweep
O=gpurun_out/r02h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_updates.py -q -x --timeout 500 > $O/pytest_updates.log 2>&1; tail -2 $O/pytest_updates.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/matrix.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
# c5 multi-embedding: 50M/8 rows per GPU, V=8, U=1 and U=32
B --items 6250000 --vectors 8 --batch 1 --steps 300
B --items 6250000 --vectors 8 --batch 32 --steps 50
B --items 50000000 --vectors 8 --batch 1 --steps 100
# c3 G=1 scaling base: 100M int8 d=128; c4 1B int8 d=64 on one GPU
B --items 100000000 --dtype i8 --dim 128 --steps 100
B --items 1000000000 --dtype i8 --dim 64 --steps 20 --warmup 3
B --items 1000000000 --dtype i8 --dim 64 --preset LOW --steps 20 --warmup 3
# c4 shard (125M) live updates: 0 / 300 / 600 / 1e5 rows/s
for r in 0 300 600 100000; do B --items 125000000 --dtype i8 --dim 64 --update-rate $r --steps 2000 --pipeline 1; done
# c2 updates at 1e5 rows/s
B --update-rate 100000 --steps 5000 --pipeline 1
# small batches: GEMV (default) vs tcgen05 (LINR_TC_MIN=2)
for b in 2 4 8 12; do B --batch $b --steps 200; LINR_TC_MIN=2 B --batch $b --steps 200; done
# c4 shard L2 fetch granularity
for g in 32 64 128; do LINR_L2_FETCH=$g B --items 125000000 --dtype i8 --dim 64 --steps 200; done
(cd scripts/micro && ./gather64 125000000 64 > ../../$O/gather64.txt 2>&1; ./gather64 100000000 128 >> ../../$O/gather64.txt 2>&1); cat $O/gather64.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $O/gather64_ncu.csv scripts/micro/gather64 125000000 64 > /dev/null 2>&1
for g in 32 128; do LINR_L2_FETCH=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan_ws -c 3 --csv --log-file $O/c4_l2fetch_$g.csv python bench.py --no-cpu-baseline --items 125000000 --dtype i8 --dim 64 --steps 2 --warmup 1 > /dev/null 2>&1; done
ls $O
