# new tcgen05 main-pass epilogue (per-thread hot masks, TMEM re-read of hot columns): parity + bench
O=gpurun_out/r02i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_updates.py tests/test_gpu_fullsize.py -q -x --timeout 600 -k "batched or tensor or updates or version or fullsize" > $O/pytest.log 2>&1; tail -3 $O/pytest.log; grep -m3 "Error\|error" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 256 --steps 100
B --batch 16 --steps 100
B --items 6250000 --vectors 8 --batch 32 --steps 50
for b in 8 10 12; do LINR_TC_MIN=2 B --batch $b --steps 200; done
B --batch 256 --dtype i8 --dim 64 --items 125000000 --steps 10 --warmup 3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o $O/tc_b256 python bench.py --no-cpu-baseline --batch 256 --steps 2 --warmup 1 > /dev/null 2>&1
ls $O
