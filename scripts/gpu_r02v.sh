# union path with per-lane candidate tests (V = 1)
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_union.py tests/test_gpu_parity.py -q -x --timeout 600 -k "union or batches or variants" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
for b in 2 4 8; do B --batch $b --steps 300; done
B --batch 8 --preset LOW --steps 300
B --batch 8 --preset ALL --steps 100
B --items 125000000 --dtype i8 --dim 64 --batch 8 --steps 50
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 2 -c 1 -o $O/union_b8 python bench.py --no-cpu-baseline --batch 8 --steps 2 --warmup 1 > /dev/null 2>&1
ncu -i $O/union_b8.ncu-rep --page source --csv --print-source sass > /tmp/u.csv 2>/dev/null; python scripts/sass_hot.py /tmp/u.csv 25 > $O/union_b8_hot.txt; head -28 $O/union_b8_hot.txt
