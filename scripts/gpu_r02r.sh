# gather_regions with all loads in flight; fallback early exit; merge ncu source capture
O=gpurun_out/r02r; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_updates.py -q -x --timeout 900 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m3 "FAILED\|Error" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 256 --steps 100
B --batch 16 --steps 200
B --batch 12 --steps 200
B --items 6250000 --vectors 8 --batch 32 --steps 100
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_b256.csv python bench.py --no-cpu-baseline --steps 3 --warmup 1 --batch 256 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:merge_kernel -s 5 -c 1 -o $O/merge_high python bench.py --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1
ls $O
