# tcgen05 sample pass with rolled clause loop (code 22K -> 5.6K instructions)
O=gpurun_out/r02m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_updates.py -q -x --timeout 600 -k "batched or tensor or fullsize or version" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 256 --steps 100
B --batch 16 --steps 200
B --batch 12 --steps 200
B --batch 8 --steps 200
LINR_TC_MIN=2 B --batch 8 --steps 200
B --items 6250000 --vectors 8 --batch 32 --steps 100
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_b256.csv python bench.py --no-cpu-baseline --steps 3 --warmup 1 --batch 256 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 2 -c 2 -o $O/tc_b256 python bench.py --no-cpu-baseline --batch 256 --steps 2 --warmup 1 > /dev/null 2>&1
ls $O
for pr in LOW HIGH; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -10; done > $O/phases.txt 2>&1; cat $O/phases.txt
for pr in LOW HIGH ALL; do B --preset $pr --steps 1000; done
LINR_PDL=1 B --steps 1000
B --items 125000000 --dtype i8 --dim 64 --steps 200
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "not batched and not tensor" > $O/pytest2.log 2>&1; tail -2 $O/pytest2.log
