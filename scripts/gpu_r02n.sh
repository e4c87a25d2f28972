# merge: sorted-prefix merge (no bucket sort); tc main pass clause check before the TMEM re-read; TC_MIN 10; step2 variants
O=gpurun_out/r02n; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_updates.py tests/test_gpu_scorers.py tests/test_gpu_idlist.py -q -x --timeout 900 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
for pr in LOW HIGH; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -10; done > $O/phases.txt 2>&1; cat $O/phases.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
for s2 in 0 1 2; do for pr in LOW HIGH ALL; do LINR_WS_STEP2=$s2 B --preset $pr --steps 1000; done; done
B --batch 256 --steps 100
B --batch 12 --steps 200
B --batch 16 --steps 200
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o $O/tc_b256 python bench.py --no-cpu-baseline --batch 256 --steps 2 --warmup 1 > /dev/null 2>&1
ls $O
