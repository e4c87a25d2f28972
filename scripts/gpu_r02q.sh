# merge: pairwise prefix merge, two interleaved branchless searches per thread; finalize one wave
O=gpurun_out/r02q; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 900 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m3 "FAILED\|Error" $O/pytest.log
(python scripts/merge_probe.py; LINR_MERGE_BUCKET=1 python scripts/merge_probe.py) > $O/merge_probe.txt 2>&1; cat $O/merge_probe.txt
for pr in LOW HIGH; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -10; done > $O/phases.txt 2>&1; cat $O/phases.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --steps 1000
B --preset LOW --steps 1000
B --batch 256 --steps 100
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_b256.csv python bench.py --no-cpu-baseline --steps 3 --warmup 1 --batch 256 > /dev/null 2>&1
ls $O
