# merge: 8-way prefix merge rounds; tc: no dbg code, SHF tree, 2-clause fast path
O=gpurun_out/r02p; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_updates.py -q -x --timeout 900 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m3 "FAILED\|Error" $O/pytest.log
(python scripts/merge_probe.py; LINR_MERGE_BUCKET=1 python scripts/merge_probe.py) > $O/merge_probe.txt 2>&1; cat $O/merge_probe.txt
for pr in LOW HIGH; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -10; done > $O/phases.txt 2>&1; cat $O/phases.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --steps 1000
B --batch 256 --steps 100
B --batch 256 --dtype i8 --dim 128 --items 100000000 --steps 10 --warmup 3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o $O/tc_b256 python bench.py --no-cpu-baseline --batch 256 --steps 2 --warmup 1 > /dev/null 2>&1
ls $O
