# single step2 producer loop; merge probe (warm vs cold, prefix merge vs bucket sort)
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
(python scripts/merge_probe.py; LINR_MERGE_BUCKET=1 python scripts/merge_probe.py) > $O/merge_probe.txt 2>&1; cat $O/merge_probe.txt
for pr in LOW HIGH; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -10; echo "-- bucket"; LINR_MERGE_BUCKET=1 python scripts/phase_timers.py --preset $pr 2>&1 | tail -1; done > $O/phases.txt 2>&1; cat $O/phases.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
for pr in LOW HIGH ALL; do B --preset $pr --steps 1000; done
B --items 125000000 --dtype i8 --dim 64 --steps 200
B --items 100000000 --dtype i8 --dim 128 --steps 100
