# LOW preset: phase timers, two-tile producer step for 256 B rows (LINR_WS_STEP2)
O=gpurun_out/r02k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "variants" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for pr in LOW HIGH ALL; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -12; echo "-- step2"; LINR_WS_STEP2=1 python scripts/phase_timers.py --preset $pr 2>&1 | tail -12; done > $O/phases.txt 2>&1
cat $O/phases.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
for pr in LOW HIGH ALL; do B --preset $pr --steps 500; LINR_WS_STEP2=1 B --preset $pr --steps 500; done
B --items 100000000 --dtype i8 --dim 128 --steps 100
LINR_WS_STEP2=1 B --items 100000000 --dtype i8 --dim 128 --steps 100
