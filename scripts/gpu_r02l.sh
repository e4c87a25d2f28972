# adaptive two-tile producer step, PDL merge launch, register bitonic sort in the merge
O=gpurun_out/r02l; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_idlist.py tests/test_gpu_codes.py -q -x --timeout 900 > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for pr in LOW HIGH ALL; do echo "== $pr"; python scripts/phase_timers.py --preset $pr 2>&1 | tail -10; done > $O/phases.txt 2>&1
cat $O/phases.txt
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
for pr in LOW HIGH ALL; do B --preset $pr --steps 1000; done
LINR_NO_PDL=1 B --steps 1000
B --batch 4 --steps 300
B --items 125000000 --dtype i8 --dim 64 --steps 200
