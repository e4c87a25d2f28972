# union path (2 <= B*V <= 8): parity + bench vs LINR_UNION=0
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_union.py -q -x --timeout 600 > $O/pytest_union.log 2>&1; tail -3 $O/pytest_union.log; grep -m5 "Error\|FAILED\|assert" $O/pytest_union.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_updates.py tests/test_gpu_idlist.py -q -x --timeout 900 > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
for b in 2 4 8; do B --batch $b --steps 300; LINR_UNION=0 B --batch $b --steps 300; done
B --batch 8 --preset LOW --steps 300
B --batch 8 --preset ALL --steps 100
B --items 6250000 --vectors 8 --batch 1 --steps 300
B --items 125000000 --dtype i8 --dim 64 --batch 8 --steps 50
LINR_UNION=0 B --items 125000000 --dtype i8 --dim 64 --batch 8 --steps 50
