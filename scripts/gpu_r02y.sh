# region gather: eight loads in flight per thread
O=gpurun_out/r02y2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 -k "batched or tensor or fullsize or certification" > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -m5 "Error\|FAILED" $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --batch 256 --steps 100
B --items 6250000 --vectors 8 --batch 32 --steps 100
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_b256.csv python bench.py --no-cpu-baseline --steps 3 --warmup 1 --batch 256 > /dev/null 2>&1
python scripts/ncu_summary.py r02y2_b256 --launches $O/launches_b256.csv > /dev/null; cp profiles/r02y2_b256_launches.md $O/; sed -n 5,12p $O/r02y2_b256_launches.md
