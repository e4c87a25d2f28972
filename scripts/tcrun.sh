timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k batched --timeout 300 2>&1 | tail -2
python scripts/tc_timers.py 256 | tail -1
for bsz in 16 64 256; do timeout 300 python bench.py --no-cpu-baseline --batch $bsz --steps 50 --warmup 3 2>&1 | tail -1; done
