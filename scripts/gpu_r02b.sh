# round-2 check: GPU tests (new parity cases), compute-sanitizer on every search kernel, quick bench
mkdir -p gpurun_out/r02b
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/r02b/pytest_gpu.log 2>&1; tail -5 gpurun_out/r02b/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  for c in ws gemv tc fb; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py $c > gpurun_out/r02b/san_${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize case' gpurun_out/r02b/san_${tool}_$c.log | tr '\n' ' ')"
  done
done
timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1 | python scripts/fmt_bench.py
timeout 300 python bench.py --no-cpu-baseline --steps 30 --batch 256 2>/dev/null | tail -1 | python scripts/fmt_bench.py
