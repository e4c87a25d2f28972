mkdir -p gpurun_out/r02c
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02c/pytest_gpu.log 2>&1; tail -8 gpurun_out/r02c/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py fb > gpurun_out/r02c/san_${tool}_fb.log 2>&1
  echo "$tool fb rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize case' gpurun_out/r02c/san_${tool}_fb.log | tr '\n' ' ')"
done
timeout 300 python bench.py --no-cpu-baseline --steps 30 --batch 256 2>/dev/null | tail -1 | python scripts/fmt_bench.py
