O=gpurun_out/r02u2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_union.py -q --timeout 600 > $O/pytest_union.log 2>&1; tail -3 $O/pytest_union.log; grep -m8 "Error\|FAILED\|assert" $O/pytest_union.log
