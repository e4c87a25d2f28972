# quantised path: regression subset, bench lines (1B x 64-bit top-50M; V3 at 10M 512-bit), ncu
mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_gpu_codes.py -q -x --timeout 600 -k "bit_exact or v3" > gpurun_out/r02e/pytest_codes.log 2>&1; tail -2 gpurun_out/r02e/pytest_codes.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/r02e/bench.err | tail -1 | tee -a gpurun_out/r02e/codes.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'ms', round(d['ms_per_step'],3), 'lat', {k: round(v,3) for k,v in d['latency_ms'].items()}, 'frac', d['roofline']['frac'], 'pass1', d['roofline']['pass1_ms_per_launch'], 'rest', d['roofline']['rest_ms_per_launch'], 'recall', d['recall_at_K_vs_exact'], 'e2e ms', round(d['e2e']['ms_per_step'],3))" || tail -5 gpurun_out/r02e/bench.err; }
B --path codes --dtype f16 --dim 64 --items 1000000000 --preset ALL --code-bits 64 --steps 20 --warmup 3
B --path codes --dtype f16 --dim 64 --items 1000000000 --preset HIGH --code-bits 64 --steps 20 --warmup 3
B --path codes --dtype bf16 --dim 128 --items 10000000 --preset HIGH --code-bits 512 --topk 1000 --steps 100
for keep in 0.001 0.01 0.1; do B --path v3 --dtype bf16 --dim 128 --items 10000000 --preset HIGH --code-bits 512 --keep $keep --steps 100; done
B --path v3 --dtype bf16 --dim 128 --items 10000000 --preset HIGH --code-bits 256 --keep 0.01 --steps 100
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02e/launches_codes.csv python bench.py --no-cpu-baseline --path codes --dtype f16 --dim 64 --items 100000000 --preset ALL --code-bits 64 --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02e/launches_v3.csv python bench.py --no-cpu-baseline --path v3 --dtype bf16 --dim 128 --items 10000000 --preset HIGH --code-bits 512 --keep 0.01 --steps 2 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out/r02e
