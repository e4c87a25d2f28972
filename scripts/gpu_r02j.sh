# count kernel (one attribute read for all users), V=8 GEMV append fix, smem budget fix; launch lists
O=gpurun_out/r02j; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "batched or tensor or multivector or variants" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
B() { timeout 900 python bench.py --no-cpu-baseline "$@" 2>>$O/bench.err | tail -1 | tee -a $O/bench.jsonl | python scripts/fmt_line.py || tail -3 $O/bench.err; }
B --items 6250000 --vectors 8 --batch 1 --steps 300
B --batch 8 --steps 200
LINR_TC_MIN=2 B --batch 8 --steps 200
LINR_TC_MIN=2 B --batch 4 --steps 200
B --batch 256 --steps 100
B --preset LOW --steps 500
L() { timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_$1.csv python bench.py --no-cpu-baseline --steps 3 --warmup 1 "${@:2}" > /dev/null 2>&1; }
L b256 --batch 256
LINR_TC_MIN=2 L b8tc --batch 8
L low --preset LOW
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o $O/ws_low python bench.py --no-cpu-baseline --preset LOW --steps 2 --warmup 1 > /dev/null 2>&1
ls $O
