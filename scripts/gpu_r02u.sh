# union path B=8 HIGH: ncu of the multi-user ring scan
O=gpurun_out/r02u; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 2 -c 1 -o $O/union_b8 python bench.py --no-cpu-baseline --batch 8 --steps 2 --warmup 1 > /dev/null 2>&1
ncu -i $O/union_b8.ncu-rep --page source --csv --print-source sass > /tmp/u.csv 2>/dev/null; python scripts/sass_hot.py /tmp/u.csv 40 > $O/union_b8_hot.txt; head -45 $O/union_b8_hot.txt
python scripts/ncu_summary.py r02u --rep $O/union_b8.ncu-rep > /dev/null; cp profiles/r02u_union_b8.md $O/
ls $O
