O=gpurun_out/r02c5; mkdir -p $O
(python scripts/phase_timers.py --items 6250000 --V 8; python scripts/phase_timers.py --items 6250000 --V 1) > $O/phases.txt 2>&1; cat $O/phases.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o $O/c5_u1 python bench.py --no-cpu-baseline --items 6250000 --vectors 8 --steps 2 --warmup 1 > /dev/null 2>&1
ncu -i $O/c5_u1.ncu-rep --page source --csv --print-source sass > /tmp/c.csv 2>/dev/null; python scripts/sass_hot.py /tmp/c.csv 30 > $O/c5_u1_hot.txt; head -32 $O/c5_u1_hot.txt
python scripts/ncu_summary.py r02c5 --rep $O/c5_u1.ncu-rep > /dev/null; cp profiles/r02c5_c5_u1.md $O/; grep -E "Duration|Issue|dram__bytes_read.sum =" $O/r02c5_c5_u1.md
