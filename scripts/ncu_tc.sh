# usage: bash scripts/ncu_tc.sh <batch> <tag>  (ncu --set full of the main tcgen05 pass + hot SASS list)
B=$1; TAG=$2
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o /tmp/$TAG python scripts/prof_search.py --iters 2 --batch $B --no-pass > /dev/null 2>&1
python scripts/ncu_summary.py $TAG --rep /tmp/$TAG.ncu-rep
cp profiles/${TAG}_${TAG}.md gpurun_out/ 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > /tmp/$TAG.src.csv 2>/dev/null
python scripts/sass_hot.py /tmp/$TAG.src.csv 70 > gpurun_out/${TAG}_hot.txt 2>&1
python scripts/sass_hot.py /tmp/$TAG.src.csv 70 exec > gpurun_out/${TAG}_hot_exec.txt 2>&1
gzip -c /tmp/$TAG.src.csv > gpurun_out/${TAG}.src.csv.gz
