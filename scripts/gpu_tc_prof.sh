# usage: bash scripts/gpu_tc_prof.sh <tag> -- ncu --set full of the batched tcgen05 scan (B=256 and B=16) + summaries
TAG=${1:-r01c}
mkdir -p gpurun_out/$TAG
for b in 256 16; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o /tmp/${TAG}_tc_scan_b$b python scripts/prof_search.py --iters 2 --batch $b --no-pass > /dev/null 2>&1
  python scripts/ncu_summary.py $TAG --rep /tmp/${TAG}_tc_scan_b$b.ncu-rep
  ncu -i /tmp/${TAG}_tc_scan_b$b.ncu-rep --page source --csv --print-source sass > /tmp/tc$b.src.csv 2>/dev/null
  python scripts/sass_hot.py /tmp/tc$b.src.csv 40 > gpurun_out/$TAG/tc_scan_b${b}_hot.txt 2>&1
done
cp profiles/${TAG}_${TAG}_tc_scan_b* gpurun_out/$TAG/
ls -la gpurun_out/$TAG
