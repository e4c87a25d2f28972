# usage: bash scripts/gpu_ab.sh [tag] -- A/B bench of the warp-specialised vs per-warp GEMV scan + ncu of the WS kernel
TAG=${1:-ws}
mkdir -p gpurun_out
for pre in HIGH ALL LOW; do
  echo "WS $pre: $(timeout 300 python bench.py --no-cpu-baseline --steps 200 --preset $pre 2>&1 | tail -1 | python scripts/fmt_bench.py)"
  echo "OLD $pre: $(LINR_NO_WS=1 timeout 300 python bench.py --no-cpu-baseline --steps 200 --preset $pre 2>&1 | tail -1 | python scripts/fmt_bench.py)"
done
ncu --set full --import-source on --clock-control none -k regex:scan_ws -s 3 -c 1 -o /tmp/$TAG python scripts/prof_search.py --iters 5 > /dev/null 2>&1
cp /tmp/$TAG.ncu-rep gpurun_out/
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > /tmp/$TAG.src.csv 2>/dev/null
python scripts/sass_hot.py /tmp/$TAG.src.csv 60 > gpurun_out/${TAG}_hot.txt 2>&1
gzip -c /tmp/$TAG.src.csv > gpurun_out/${TAG}.src.csv.gz
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
