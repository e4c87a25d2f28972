# usage: bash scripts/ncu_gemv.sh <tag> [prof_search args]  (ncu --set full of one scan_gemv launch + hot SASS)
TAG=$1; shift
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:scan_gemv -s 3 -c 1 -o /tmp/$TAG python scripts/prof_search.py --iters 5 "$@" > /dev/null 2>&1
cp /tmp/$TAG.ncu-rep gpurun_out/
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > /tmp/$TAG.src.csv 2>/dev/null
python scripts/sass_hot.py /tmp/$TAG.src.csv 60 > gpurun_out/${TAG}_hot.txt 2>&1
gzip -c /tmp/$TAG.src.csv > gpurun_out/${TAG}.src.csv.gz
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
