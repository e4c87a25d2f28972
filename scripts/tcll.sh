# launch list of the batched path at a few batch sizes (bench search: no pass counts)
mkdir -p gpurun_out
for b in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$b.csv python bench.py --no-cpu-baseline --batch $b --steps 1 --warmup 3 > /dev/null 2>&1
  echo "B=$b"; python scripts/launch_list.py gpurun_out/ll_$b.csv | tail -4
done
