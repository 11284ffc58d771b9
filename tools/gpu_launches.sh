#!/bin/bash
# ncu launch lists (per-launch duration + DRAM bytes, clock-control none) of one step, per config
mkdir -p gpurun_out
tag=${1:-r2}
for cfg in wan13 dit; do
  timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}_${cfg}.csv python tools/one_step.py $cfg > /dev/null 2>&1
  echo "== $cfg"; python tools/launch_table.py gpurun_out/launches_${tag}_${cfg}.csv
done
