#!/bin/bash
# ncu --set full of every kernel of one Wan2.1-1.3B step and of the DiT fine kernels, summarised
mkdir -p gpurun_out
tag=${1:-r2}
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/full_${tag}_wan13 -f python tools/one_step.py wan13 > gpurun_out/ncu_full_${tag}.log 2>&1
echo "wan13 rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:'fine_' -o gpurun_out/full_${tag}_dit -f python tools/one_step.py dit >> gpurun_out/ncu_full_${tag}.log 2>&1
echo "dit rc=$?"
python tools/ncu_summary.py gpurun_out/full_${tag}_wan13.ncu-rep > gpurun_out/ncu_${tag}_kernels.json
python tools/ncu_summary.py gpurun_out/full_${tag}_dit.ncu-rep > gpurun_out/ncu_${tag}_dit_kernels.json
python - <<PY
import json
for f in ("gpurun_out/ncu_${tag}_kernels.json", "gpurun_out/ncu_${tag}_dit_kernels.json"):
    for k in json.load(open(f))["kernels"]:
        print(k["kernel"].split("(")[0][-40:], k["duration_ms"], "tc%", k["tensor_pipe_active_pct"], "smem tc/lsu", k["smem_tc_wavefronts_pct"], k["smem_lsu_wavefronts_pct"], "dram%", k["dram_throughput_pct"])
PY
