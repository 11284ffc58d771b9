#!/bin/bash
# ncu --set full of the fp32 coarse kernels of one Wan2.1-1.3B step (SIMT GEMMs, softmax / top-k)
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'gemm_f32_pipe|coarse_softmax_topk' -c 5 -o gpurun_out/ncu_coarse -f python tools/one_step.py wan13 > gpurun_out/ncu_coarse.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ncu_coarse.ncu-rep --page details --csv > gpurun_out/ncu_coarse_details.csv 2>&1
ncu -i gpurun_out/ncu_coarse.ncu-rep --page raw --csv > gpurun_out/ncu_coarse_raw.csv 2>&1
ls -la gpurun_out/ncu_coarse*
