#!/bin/bash
# ncu evidence for profiles/: (1) launch list of one Wan2.1-1.3B step (per-launch
# gpu__time_duration, clock-control none), (2) a full-set capture of the fine kernels.
mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python tools/one_step.py
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'fine_(fwd|dkdv|dq_gemm)|tile_pool|prologue' -c 6 -o gpurun_out/prof -f python tools/one_step.py
