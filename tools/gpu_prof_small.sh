#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'coarse_softmax|tile_pool|prologue_kernel' -c 3 -o gpurun_out/prof_small -f python tools/one_step.py > gpurun_out/ncu_small.log 2>&1
tail -3 gpurun_out/ncu_small.log
