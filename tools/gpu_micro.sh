#!/bin/bash
mkdir -p gpurun_out
./tests/cuda/bin/tmem_bench > gpurun_out/tmem.txt 2>&1
cat gpurun_out/tmem.txt
