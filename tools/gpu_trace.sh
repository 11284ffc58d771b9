#!/bin/bash
mkdir -p gpurun_out
for c in wan13 dit; do echo "== $c"; VSA_LIB_PATH=paper_2505_13389_b200/_lib/variants/libvsa_trace.so timeout 120 python tools/trace_fwd.py $c; done > gpurun_out/trace_fwd.txt 2>&1
cat gpurun_out/trace_fwd.txt
