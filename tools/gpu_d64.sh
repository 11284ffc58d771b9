#!/bin/bash
# d = 64 experiments: MUFU throughput, poly-exp variants of the fine kernels on the DiT config
mkdir -p gpurun_out
./tests/cuda/bin/mufu_bench > gpurun_out/mufu.txt 2>&1
summ() { python -c "import json,sys; d=[json.loads(l) for l in sys.stdin if l.startswith('{')][0]; print(d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['stages'].items()})"; }
for cfg in dit wan13; do
  for v in base fpoly bpoly; do
    if [ $v = base ]; then lib=""; else lib=paper_2505_13389_b200/_lib/variants/libvsa_$v.so; fi
    echo -n "$cfg $v: "; VSA_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --no-dense --no-cpu --steps 10 2>&1 | summ
  done
done > gpurun_out/d64.txt 2>&1
cat gpurun_out/mufu.txt gpurun_out/d64.txt
