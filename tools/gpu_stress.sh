#!/bin/bash
# Hang stress of the d = 64 forward: bench runs (default and a timing variant), the sweep, tiny configs
mkdir -p gpurun_out
for i in 1 2 3 4 5; do
  timeout 120 python bench.py --config dit --no-cpu --no-dense > gpurun_out/st_$i.log 2>&1; echo "dit $i rc=$? $(grep -o '"fine_fwd": {"ms": [0-9.]*' gpurun_out/st_$i.log)"
done
for i in 1 2 3; do
  VSA_LIB_PATH=paper_2505_13389_b200/_lib/variants/libvsa_poly2.so timeout 120 python bench.py --config dit --no-cpu --no-dense > gpurun_out/stp_$i.log 2>&1; echo "poly2 $i rc=$?"
done
timeout 120 python bench.py --config tiny --no-cpu > gpurun_out/st_tiny.log 2>&1; echo "tiny rc=$?"
timeout 600 python tools/sweep.py --reps 10 --dims 64 --out gpurun_out/sweep_d64.json > gpurun_out/sweep_d64.log 2>&1; echo "sweep d64 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/sweep_d64.json'))
for r in d['rows']: print(r['grid'], r['k'], r['fine_fwd_ms'], r['fine_fwd_tflops'], r['fine_bwd_tflops'], r['speedup_step'])"
