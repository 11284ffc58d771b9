#!/bin/bash
# Experimental d = 64 ping-pong forward (VSA_FWD_PP=1): hang check (3 runs of the poly timing variant),
# parity tests with the kernel enabled, DiT bench A/B.
mkdir -p gpurun_out
for i in 1 2 3; do
  VSA_FWD_PP=1 VSA_LIB_PATH=paper_2505_13389_b200/_lib/variants/libvsa_poly2.so timeout 120 python bench.py --config dit --no-cpu --no-dense > gpurun_out/pp_poly2_$i.log 2>&1
  echo "poly2 run $i rc=$? $(grep -o '"fine_fwd": {"ms": [0-9.]*' gpurun_out/pp_poly2_$i.log)"
done
VSA_FWD_PP=1 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/pp_pytest.log 2>&1; echo "pytest (pp) rc=$?"; tail -2 gpurun_out/pp_pytest.log
for v in 1 0 1 0; do
  VSA_FWD_PP=$v timeout 300 python bench.py --config dit --no-cpu --no-dense 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('dit VSA_FWD_PP=$v', d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()})"
done
