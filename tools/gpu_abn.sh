#!/bin/bash
# Interleaved A/B: N rounds of (default library, variants...) on one config, printing the
# per-stage times of every run (the box's power / thermal state drifts between runs, so
# a single A-then-B pair is not evidence). usage: tools/gpu_abn.sh <config> <rounds> <variant>...
mkdir -p gpurun_out
cfg=$1; n=$2; shift 2
for i in $(seq 1 $n); do
  for v in base "$@"; do
    lib=""; [ $v != base ] && lib=paper_2505_13389_b200/_lib/variants/libvsa_$v.so
    VSA_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --no-cpu --no-dense > gpurun_out/abn_${cfg}_$v.log 2>&1
    python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/abn_${cfg}_$v.log') if l.startswith('{')][0]
s=d['stages']; print('$cfg %-6s' % '$v', d['ms_per_step'], 'fwd', s['fine_fwd']['ms'], 'bwd', s['fine_bwd']['ms'])" 2>/dev/null || echo "$cfg $v FAILED"
  done
done
