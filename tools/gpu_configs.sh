#!/bin/bash
# bench line of every BASELINE config on one B200 (+ the dense baseline where it fits), and the paper sweep
mkdir -p gpurun_out
tag=${1:-r2}
for cfg in wan13 dit sweep32 wan14 tiny; do
  extra=""; [ $cfg = wan14 ] && extra="--no-dense"
  timeout 900 python bench.py --config $cfg --no-cpu $extra > gpurun_out/cfg_${tag}_$cfg.log 2>&1
  python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/cfg_${tag}_$cfg.log') if l.startswith('{')][0]
print('$cfg', d['ms_per_step'], d['value'], 'dense', (d.get('dense_baseline') or {}).get('speedup_vsa_vs_dense'), {k: v['ms'] for k, v in d['stages'].items()})" || tail -3 gpurun_out/cfg_${tag}_$cfg.log
done
timeout 1200 python tools/sweep.py --out gpurun_out/sweep_${tag}.json > gpurun_out/sweep_${tag}.log 2>&1; echo "sweep rc=$?"
