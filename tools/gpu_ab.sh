#!/bin/bash
# A/B harness: quick d=64/d=128 parity (hang guard), then bench lines for the default library and
# the variant libraries named on the command line (paper_2505_13389_b200/_lib/variants/libvsa_<name>.so).
# usage: tools/gpu_ab.sh "<pytest -k expr>" "<configs>" <variant>...
mkdir -p gpurun_out
kexpr=${1:-"tiny or padded or odd or maskpad or dit or sweep"}; cfgs=${2:-"dit"}; shift 2
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_maskpad.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "$kexpr" > gpurun_out/ab_quick.log 2>&1; echo "quick rc=$?" >> gpurun_out/ab_quick.log
tail -3 gpurun_out/ab_quick.log
grep -q "quick rc=0" gpurun_out/ab_quick.log || exit 1
for cfg in $cfgs; do
  for v in base "$@"; do
    lib=""; [ $v != base ] && lib=paper_2505_13389_b200/_lib/variants/libvsa_$v.so
    VSA_LIB_PATH=$lib timeout 300 python bench.py --config $cfg --no-cpu --no-dense > gpurun_out/ab_${cfg}_$v.log 2>&1
    python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/ab_${cfg}_$v.log') if l.startswith('{')][0]
print('$cfg $v', d['ms_per_step'], {k: v['ms'] for k, v in d['stages'].items()})" 2>/dev/null || echo "$cfg $v FAILED"
  done
done
