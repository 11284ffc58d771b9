#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_coarse_bf16.py -q -x -p no:cacheprovider > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f.log
timeout 300 python bench.py --no-cpu --no-dense > gpurun_out/bench_f.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_f.log
tail -5 gpurun_out/pytest_f.log
python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/bench_f.log') if l.startswith('{')][0]
print(d['coarse_mode'], d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['stages'].items()}, d['other_coarse_mode'])"
