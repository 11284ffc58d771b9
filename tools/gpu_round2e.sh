#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_e.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_e.log
tail -15 gpurun_out/pytest_e.log
python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/bench_e.log') if l.startswith('{')][0]
print(d['coarse_mode'], d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['stages'].items()}, d['other_coarse_mode'])"
