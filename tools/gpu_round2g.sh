#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g.log
timeout 300 python bench.py --no-cpu --no-dense > gpurun_out/bench_g.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_g.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_g.csv python tools/one_step.py > /dev/null 2>&1
tail -5 gpurun_out/pytest_g.log
python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/bench_g.log') if l.startswith('{')][0]
print(d['coarse_mode'], d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['stages'].items()}, d['other_coarse_mode'])"
python tools/launch_table.py gpurun_out/launches_g.csv
