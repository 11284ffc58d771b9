#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_c.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c.log
tail -15 gpurun_out/pytest_c.log; tail -c 600 gpurun_out/bench_c.log
