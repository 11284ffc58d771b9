#!/bin/bash
# Round-end style check on one B200: GPU test suite, default bench line, reference arm.
mkdir -p gpurun_out
tag=${1:-check}
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/benchref_$tag.log 2>&1; echo "ref rc=$?" >> gpurun_out/benchref_$tag.log
tail -5 gpurun_out/pytest_$tag.log
tail -3 gpurun_out/bench_$tag.log | cut -c1-1500
tail -2 gpurun_out/benchref_$tag.log | cut -c1-600
