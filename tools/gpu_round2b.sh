#!/bin/bash
# round-2 evidence run: new GPU tests, bench, sweep, ncu launch list + full capture of every kernel of one step
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_counters.py tests/test_gpu_cpp.py tests/test_gpu_bench_contract.py -q -x -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 300 python bench.py > gpurun_out/bench_b.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_b.log
timeout 600 python tools/sweep.py --out gpurun_out/sweep_r2.json > gpurun_out/sweep_b.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep_b.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r2a.csv python tools/one_step.py > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -c 20 -o gpurun_out/prof_r2a -f python tools/one_step.py > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
tail -3 gpurun_out/pytest_b.log; tail -c 1500 gpurun_out/bench_b.log; tail -3 gpurun_out/sweep_b.log; tail -3 gpurun_out/ncu_full.log
