mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "pipeline or host" -p no:cacheprovider > gpurun_out/e2e_test.log 2>&1; echo rc=$? >> gpurun_out/e2e_test.log
timeout 600 python tools/e2e_sweep.py > gpurun_out/e2e_sweep.log 2>&1; echo rc=$? >> gpurun_out/e2e_sweep.log
timeout 120 python tools/pcie_probe.py >> gpurun_out/e2e_sweep.log 2>&1
tail -3 gpurun_out/e2e_test.log; cat gpurun_out/e2e_sweep.log
