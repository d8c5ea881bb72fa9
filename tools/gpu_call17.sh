timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02_pytest_persist.log 2>&1; tail -3 gpurun_out/r02_pytest_persist.log
timeout 300 python tools/order_sweep.py 2 4 8 12 16 2>&1
