mkdir -p gpurun_out/s5
timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py tests/test_gpu_random.py -x -q > gpurun_out/s5/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s5/tests.log
timeout 900 python tools/small_sweep.py --json gpurun_out/s5/sweep.json > gpurun_out/s5/sweep.log 2>&1
