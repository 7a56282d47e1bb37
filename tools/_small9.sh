mkdir -p gpurun_out/s9
timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/s9/small.log 2>&1; echo "rc=$?" >> gpurun_out/s9/small.log
timeout 900 python -m pytest tests/test_gpu_multimat.py tests/test_gpu_random.py tests/test_gpu_parity.py -x -q > gpurun_out/s9/rest.log 2>&1; echo "rc=$?" >> gpurun_out/s9/rest.log
