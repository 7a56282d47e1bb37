mkdir -p gpurun_out/s8
timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py tests/test_gpu_random.py -x -q > gpurun_out/s8/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s8/tests.log
LF_SMALL_GRID=1 timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/s8/tests_grid.log 2>&1; echo "rc=$?" >> gpurun_out/s8/tests_grid.log
LF_SMALL_GRID=0 timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/s8/tests_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/s8/tests_cluster.log
