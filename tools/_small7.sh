mkdir -p gpurun_out/s7
timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py -x -q > gpurun_out/s7/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s7/tests.log
LF_SMALL_GRID=1 timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/s7/tests_grid.log 2>&1; echo "rc=$?" >> gpurun_out/s7/tests_grid.log
timeout 900 python tools/small_sweep.py --json gpurun_out/s7/sweep.json > gpurun_out/s7/sweep.log 2>&1
LF_SMALL_GRID=0 timeout 900 python tools/small_sweep.py --small-only --json gpurun_out/s7/sweep_cluster.json > gpurun_out/s7/sweep_cluster.log 2>&1
LF_SMALL_GRID=1 timeout 900 python tools/small_sweep.py --small-only --json gpurun_out/s7/sweep_grid.json > gpurun_out/s7/sweep_grid.log 2>&1
