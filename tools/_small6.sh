mkdir -p gpurun_out/s6
timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/s6/small.log 2>&1; echo "rc=$?" >> gpurun_out/s6/small.log
