mkdir -p gpurun_out/mm
timeout 900 python -m pytest tests/test_gpu_multimat.py -x -q > gpurun_out/mm/tests.log 2>&1; echo "rc=$?" >> gpurun_out/mm/tests.log
timeout 600 python bench.py --workload triple_point --steps 100 --warmup 5 > gpurun_out/mm/tp.json 2> gpurun_out/mm/tp.err
