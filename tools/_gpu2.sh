set -x
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python tools/dist_threads.py > $O/dist.log 2>&1; echo "dist rc=$?" >> $O/dist.log
timeout 900 python tools/dist_threads.py --config5-strip > $O/dist5.log 2>&1; echo "dist5 rc=$?" >> $O/dist5.log
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_baseline_configs.py::test_config4_full_16384_equal_reference > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench.json 2> $O/bench.err
