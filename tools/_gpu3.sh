set -x
O=gpurun_out/r2c; mkdir -p $O
export LF_NCCL_LIB=$PWD/tests/fake_nccl/libfakenccl.so
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_baseline_configs.py::test_config4_full_16384_equal_reference > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for M in exact contract; do
  python tools/prof_steps.py 16384 3 fused $M > $O/plain_f_$M.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 \
      -o gpurun_out/prof_f16k_${M}_r02c python tools/prof_steps.py 16384 3 fused $M > $O/ncu_f_$M.log 2>&1
done
