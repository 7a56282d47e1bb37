set -x
O=gpurun_out/r2e; mkdir -p $O
for M in exact contract; do
  python tools/prof_steps.py 16384 3 fused $M > $O/plain_f_$M.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 \
      -o gpurun_out/prof_f16k_${M}_r02e python tools/prof_steps.py 16384 3 fused $M > $O/ncu_f_$M.log 2>&1
done
