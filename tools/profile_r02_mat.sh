# Round-2 evidence for the multimaterial path on one GPU (run under gpurun; outputs in
# gpurun_out/): ncu --set full of the two-pass material kernels on the triple point at
# 8192x3512 (3 materials), after the same command exited 0 without ncu, and the bench line.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
python tools/prof_mat.py 8192 3512 4 > gpurun_out/plain_mat.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_pass_mat -s 4 -c 2 \
    -o gpurun_out/prof_mat_$TAG python tools/prof_mat.py 8192 3512 4 > gpurun_out/ncu_mat.log 2>&1
python bench.py --workload triple_point --steps 100 --warmup 5 > gpurun_out/tp_$TAG.json 2> gpurun_out/tp_$TAG.err
python tools/bench_triple_point.py > gpurun_out/tp_sizes_$TAG.log 2>&1
