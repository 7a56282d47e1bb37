# Round-2 evidence on one GPU (run from the repo root under gpurun; outputs in gpurun_out/):
# ncu --set full of the fused step in both arithmetics at 16384^2 (each only after the
# same command exited 0 without ncu) and the launch list of a short bench run.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
for M in exact contract; do
  python tools/prof_steps.py 16384 3 fused $M > gpurun_out/plain_f_$M.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 \
      -o gpurun_out/prof_f16k_${M}_$TAG python tools/prof_steps.py 16384 3 fused $M \
      > gpurun_out/ncu_f_$M.log 2>&1
done
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-contract > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu \
    --no-e2e --no-contract > gpurun_out/ncu_l.log 2>&1
ls -la gpurun_out
