# Round-end evidence on one GPU: bench (both arms), ncu launch list, ncu --set full captures.
# Run from the repo root under gpurun; outputs land in gpurun_out/ (summarise with tools/ncu_summary.py).
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_l.log 2>&1
python tools/prof_steps.py 16384 3 twopass > gpurun_out/plain_tp.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_pass -s 2 -c 2 -o gpurun_out/prof_tp16k_r1 python tools/prof_steps.py 16384 3 twopass > gpurun_out/ncu_tp.log 2>&1
python tools/prof_steps.py 16384 3 fused > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 -o gpurun_out/prof_f16k_r1 python tools/prof_steps.py 16384 3 fused > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out
