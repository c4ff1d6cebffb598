set -x
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/prof_gauss.py --case kusari --mode phase --reps 2 > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_items -s 1 -c 1 -o gpurun_out/gauss_phase_kusari python tools/prof_gauss.py --case kusari --mode phase --reps 2 > gpurun_out/ncu_full.log 2>&1
for mode in ref atan phase; do
python tools/prof_gauss.py --case torus --mode $mode --reps 1 > gpurun_out/plain_torus_$mode.log 2>&1 && \
ncu --metrics $M --clock-control none --csv -k regex:gauss_items --log-file gpurun_out/counts_torus_$mode.csv python tools/prof_gauss.py --case torus --mode $mode --reps 1 > gpurun_out/ncu_torus_$mode.log 2>&1
done
ls -la gpurun_out
