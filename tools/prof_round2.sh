# Round-2 profile set (GPU box): bench line, launch list of the step, full ncu of the fused
# Gauss kernel (pair-claiming, Kusari), FP64 op counts per segment pair (torus 2,3 x 1024:
# phase / atan / ref / anglesum; ribbon 100k phase).  Each ncu run is preceded by the same
# command exiting 0 without ncu.
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/step_table.py gpurun_out/launches.csv > gpurun_out/step_table.md
python tools/prof_gauss.py --case kusari --mode phase --reps 3 > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_pairs -s 2 -c 1 -o gpurun_out/gauss_pairs_kusari python tools/prof_gauss.py --case kusari --mode phase --reps 3 > gpurun_out/ncu_full.log 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for mode in ref atan phase anglesum; do
python tools/prof_gauss.py --case torus --mode $mode --reps 1 > gpurun_out/plain_torus_$mode.log 2>&1 && \
ncu --metrics $M --clock-control none --csv -k regex:gauss_items --log-file gpurun_out/counts_torus_$mode.csv python tools/prof_gauss.py --case torus --mode $mode --reps 1 > gpurun_out/ncu_torus_$mode.log 2>&1
done
python tools/prof_gauss.py --case ribbon --n 100000 --mode phase --reps 1 > gpurun_out/plain_ribbon.log 2>&1 && \
ncu --metrics $M --clock-control none --csv -k regex:gauss_items --log-file gpurun_out/counts_ribbon_phase.csv python tools/prof_gauss.py --case ribbon --n 100000 --mode phase --reps 1 > gpurun_out/ncu_ribbon.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu.txt; lscpu > gpurun_out/lscpu.txt
