# Round profile set (GPU box): bench line, launch list, full ncu of the Gauss kernel and of the
# front-end kernels, FP64 op counts.  Each ncu run is preceded by the same command exiting 0 without ncu.
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/step_table.py gpurun_out/launches.csv > gpurun_out/step_table.md
python tools/prof_gauss.py --case kusari --mode phase --reps 2 > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_items -s 1 -c 1 -o gpurun_out/gauss_phase_kusari python tools/prof_gauss.py --case kusari --mode phase --reps 2 > gpurun_out/ncu_full.log 2>&1
bash tools/prof_stages.sh
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
for mode in ref atan phase; do
python tools/prof_gauss.py --case torus --mode $mode --reps 1 > gpurun_out/plain_torus_$mode.log 2>&1 && \
ncu --metrics $M --clock-control none --csv -k regex:gauss_items --log-file gpurun_out/counts_torus_$mode.csv python tools/prof_gauss.py --case torus --mode $mode --reps 1 > gpurun_out/ncu_torus_$mode.log 2>&1
done
python tools/prof_gauss.py --case ribbon --n 100000 --mode phase --reps 1 > gpurun_out/plain_ribbon.log 2>&1 && \
ncu --metrics $M --clock-control none --csv -k regex:gauss_items --log-file gpurun_out/counts_ribbon_phase.csv python tools/prof_gauss.py --case ribbon --n 100000 --mode phase --reps 1 > gpurun_out/ncu_ribbon.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/gpu.txt; lscpu > gpurun_out/lscpu.txt
# Barnes-Hut (csrc/bh.cu): probe line + launch list of its kernels (forest build, traversal levels)
python tools/bh_probe.py --sizes 1000000 --ds-max 0 > gpurun_out/bh_probe.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:bh_ -c 400 --log-file gpurun_out/bh_launches.csv python tools/bh_probe.py --sizes 1000000 --ds-max 0 > gpurun_out/ncu_bh.log 2>&1
