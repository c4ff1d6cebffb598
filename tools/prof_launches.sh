# launch list of one bench device step (ncu, serialized, cold): per-kernel durations
CMD="python tools/prof_gauss.py --case kusari --mode phase --reps 3"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log
