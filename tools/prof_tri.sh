CMD="python tools/prof_gauss.py --case kusari --mode phase --reps 2"
$CMD > gpurun_out/plain_tri.log 2>&1 && \
ncu --set full --clock-control none -k regex:tri_slots -s 1 -c 1 -o gpurun_out/tri $CMD > gpurun_out/ncu_tri.log 2>&1
tail -n 2 gpurun_out/ncu_tri.log
