CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_brute.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"brute_any|grid_query_warp" -c 2 -o gpurun_out/brute $CMD > gpurun_out/ncu_brute.log 2>&1
tail -n 2 gpurun_out/ncu_brute.log
