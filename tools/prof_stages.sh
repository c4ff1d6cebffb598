# Full ncu sections for the non-Gauss kernels of one fused pipeline run (GPU box).
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_stages.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"brute_kernel|grid_query_warp|seg_boxes|loop_boxes|export_results|write_all|DeviceScanKernel" \
    -c 9 -o gpurun_out/stages $CMD > gpurun_out/ncu_stages.log 2>&1
tail -n 3 gpurun_out/ncu_stages.log
