# Refresh of the round-2 bench artefacts at HEAD (GPU box): bench line, reference
# arm, launch list + step table, and the pass-1 kernel's ncu summary.  Each ncu run is
# preceded by the same command exiting 0 without ncu.
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/step_table.py gpurun_out/launches.csv > gpurun_out/step_table.md
python tools/step_time.py --steps 3 > gpurun_out/plain_step.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:brute_any -c 1 -o gpurun_out/brute_any_kusari python tools/step_time.py --steps 3 > gpurun_out/ncu_brute.log 2>&1
python tools/prof_gauss.py --case kusari --mode phase --reps 3 > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_pairs -s 2 -c 1 -o gpurun_out/gauss_pairs_kusari python tools/prof_gauss.py --case kusari --mode phase --reps 3 > gpurun_out/ncu_full.log 2>&1
