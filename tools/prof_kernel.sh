# usage: bash tools/prof_kernel.sh <modes> <tag>   (profiles the first Kusari and first ribbon launch)
MODES=${1:-3}
TAG=${2:-p2}
CMD="python tools/kbench.py --modes $MODES --reps 1"
$CMD > gpurun_out/plain_kb_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_items -s 0 -c 1 -o gpurun_out/kb_${TAG}_kusari $CMD > gpurun_out/ncu_kb_$TAG.log 2>&1
$CMD > gpurun_out/plain_kb2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_items -s 3 -c 1 -o gpurun_out/kb_${TAG}_ribbon $CMD > gpurun_out/ncu_kb2_$TAG.log 2>&1
tail -n 3 gpurun_out/ncu_kb_$TAG.log gpurun_out/ncu_kb2_$TAG.log
