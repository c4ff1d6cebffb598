for v in "" pc pi pci; do
  if [ -n "$v" ]; then export LINKCERT_LIB=paper_2106_12655_b200/_build_$v/liblinkcert_b200.so; else unset LINKCERT_LIB; fi
  echo "== variant ${v:-base}"; python tools/kbench.py --modes 0 --reps 10 2>&1 | grep -v "^$"
done
unset LINKCERT_LIB
python tools/prof_gauss.py --case kusari --mode phase --reps 2 > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gauss_items -s 1 -c 1 -o gpurun_out/gauss_phase_kusari python tools/prof_gauss.py --case kusari --mode phase --reps 2 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
