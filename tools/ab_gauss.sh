# Gauss-kernel A/B on the GPU box: product build modes + variant builds (python -m ...build --variant NAME -D ...)
for v in "" $VARIANTS; do
  if [ -n "$v" ]; then export LINKCERT_LIB=paper_2106_12655_b200/_build_$v/liblinkcert_b200.so; else unset LINKCERT_LIB; fi
  echo "== variant ${v:-base}"; python tools/kbench.py --modes ${MODES:-0} --reps 10 2>&1 | grep -v "^$"
done
