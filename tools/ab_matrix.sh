# Whole-step A/B matrix on the GPU box: library variants x environment switches, twice.
#   VARIANTS="v1 v2" ENVS="X=1 Y=0" bash tools/ab_matrix.sh
for r in 1 2; do
for v in base $VARIANTS; do
for e in none $ENVS; do
  if [ "$v" = base ]; then unset LINKCERT_LIB; else export LINKCERT_LIB=paper_2106_12655_b200/_build_$v/liblinkcert_b200.so; fi
  if [ "$e" = none ]; then envs=""; else envs="$e"; fi
  env $envs python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$e', round(d['ms_per_step'],4), {k: round(v, 4) for k, v in d['stage_ms'].items()})"
done; done; done
