# Whole-step A/B on the GPU box: product build vs variant builds
# (python -m paper_2106_12655_b200.build --variant NAME ...), interleaved twice.
#   VARIANTS="name1 name2" bash tools/ab_frontend.sh
for r in 1 2; do
for v in base $VARIANTS; do
  if [ "$v" = base ]; then unset LINKCERT_LIB; else export LINKCERT_LIB=paper_2106_12655_b200/_build_$v/liblinkcert_b200.so; fi
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), d['stage_ms'])"
done; done
