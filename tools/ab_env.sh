# Whole-step A/B of environment switches on the GPU box, interleaved twice:
#   ENVS="LINKCERT_PAIR_EXPORT=1 LINKCERT_X=1" bash tools/ab_env.sh
for r in 1 2; do
for e in base $ENVS; do
  if [ "$e" = base ]; then envs=""; else envs="$e"; fi
  env $envs python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', round(d['ms_per_step'],4), {k: round(v, 4) for k, v in d['stage_ms'].items()})"
done; done
