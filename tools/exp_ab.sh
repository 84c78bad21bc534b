# Interleaved A/B of environment variants of the fused step (same box, R rounds):
#   VARIANTS="base AGENTRL_THROTTLE_LEAD=96 AGENTRL_GROUP_M_BWD=16" R=3 bash tools/exp_ab.sh
# (a variant may set several variables, comma-separated; COMMON is applied to every run)
for r in $(seq ${R:-3}); do
  for v in ${VARIANTS:-base}; do
    if [ "$v" = base ]; then e=""; else e="${v//,/ }"; fi
    env $COMMON $e timeout 600 python bench.py --no-cpu --no-e2e --steps ${STEPS:-10} > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {n: round(v[0],2) for n, v in k.items() if v[0] > 1})"
  done
done
