# Interleaved A/B of library builds of the fused step (same box, R rounds; box-to-box clock
# spread under the power cap is +-3%, so defaults are chosen by same-box alternation):
#   LIBS="default build/ref_merge/paper_2510_04206_b200/libagentrl.so" R=3 bash tools/exp_ab.sh
# (a variant name from build.py VARIANTS is resolved to build/variants/<name>/libagentrl.so;
# ARGS is passed to every bench run)
for r in $(seq ${R:-3}); do
  for v in ${LIBS:-default}; do
    if [ "$v" = default ]; then e=""
    elif [ -f "$v" ]; then e="AGENTRL_LIB=$v"
    else e="AGENTRL_LIB=build/variants/$v/libagentrl.so"; fi
    env $e timeout 600 python bench.py --no-cpu --no-e2e --steps ${STEPS:-10} $ARGS > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {n: round(v[0],2) for n, v in k.items() if v[0] > 1})"
  done
done
