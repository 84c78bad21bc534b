# A/B of two schedule builds against the default at glm9b (3 interleaved rounds); the variant names are set below (last run: forward raster group 16 vs 12 vs 24)
set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
L64=$(python -c "import sys; sys.path.insert(0,'tests'); from variants import variant_env; print(variant_env('gm12')['AGENTRL_LIB'])")
L160=$(python -c "import sys; sys.path.insert(0,'tests'); from variants import variant_env; print(variant_env('gm24')['AGENTRL_LIB'])")
rm -f gpurun_out/sched_ab.txt
for r in 1 2 3; do
  for v in new l64 l160; do
    case $v in new) unset AGENTRL_LIB ;; l64) export AGENTRL_LIB=$L64 ;; l160) export AGENTRL_LIB=$L160 ;; esac  # l64 / l160: the two variant builds named above
    timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1000,1), {n: round(v[0],2) for n, v in k.items() if v[0] > 1})" | tee -a gpurun_out/sched_ab.txt
  done
done
