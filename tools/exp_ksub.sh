# A/B of forward-GEMM options on the glm9b bench (usage: bash tools/exp_ksub.sh)
python -m pytest tests -m gpu -x -q -k "not slow" 2>&1 | tail -3
for v in "1 1" "2 1" "2 4" "2 8" "2 4"; do set -- $v
  AGENTRL_FWD_KSUB=$1 AGENTRL_FWD_CHUNKS=$2 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_$1_$2.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_$1_$2.json'));print('ksub $1 chunks $2',round(d['ms_per_step'],2),d['clocks']['sm_mhz'],d['gpu_launches'],{k:round(v[0],2) for k,v in d['kernel_ms'].items()})"
done
