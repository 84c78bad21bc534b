# per-rank compute of the glm9b strong-scaling shards on one GPU (AGENTRL_BENCH_SHARD = n: rank
# 0's LPT shard of an n-GPU run, no communication), interleaved twice with the full batch
python paper_2510_04206_b200/build.py > /dev/null
for r in 1 2; do
  for n in 1 2 4 8; do
    AGENTRL_BENCH_SHARD=$n timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/sh.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/sh.json')); print('SHARD', $n, round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['config'].get('T'), d['config'].get('T_eff'))" | tee -a gpurun_out/shard_proj.txt
  done
done
