# bench lines at the final head: qwen7b (BASELINE configs[1]), qwen32b and skew14b whole batches
# on one GPU, and rank 0's per-rank compute of the glm9b 2/4/8-GPU shards (no communication)
python paper_2510_04206_b200/build.py > /dev/null
timeout 600 python bench.py --config qwen7b --no-cpu > gpurun_out/final_qwen7b.json 2> gpurun_out/final_qwen7b.err
timeout 900 python bench.py --config qwen32b --no-cpu --no-e2e --steps 5 > gpurun_out/final_qwen32b.json 2> gpurun_out/final_qwen32b.err
timeout 900 python bench.py --config skew14b --no-cpu --no-e2e --steps 5 > gpurun_out/final_skew14b.json 2> gpurun_out/final_skew14b.err
for n in 2 4 8; do
  AGENTRL_BENCH_SHARD=$n timeout 600 python bench.py --no-cpu --no-e2e --steps 20 > gpurun_out/final_shard$n.json 2> gpurun_out/final_shard$n.err
done
for f in gpurun_out/final_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['config'].get('workload'), round(d['ms_per_step'],2), round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"; done
