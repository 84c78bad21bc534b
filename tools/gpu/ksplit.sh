# grad_hidden split-K: parity (forced 3-way build), then per-rank compute of the 2/4/8-GPU glm9b
# shards and the 8-GPU skew14b shard on one GPU, heuristic default vs never-split, interleaved
set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
python -c "
import importlib.util; s=importlib.util.spec_from_file_location('b','paper_2510_04206_b200/build.py'); b=importlib.util.module_from_spec(s); s.loader.exec_module(b); b.build_variant('ksplit3'); b.build_variant('ksplit1')" > /dev/null
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -m gpu -k "ksplit3" 2>&1 | tail -3 | tee gpurun_out/ksplit_pytest.log
for r in 1 2; do
for cs in "glm9b 2" "glm9b 4" "skew14b 8"; do
  set -- $cs
  for v in default ksplit1; do
    if [ $v = default ]; then e=""; else e="AGENTRL_LIB=build/variants/$v/libagentrl.so"; fi
    env $e AGENTRL_BENCH_SHARD=$2 timeout 600 python bench.py --config $1 --no-cpu --no-e2e --steps 20 > gpurun_out/ks.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ks.json')); k=d.get('kernel_ms', {}); print('KS', '$1/$2', '$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {n: round(v[0],3) for n, v in k.items() if v[0] > 0.5})" | tee -a gpurun_out/ksplit_ab.txt
  done
done
done
