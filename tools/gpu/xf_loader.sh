# XF transform with a loader warp for its inputs: parity, A/B vs the merge build, ncu, adv sweep
set -o pipefail
python tools/probe_multicast.py > gpurun_out/probe_mc.txt 2>&1
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
(cd ab_ref && python paper_2510_04206_b200/build.py > /dev/null)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/ld_pytest.log
timeout 600 python tools/adv_sweep.py --sizes 17 --configs glm9b,qwen7b,skew14b,qwen32b --iters 30 > gpurun_out/adv_sweep7.jsonl 2>&1
for r in 1 2 3; do
  for v in default ref; do
    if [ $v = ref ]; then (cd ab_ref && timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > /root/repo/gpurun_out/ab.json 2>/dev/null)
    else timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab.json 2>/dev/null; fi
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1000,1), {n: round(v[0],2) for n, v in k.items() if v[0] > 1})" | tee -a gpurun_out/ab_loader.txt
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100_pair_kernel --launch-skip 1 --launch-count 2 \
   -o gpurun_out/bwd_loader -f python tools/one_step.py qwen7b > gpurun_out/ncu_bwd_loader.log 2>&1
ncu -i gpurun_out/bwd_loader.ncu-rep --page raw --csv > gpurun_out/bwd_loader.raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_bwd_loader.log
