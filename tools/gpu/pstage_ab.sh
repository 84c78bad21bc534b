# forward P~ stores staged through smem (full-sector rows) vs 16 B per row: parity, interleaved
# bench A/B on one lease, ncu of the forward GEMM for both builds
set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
P0=$(python -c "import sys; sys.path.insert(0,'tests'); from variants import variant_env; print(variant_env('pstage0')['AGENTRL_LIB'])")
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_logprob.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pstage_pytest.log
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -m gpu -k "pair0 or ksub1" 2>&1 | tail -2 | tee -a gpurun_out/pstage_pytest.log
rm -f gpurun_out/pstage_ab.txt
for r in 1 2 3; do
  for v in new p0; do
    if [ $v = p0 ]; then export AGENTRL_LIB=$P0; else unset AGENTRL_LIB; fi
    timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1000,1), {n: round(v[0],2) for n, v in k.items() if v[0] > 1})" | tee -a gpurun_out/pstage_ab.txt
  done
done
unset AGENTRL_LIB
for v in new p0; do
  if [ $v = p0 ]; then export AGENTRL_LIB=$P0; else unset AGENTRL_LIB; fi
  timeout 900 ncu --set full --clock-control none -k regex:gemm_sm100_pair_kernel -c 1 \
     -o gpurun_out/fwd_$v -f python tools/one_step.py glm9b > gpurun_out/ncu_fwd_$v.log 2>&1
  ncu -i gpurun_out/fwd_$v.ncu-rep --page raw --csv > gpurun_out/fwd_$v.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/fwd_$v.raw.csv | tee gpurun_out/fwd_$v.summary.txt | grep -E "time_dur|tensor_cycles_active.avg|dram__bytes|cycles_elapsed.max"
done
unset AGENTRL_LIB
