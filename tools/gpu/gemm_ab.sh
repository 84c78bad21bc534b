# one GEMM schedule/epilogue switch: parity, interleaved bench A/B on one lease against the
# variant build $1 (the old behaviour), ncu of the GEMM kernels $2 (skip count) for both
set -o pipefail
V=$1; SKIP=${2:-1}
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
if [ -f "$V" ]; then P0=$PWD/$V; else  # a library path (e.g. ab_head/libagentrl.so) or a variant name
P0=$(python -c "import sys; sys.path.insert(0,'tests'); from variants import variant_env; print(variant_env('$V')['AGENTRL_LIB'])")
fi
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vocab_parallel.py tests/test_gpu_multirank.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/gab_pytest.log
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -m gpu -k "pair0 or ksplit3" 2>&1 | tail -2 | tee -a gpurun_out/gab_pytest.log
rm -f gpurun_out/gab_ab.txt
for r in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export AGENTRL_LIB=$P0; else unset AGENTRL_LIB; fi
    timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1000,1), {n: round(v[0],2) for n, v in k.items() if v[0] > 1})" | tee -a gpurun_out/gab_ab.txt
  done
done
unset AGENTRL_LIB
for v in new old; do
  if [ $v = old ]; then export AGENTRL_LIB=$P0; else unset AGENTRL_LIB; fi
  timeout 900 ncu --set full --clock-control none -k regex:gemm_sm100_pair_kernel --launch-skip $SKIP -c 1 \
     -o gpurun_out/gab_$v -f python tools/one_step.py glm9b > gpurun_out/ncu_gab_$v.log 2>&1
  ncu -i gpurun_out/gab_$v.ncu-rep --page raw --csv > gpurun_out/gab_$v.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/gab_$v.raw.csv | tee gpurun_out/gab_$v.summary.txt | grep -E "===|time_dur|tensor_cycles_active.avg|dram__bytes|cycles_elapsed.max"
done
unset AGENTRL_LIB
