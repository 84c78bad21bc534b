# L2 prefetch ahead of the backward GEMMs' TMA ring: interleaved A/B (glm9b), bitwise check
set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
python -c "
import importlib.util; s=importlib.util.spec_from_file_location('b','paper_2510_04206_b200/build.py'); b=importlib.util.module_from_spec(s); s.loader.exec_module(b); b.build_variant('pf0'); b.build_variant('pf16')" > /dev/null
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -m gpu -k "pf0" 2>&1 | tail -2 | tee gpurun_out/pf_pytest.log
for r in 1 2 3; do
  for v in default pf0 pf16; do
    if [ $v = default ]; then e=""; else e="AGENTRL_LIB=build/variants/$v/libagentrl.so"; fi
    env $e timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1000,1), {n: round(v[0],2) for n, v in k.items() if v[0] > 1})" | tee -a gpurun_out/ab_pf.txt
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100_pair_kernel --launch-skip 1 --launch-count 2 \
   -o gpurun_out/bwd_pf -f python tools/one_step.py glm9b > gpurun_out/ncu_bwd_pf.log 2>&1
ncu -i gpurun_out/bwd_pf.ncu-rep --page raw --csv > gpurun_out/bwd_pf.raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/bwd_pf.raw.csv | grep -E "===|time_dur|tensor_cycles_active.avg|dram__bytes|cycles_elapsed.max"
