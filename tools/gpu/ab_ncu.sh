# interleaved A/B of the XF build (.) against the merge build (ab_ref = bcab47c), then ncu --set
# full of both builds' backward GEMMs at qwen7b.  One GPU.
python paper_2510_04206_b200/build.py > /dev/null
(cd ab_ref && python paper_2510_04206_b200/build.py > /dev/null)
for r in 1 2 3; do
  for tree in . ab_ref; do
    (cd $tree && timeout 600 python bench.py --no-cpu --no-e2e --steps 10 > /root/repo/gpurun_out/ab.json 2>/dev/null)
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d.get('kernel_ms', {}); print('AB', '$tree', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1000,1), {n: round(v[0],2) for n, v in k.items() if v[0] > 1})" | tee -a gpurun_out/ab_xf_vs_merge.txt
  done
done
for tree in . ab_ref; do
  tag=$( [ "$tree" = "." ] && echo xf || echo ref )
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100_pair_kernel --launch-skip 1 --launch-count 2 \
     -o gpurun_out/bwd_$tag -f python $tree/tools/one_step.py qwen7b > gpurun_out/ncu_bwd_$tag.log 2>&1
  ncu -i gpurun_out/bwd_$tag.ncu-rep --page raw --csv > gpurun_out/bwd_$tag.raw.csv 2>/dev/null
  ncu -i gpurun_out/bwd_$tag.ncu-rep --page details --csv > gpurun_out/bwd_$tag.details.csv 2>/dev/null
  tail -2 gpurun_out/ncu_bwd_$tag.log
done
ls -la gpurun_out/bwd_*
