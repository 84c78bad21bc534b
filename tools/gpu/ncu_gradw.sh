# ncu --set full of the grad_W GEMM (qwen7b): the XF build and the previous merge build
python paper_2510_04206_b200/build.py > /dev/null
M="gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum"
for tree in . build/ref_merge; do
  tag=$( [ "$tree" = "." ] && echo xf || echo ref )
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100_pair_kernel --launch-skip 1 --launch-count 2 \
     -o gpurun_out/gradw_$tag -f python $tree/tools/one_step.py qwen7b > gpurun_out/ncu_gradw_$tag.log 2>&1
  ncu -i gpurun_out/gradw_$tag.ncu-rep --page details --csv > gpurun_out/gradw_$tag.details.csv 2>/dev/null
  ncu -i gpurun_out/gradw_$tag.ncu-rep --page raw --csv > gpurun_out/gradw_$tag.raw.csv 2>/dev/null
  ncu -i gpurun_out/gradw_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/gradw_$tag.sass.csv 2>/dev/null
  tail -3 gpurun_out/ncu_gradw_$tag.log
done
ls -la gpurun_out/gradw_*
