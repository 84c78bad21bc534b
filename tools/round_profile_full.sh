# One ncu --set full capture of each GEMM of one glm9b step (4 forward row chunks, grad_W,
# grad_hidden) and of the merge kernel; summaries via tools/ncu_summary.py.  One GPU.
C=${CONFIG:-glm9b}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100 -c 6 \
    -o gpurun_out/full_gemm_$C python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu \
    > gpurun_out/full_gemm_$C.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_merge_g -c 1 \
    -o gpurun_out/full_merge_$C python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu \
    > gpurun_out/full_merge_$C.log 2>&1
for r in full_gemm_$C full_merge_$C; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/$r.raw.csv > gpurun_out/$r.summary.txt
done
