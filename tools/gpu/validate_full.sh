# round validation on one GPU: full GPU suite, bench line, launch list + per-kernel DRAM bytes,
# one ncu --set full capture of the three GEMMs of a glm9b step
set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; tail -c 600 gpurun_out/bench_main.json
bash tools/round_profile.sh
cat gpurun_out/launches_glm9b_summary.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_sm100 -c 3 \
    -o gpurun_out/full_gemm_glm9b -f python bench.py --config glm9b --steps 1 --warmup 0 --no-e2e --no-cpu \
    > gpurun_out/full_gemm_glm9b.log 2>&1
ncu -i gpurun_out/full_gemm_glm9b.ncu-rep --page raw --csv > gpurun_out/full_gemm_glm9b.raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/full_gemm_glm9b.raw.csv > gpurun_out/full_gemm_glm9b.summary.txt; cat gpurun_out/full_gemm_glm9b.summary.txt | grep -E "===|time_dur|tensor_cycles_active.avg|dram__bytes"
