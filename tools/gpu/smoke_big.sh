python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 900 python bench.py --config qwen32b --no-cpu --steps 3 > gpurun_out/bench_qwen32b_1gpu.json 2> gpurun_out/bench_qwen32b_1gpu.err; tail -c 300 gpurun_out/bench_qwen32b_1gpu.json; tail -3 gpurun_out/bench_qwen32b_1gpu.err
timeout 900 python bench.py --config skew14b --no-cpu --steps 5 > gpurun_out/bench_skew14b_1gpu.json 2> gpurun_out/bench_skew14b_1gpu.err; tail -c 300 gpurun_out/bench_skew14b_1gpu.json
