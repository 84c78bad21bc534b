# head validation on one GPU: full GPU suite, bench line, launch list + per-kernel DRAM, sanitizer
set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; tail -c 3000 gpurun_out/bench_main.json
bash tools/round_profile.sh
cat gpurun_out/launches_glm9b_summary.txt
bash tools/gpu/sanitize.sh
