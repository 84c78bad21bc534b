# full GPU validation + bench + profiles (one gpurun call)
set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; tail -c 2500 gpurun_out/bench_main.json
bash tools/round_profile.sh
cat gpurun_out/launches_glm9b_summary.txt
