# full GPU validation + bench + profiles (one gpurun call)
set -o pipefail
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; tail -c 1500 gpurun_out/bench_main.json
bash tools/round_profile.sh
cat gpurun_out/launches_glm9b_summary.txt
