# new tests + smoke + the reference arm on one GPU box
set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_bench_multirank.py -q -m gpu 2>&1 | tail -3 | tee gpurun_out/quick_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/quick_smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/quick_ref.json 2> gpurun_out/quick_ref.err; tail -c 800 gpurun_out/quick_ref.json
