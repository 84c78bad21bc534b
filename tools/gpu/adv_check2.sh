set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
timeout 300 python tools/adv_sweep.py --sizes 17 --configs glm9b,qwen7b,skew14b,qwen32b --iters 30 > gpurun_out/adv_sweep8.jsonl 2>&1; cat gpurun_out/adv_sweep8.jsonl | cut -c1-250
timeout 1500 python -m pytest tests/test_gpu_adv_layouts.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_edge_cases.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/adv2_pytest.log
