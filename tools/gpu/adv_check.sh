# new small adv-norm driver + vocab-parallel row stats: the affected GPU tests, the latency sweep
set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 1500 python -m pytest tests/test_gpu_adv_layouts.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_vocab_parallel.py tests/test_gpu_edge_cases.py tests/test_gpu_graph.py tests/test_gpu_loss_variants.py -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/adv_pytest.log
timeout 300 python tools/adv_sweep.py --sizes 17,20,24,27 --iters 20 > gpurun_out/adv_sweep.jsonl 2>&1; cat gpurun_out/adv_sweep.jsonl
