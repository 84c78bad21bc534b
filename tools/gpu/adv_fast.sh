set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 300 python tools/adv_sweep.py --sizes 20,24,27 --iters 20 > gpurun_out/adv_sweep13.jsonl 2>&1; cut -c1-200 gpurun_out/adv_sweep11.jsonl
timeout 1500 python -m pytest tests/test_gpu_adv_layouts.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_edge_cases.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/adv_fast3_pytest.log
