# NVTX ranges: tests still pass, the bench is unchanged, and ncu filters kernels by range
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/nvtx_pytest.log
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/nvtx_bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/nvtx_bench.json')); print('bench', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['gpu_launches'])"
timeout 600 ncu --nvtx --nvtx-include "agentrl_grpo_step/gemm_grad_W/" --metrics gpu__time_duration.sum -c 2 python tools/one_step.py qwen7b > gpurun_out/nvtx_ncu.log 2>&1; grep -E "gemm|==PROF==|NVTX" gpurun_out/nvtx_ncu.log | head -12
