# quick validation + bench (one gpurun call)
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_loss_variants.py tests/test_gpu_adv_layouts.py -x -q 2>&1 | tail -4 | tee gpurun_out/quick_pytest.log
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python -c "
import json; d=json.load(open('gpurun_out/quick_bench.json')); print('ms', d['ms_per_step'], 'mhz', d['clocks']['sm_mhz'], {k: round(v[0],3) for k, v in d['kernel_ms'].items()}, 'adv', d['adv_norm']['latency_us'], d['adv_norm']['bandwidth_point'])"
timeout 300 python tools/adv_sweep.py --sizes 24,27 --configs glm9b --iters 10 > gpurun_out/quick_adv.jsonl 2>&1; cat gpurun_out/quick_adv.jsonl
