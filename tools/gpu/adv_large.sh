# three-launch large adv-norm driver: sweep, layout tests (all drivers), ncu of the launches at 2^27
set -o pipefail
python paper_2510_04206_b200/build.py --variants > /dev/null
python -c "import oracle; oracle.build()"
timeout 300 python tools/adv_sweep.py --sizes 20,24,27 --configs glm9b --iters 20 > gpurun_out/adv_sweep10.jsonl 2>&1; cut -c1-300 gpurun_out/adv_sweep10.jsonl
timeout 1500 python -m pytest tests/test_gpu_adv_layouts.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_variants.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/adv_large_pytest.log
timeout 600 ncu --set full --clock-control none -k regex:k_adv_large -c 3 -o gpurun_out/adv_large_2e27 -f python tools/adv_sweep.py --sizes 27 --configs "" --iters 1 > gpurun_out/ncu_adv_large.log 2>&1
ncu -i gpurun_out/adv_large_2e27.ncu-rep --page raw --csv > gpurun_out/adv_large_2e27.raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_adv_large.log
