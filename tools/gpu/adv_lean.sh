# large adv-norm driver A/B: adv tests under every driver, interleaved sweep against the
# round's start (ab_old/) and the previous step (ab_prev/) and one variant build, ncu --set full
# of the three large launches at 2^27 with per-line source views
set -o pipefail
python paper_2510_04206_b200/build.py > /dev/null
python -c "import oracle; oracle.build()"
timeout 1500 python -m pytest tests/test_gpu_adv_layouts.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/adv_lean_pytest.log
for r in 1 2; do
  for v in new prev; do
    case $v in
      old) export AGENTRL_LIB=$PWD/ab_old/libagentrl.so ;;
      prev) export AGENTRL_LIB=$PWD/ab_prev/libagentrl.so ;;
      *) unset AGENTRL_LIB ;;
    esac
    timeout 300 python tools/adv_sweep.py --sizes 20,24,27 --configs glm9b --iters 20 > gpurun_out/adv_lean_$v.jsonl 2>&1
    python -c "
import json
for l in open('gpurun_out/adv_lean_$v.jsonl'):
    try: d = json.loads(l)
    except Exception: continue
    print('AB', '$v', d['case'], 'graph' if d['graph'] else 'direct', round(d['latency_us'], 1), round(d['frac_hbm'], 3), d.get('phase_us'))" | tee -a gpurun_out/adv_lean_ab.txt
  done
done
unset AGENTRL_LIB
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_adv_large -c 3 -o gpurun_out/adv_lean_2e27 -f python tools/adv_sweep.py --sizes 27 --configs "" --iters 1 > gpurun_out/ncu_adv_lean.log 2>&1
ncu -i gpurun_out/adv_lean_2e27.ncu-rep --page raw --csv > gpurun_out/adv_lean_2e27.raw.csv 2>/dev/null
ncu -i gpurun_out/adv_lean_2e27.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:k_adv_large_stats > gpurun_out/adv_lean_stats_source.csv 2>/dev/null
ncu -i gpurun_out/adv_lean_2e27.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:k_adv_large_apply > gpurun_out/adv_lean_apply_source.csv 2>/dev/null
tail -2 gpurun_out/ncu_adv_lean.log
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -m gpu -k "coop0" 2>&1 | tail -2 | tee -a gpurun_out/adv_lean_pytest.log
