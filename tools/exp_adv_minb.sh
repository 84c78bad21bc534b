# adv-norm register budget A/B (ADV_MIN_BLOCKS = resident blocks per SM) on the sweep sizes
for mb in ${SETS:-2 3 4}; do
  AGENTRL_NVCC_EXTRA="-DADV_MIN_BLOCKS=$mb" python -c "
import importlib.util, sys
sp = importlib.util.spec_from_file_location('b', 'paper_2510_04206_b200/build.py'); m = importlib.util.module_from_spec(sp); sp.loader.exec_module(m); m.build(force=True)" > /dev/null
  echo "ADV_MIN_BLOCKS=$mb"
  timeout 300 python tools/adv_sweep.py --sizes 24,27 --configs glm9b --iters 10 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l)
    print(' ', d['case'], 'graph' if d['graph'] else 'plain', round(d['latency_us'], 1), 'us', round(d['GBps']), 'GB/s', d.get('phase_us'))"
done
python -m pytest tests/test_gpu_parity.py -x -q -k "adv" 2>&1 | tail -2
