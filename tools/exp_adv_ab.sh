# A/B of two adv_coop.cu versions on the same box: gpurun_in/adv_coop_old.cu vs the tree's
B='import importlib.util; sp = importlib.util.spec_from_file_location("b", "paper_2510_04206_b200/build.py"); m = importlib.util.module_from_spec(sp); sp.loader.exec_module(m); m.build(force=True)'
run() { timeout 300 python tools/adv_sweep.py --sizes 24,27 --configs glm9b --iters 10 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l)
    print(' ', d['case'], 'graph' if d['graph'] else 'plain', round(d['latency_us'], 1), 'us', round(d['GBps']), 'GB/s', d.get('phase_us'))"; }
cp paper_2510_04206_b200/csrc/adv_coop.cu /tmp/adv_new.cu
cp gpurun_in/adv_coop_old.cu paper_2510_04206_b200/csrc/adv_coop.cu; python -c "$B"; echo OLD; run
cp /tmp/adv_new.cu paper_2510_04206_b200/csrc/adv_coop.cu; python -c "$B"; echo NEW; run
