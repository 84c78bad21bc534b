# adv-norm build variants on one box (A/B through AGENTRL_LIB; in-tree builds under exp/):
#   VARIANTS="name:-DFLAGS ..." e.g. "r4:-DADV_RING=4 m3:-DADV_LARGE_MINB=3 bulk:-DADV_LDGSTS=0"
# Run from the repo root; every library is built here before the gpurun call.
for v in ${VARIANTS:-base}; do
  n=${v%%:*}; f=${v#*:}
  if [ "$n" = base ]; then L=""; else L=$PWD/paper_2510_04206_b200/exp/lib_$n.so; fi
  echo "== $n"
  AGENTRL_LIB=$L timeout 300 python tools/adv_sweep.py --sizes ${SIZES:-24,27} --configs ${CONFIGS:-glm9b} --iters 10 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l)
    if not d['graph']:
        print(' ', d['case'], round(d['latency_us'], 1), 'us', round(d['GBps']), 'GB/s', d.get('phase_us'))"
done
