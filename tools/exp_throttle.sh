# Backward-GEMM progress throttle study (AGENTRL_THROTTLE_LEAD / _EVERY): DRAM bytes and cycles
# of the first step's grad GEMMs under ncu, then live step time.  usage: bash tools/exp_throttle.sh
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "loss or fused" 2>&1 | tail -1
for v in ${SETS:-0:8 16:8 32:8 64:8 128:16}; do set -- ${v/:/ }
  AGENTRL_THROTTLE_LEAD=$1 AGENTRL_THROTTLE_EVERY=$2 timeout 600 ncu --metrics dram__bytes_read.sum,sm__cycles_elapsed.max,gpu__time_duration.sum \
     -k regex:gemm --launch-skip 4 -c 2 --csv --log-file gpurun_out/thr_$1_$2.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  AGENTRL_THROTTLE_LEAD=$1 AGENTRL_THROTTLE_EVERY=$2 timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu > gpurun_out/thrb_$1_$2.json 2>/dev/null
  python - "$1_$2" <<'PY'
import csv, json, sys
tag = sys.argv[1]
rows = [r for r in csv.DictReader([l for l in open(f"gpurun_out/thr_{tag}.csv") if l.startswith('"')])]
out = {}
for r in rows:
    k = "gW" if "<2," in r["Kernel Name"] else "gH"
    out.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
d = json.load(open(f"gpurun_out/thrb_{tag}.json"))
print(tag, {k: (round(v["dram__bytes_read.sum"] / 1e9, 1), round(v["sm__cycles_elapsed.max"] / 1e6, 2)) for k, v in out.items()},
      round(d["ms_per_step"], 1), d["clocks"]["sm_mhz"], {k: round(v[0], 1) for k, v in d["kernel_ms"].items() if "grad" in k})
PY
done
