#!/bin/bash
# L2 policy experiment: DRAM bytes (ncu, first step's GEMMs) and live step time per setting.
for pol in ${POLS:-211010 210000 210202 212020 211212 210101}; do
  AGENTRL_L2POL=$pol timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:gemm --launch-skip ${SKIP:-0} -c 3 --csv \
     --log-file gpurun_out/l2_$pol.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  AGENTRL_L2POL=$pol timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/l2b_$pol.json 2>/dev/null
  python - "$pol" <<'PY'
import csv, json, sys
pol = sys.argv[1]
rows = [r for r in csv.DictReader([l for l in open(f"gpurun_out/l2_{pol}.csv") if l.startswith('"')])]
out = {}
for r in rows:
    k = r["Kernel Name"].split("<")[1].split(",")[0]
    out.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
d = json.load(open(f"gpurun_out/l2b_{pol}.json"))
print(pol, {k: (round(float(v["dram__bytes_read.sum"]) / 1e9, 1)) for k, v in out.items()},
      round(d["ms_per_step"], 1), d["clocks"]["sm_mhz"], {k: round(v[0], 1) for k, v in d["kernel_ms"].items() if "gemm" in k})
PY
done
