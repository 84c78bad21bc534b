#!/bin/bash
# raster experiment: DRAM read bytes of the first step's GEMMs + live step time
run() {
  tag=$1; shift
  env "$@" timeout 600 ncu --metrics dram__bytes_read.sum -k regex:gemm -c 3 --csv \
     --log-file gpurun_out/r_$tag.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu > gpurun_out/rb_$tag.json 2>/dev/null
  python - "$tag" <<'PY'
import csv, json, sys
tag = sys.argv[1]
rows = [r for r in csv.DictReader([l for l in open(f"gpurun_out/r_{tag}.csv") if l.startswith('"')])]
dr = [round(float(r["Metric Value"]) / 1e9, 1) for r in rows]
d = json.load(open(f"gpurun_out/rb_{tag}.json"))
print(tag, "dramGB(fwd,gW,gH)=", dr, "ms", round(d["ms_per_step"], 1), "mhz", d["clocks"]["sm_mhz"],
      {k[5:]: round(v[0], 1) for k, v in d["kernel_ms"].items() if "gemm" in k})
PY
}
run dyn X=1
run dyn_g8 AGENTRL_GROUP_M=8 AGENTRL_GROUP_M_BWD=2
run dyn_g32 AGENTRL_GROUP_M=32 AGENTRL_GROUP_M_BWD=4
run static AGENTRL_GEMM_SCHED=static
