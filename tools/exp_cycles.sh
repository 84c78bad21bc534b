#!/bin/bash
# Clock-independent comparison of GEMM variants: cycles, tensor-active %, DRAM bytes (ncu,
# first step's three GEMMs at glm9b).  Usage: bash tools/exp_cycles.sh "tag ENV=.. ENV=.." ...
for spec in "$@"; do
  set -- $spec; tag=$1; shift
  env "$@" timeout 900 ncu --metrics gpc__cycles_elapsed.max,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
     -k regex:gemm -c 3 --csv --log-file gpurun_out/c_$tag.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  python - "$tag" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = [r for r in csv.DictReader([l for l in open(f"gpurun_out/c_{tag}.csv") if l.startswith('"')])]
out = {}
for r in rows:
    k = {"0": "fwd", "2": "gW", "1": "gH"}[r["Kernel Name"].split("<")[1].split(",")[0]]
    out.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"])
tot = sum(v["gpc__cycles_elapsed.max"] for v in out.values())
print(tag, "Mcyc total %.1f |" % (tot / 1e6), " ".join(
    "%s: %.1fMcyc tc%.0f%% dram%.0fGB hit%.0f%%" % (k, v["gpc__cycles_elapsed.max"] / 1e6,
    v["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"],
    v["dram__bytes_read.sum"] / 1e9, v["lts__t_sector_hit_rate.pct"]) for k, v in out.items()), flush=True)
PY
done
