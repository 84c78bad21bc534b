# forward-GEMM progress throttle study: DRAM bytes of the 4 forward chunks (ncu) + live step time
for L in ${SETS:-0 16 32 64 128}; do
  AGENTRL_THROTTLE_LEAD_FWD=$L timeout 600 ncu --metrics dram__bytes_read.sum,sm__cycles_elapsed.max \
     -k regex:gemm -c 4 --csv --log-file gpurun_out/thf_$L.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
  AGENTRL_THROTTLE_LEAD_FWD=$L timeout 600 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu > gpurun_out/thfb_$L.json 2>/dev/null
  python - "$L" <<'PY'
import csv, json, sys
L = sys.argv[1]
rows = [r for r in csv.DictReader([l for l in open(f"gpurun_out/thf_{L}.csv") if l.startswith('"')])]
rd = sum(float(r["Metric Value"].replace(",", "")) for r in rows if r["Metric Name"] == "dram__bytes_read.sum")
cy = sum(float(r["Metric Value"].replace(",", "")) for r in rows if r["Metric Name"] == "sm__cycles_elapsed.max")
d = json.load(open(f"gpurun_out/thfb_{L}.json"))
print("lead_fwd", L, "fwd DRAM read GB", round(rd / 1e9, 1), "Mcyc", round(cy / 1e6, 2), "| live", round(d["ms_per_step"], 1), "ms", d["clocks"]["sm_mhz"], "MHz", {k: round(v[0] * v[1] / 8, 1) for k, v in d["kernel_ms"].items() if "gemm" in k})
PY
done
