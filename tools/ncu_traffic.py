"""Per-kernel DRAM traffic of one fused step from an ncu capture
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X.csv \\
      python bench.py --config C --steps 1 --warmup 0 --no-e2e --no-cpu
and merge it into profiles/ncu_traffic.json as {config: {bench kernel name: {bytes_per_step,
launches_per_step}}} (bench.py's roofline "traffic" = bytes_per_step / launches_per_step).
Usage: python tools/ncu_traffic.py X.csv CONFIG"""
import csv
import json
import os
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(__file__))
from summarize_ncu_launches import STEP_START, short  # noqa: E402

BENCH_NAME = {"gemm_sm100_pair_kernel<FWD>": "gemm_fwd", "gemm_sm100_kernel<FWD>": "gemm_fwd",
              "gemm_sm100_pair_kernel<GRADW>": "gemm_grad_W",
              "gemm_sm100_kernel<GRADW>": "gemm_grad_W",
              "gemm_sm100_pair_kernel<GRADH>": "gemm_grad_hidden",
              "gemm_sm100_kernel<GRADH>": "gemm_grad_hidden", "k_adv_coop_all": "k_adv_coop",
              "k_adv_small_all": "k_adv_coop", "k_adv_large_all": "k_adv_coop"}


def main(path, config):
    launches = OrderedDict()  # (kernel, launch id) -> bytes
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        key = (r["ID"], short(r["Kernel Name"]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
        launches[key] = launches.get(key, 0.0) + float(r["Metric Value"].replace(",", "")) * scale
    seq = [(k[1], v) for k, v in launches.items() if not k[1].startswith("other:")]
    starts = [i for i, (n, _) in enumerate(seq) if n in STEP_START]
    # the first fused step: from an advantage normalisation followed by GEMMs to the next one
    # (bench.py's adv-norm latency probes launch it alone before the steps)
    segs = [seq[a:b] for a, b in zip(starts, starts[1:] + [len(seq)])]
    segs = [sg for sg in segs if any(n.startswith("gemm") for n, _ in sg)]
    if segs:
        seq = segs[0]
    out = OrderedDict()
    for n, b in seq:
        name = BENCH_NAME.get(n, n)
        e = out.setdefault(name, {"bytes_per_step": 0, "launches_per_step": 0})
        e["bytes_per_step"] += int(b)
        e["launches_per_step"] += 1
    dst = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
    j = json.load(open(dst)) if os.path.exists(dst) else {}
    j[config] = out
    j["_how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv, one step of "
                 "python bench.py --steps 1 --warmup 0 (tools/ncu_traffic.py)")
    with open(dst, "w") as f:
        json.dump(j, f, indent=1)
    for k, v in out.items():
        print(f"{k:24s} {v['launches_per_step']:3d} launches {v['bytes_per_step'] / 1e9:9.3f} GB/step")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
