"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel
(short name) launches, total/avg device time and share of the library's kernels.
Usage: python tools/summarize_ncu_launches.py launches.csv [--last-steps N]"""
import csv
import re
import sys
from collections import OrderedDict


# kernels that start a fused step (the advantage normalisation; bench.py's adv-norm latency
# probes launch them too, without GEMMs after them)
STEP_START = ("k_adv_coop_all", "k_adv_small_all", "k_adv_large_all", "k_adv_small_stats",
              "k_adv_large_stats", "k_count")


def short(name):
    m = re.search(r"agentrl::(\w+)", name)
    if m:
        base = m.group(1)
        t = re.search(r"gemm_sm100_(?:pair_)?kernel<(\d)", name)
        if t:
            base += {"0": "<FWD>", "1": "<GRADH>", "2": "<GRADW>", "3": "<LOGP>"}[t.group(1)]
        return base
    return "other:" + name.split("(")[0][-60:]


def main(path, last_steps=None):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        rows.append((short(r["Kernel Name"]), float(r["Metric Value"]), r["Metric Unit"]))
    ours = [r for r in rows if not r[0].startswith("other:")]
    if last_steps:
        # the advantage normalisation (k_adv_coop_all, or k_count on the 3-kernel path)
        # starts each step
        starts = [i for i, r in enumerate(ours) if r[0] in STEP_START]
        segs = [ours[a:b] for a, b in zip(starts, starts[1:] + [len(ours)])]
        segs = [sg for sg in segs if any("gemm" in r[0] for r in sg)]  # fused steps only
        if len(segs) >= last_steps:
            ours = [r for sg in segs[-last_steps:] for r in sg]
    agg = OrderedDict()
    for n, v, u in ours:
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1e-6)
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'avg ms':>10s} {'share':>7s}")
    for n, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:28s} {c:8d} {ms:10.3f} {ms / c:10.3f} {100 * ms / tot:6.1f}%")
    print(f"{'TOTAL':28s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")


if __name__ == "__main__":
    ls = None
    if "--last-steps" in sys.argv:
        ls = int(sys.argv[sys.argv.index("--last-steps") + 1])
    main(sys.argv[1], ls)
