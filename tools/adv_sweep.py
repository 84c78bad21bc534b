"""adv-norm (part 1) latency and bandwidth, single GPU, cold L2 (a 2x-L2 buffer is
written before every timed call), optionally under a CUDA graph.

    python tools/adv_sweep.py [--sizes 17,20,24,27] [--iters 20]

Algorithmic bytes per call: mask T B + adv_tok 4T B + per trajectory
offsets/ids/reward 20 B.  Prints one JSON object per size.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2510_04206_b200 as ag  # noqa: E402


def alg_bytes(b):
    return int(b["T"]) * 5 + 20 * len(b["task_id"])


def time_adv(b, iters=20, graph=False, clean=False):
    dev = "cuda"
    bd = {k: (torch.from_numpy(np.ascontiguousarray(v)).to(dev) if isinstance(v, np.ndarray) else v)
          for k, v in b.items()}
    bd["traj_offsets"] = bd["traj_offsets"].long()
    T = int(b["T"])
    n_traj = len(b["task_id"])
    ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                    b["n_tasks"]))
    adv = torch.empty(T, dtype=torch.float32, device=dev)
    ts = torch.empty(b["n_tasks"], 3, dtype=torch.float64, device=dev)
    nm = torch.empty(1, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    batch = ag.make_batch(bd)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    # clean: after the write flush, read another 2 x L2 buffer so that L2 holds clean lines
    # (the flush's dirty lines are written back outside the timed region)
    rbuf = torch.ones(2 * l2 // 4, dtype=torch.float32, device=dev) if clean else None
    stream = torch.cuda.Stream()

    def call():
        rc = ag.agentrl_task_adv_norm(batch, 1e-6, adv, ts, nm, ws, None, st, stream=stream)
        assert rc == 0

    with torch.cuda.stream(stream):
        for _ in range(3):
            call()
        g = None
        if graph:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                call()
        times, phs = [], []
        for _ in range(iters):
            flush.fill_(1.0)
            if rbuf is not None:
                rbuf.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if g is not None:
                g.replay()
            else:
                call()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            phs.append(ag.debug_adv_phase_ns())
    times.sort()
    ms = times[len(times) // 2]
    # stamps relative to stamp 0, median over the timed calls (small driver: [1] trajectory
    # table, [2] group advantages, [3] counts, [4] partial moments, [5] after the grid barrier,
    # [6] moments, [7] apply done; large driver: one per phase)
    phases = []
    for i in range(1, 8):
        v = sorted((ph[i] - ph[0]) / 1e3 for ph in phs if 0 <= ph[i] - ph[0] < 1e9)
        phases.append(round(v[len(v) // 2], 1) if v else None)
    return ms, int(nm.item()), phases


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="17,20,24,27")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--configs", default="qwen7b,glm9b,qwen32b,skew14b")
    ap.add_argument("--clean", action="store_true",
                    help="leave L2 clean before each call (write flush, then a read flush)")
    a = ap.parse_args()
    hbm = 6551.4
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        hbm = json.load(open(pk)).get("hbm_gbs", hbm)
    cases = [(f"sweep_2^{s}", synth.make_sweep_structure(1 << int(s))) for s in a.sizes.split(",") if s]
    cases += [(c, synth.make_structure(synth.CONFIGS[c])) for c in a.configs.split(",") if c]
    for name, b in cases:
        for graph in (False, True):
            ms, nm, phases = time_adv(b, a.iters, graph, a.clean)
            by = alg_bytes(b)
            print(json.dumps({"case": name, "T": int(b["T"]), "n_traj": len(b["task_id"]),
                              "graph": graph, "latency_us": ms * 1e3, "alg_bytes": by,
                              "GBps": by / (ms / 1e3) / 1e9, "frac_hbm": by / (ms / 1e3) / 1e9 / hbm,
                              "n_mask": nm, "phase_us": phases, "clean_l2": a.clean}), flush=True)


if __name__ == "__main__":
    main()
