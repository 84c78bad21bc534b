"""Context numbers only: cuBLAS (torch.matmul, bf16 -> fp32 accumulate) on the three LM-head
GEMM shapes of a config, back to back like one step, with CUDA events and nvidia-smi clocks.

    python tools/gemm_compare.py --config glm9b --iters 5
"""
import argparse
import json
import os
import subprocess
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="glm9b")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--teff", type=int, default=0)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    b = synth.make_structure(cfg)
    M = a.teff or int(b["loss_mask"].astype(bool).sum())
    d, V = cfg.d, cfg.V
    dev = "cuda"
    H = torch.randn(M, d, device=dev).to(torch.bfloat16)
    W = torch.randn(V, d, device=dev).to(torch.bfloat16)
    G = torch.randn(M, V, device=dev).to(torch.bfloat16)
    shapes = {
        "fwd  z=H W^T": lambda: torch.matmul(H, W.t()),
        "gradW G^T H": lambda: torch.matmul(G.t(), H),
        "gradH G W": lambda: torch.matmul(G, W),
    }
    flop = 2.0 * M * V * d
    rows = []
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                             "-lms", "100"], stdout=subprocess.PIPE, text=True)
    clk = []
    t = threading.Thread(target=lambda: [clk.append(float(x)) for x in proc.stdout if x.strip()],
                         daemon=True)
    t.start()
    for _ in range(2):
        for f in shapes.values():
            f()
    torch.cuda.synchronize()
    res = {k: 0.0 for k in shapes}
    for _ in range(a.iters):
        for k, f in shapes.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = f()
            e1.record()
            torch.cuda.synchronize()
            res[k] += e0.elapsed_time(e1) / a.iters
            del out
    proc.terminate()
    for k, ms in res.items():
        rows.append({"gemm": k, "ms": ms, "tflops": flop / ms / 1e9})
    clk.sort()
    print(json.dumps({"config": a.config, "M": M, "d": d, "V": V, "cublas": rows,
                      "sm_mhz_median": clk[len(clk) // 2] if clk else None}))


if __name__ == "__main__":
    main()
