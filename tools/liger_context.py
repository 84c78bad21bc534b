"""Context line (not a dependency, not the target): Liger-Kernel 0.8.0's
LigerFusedLinearGRPOLoss (chunked torch/Triton fused-linear GRPO loss, installed in the image)
against agentrl_policy_loss_fwd_bwd on the same shapes and the same values.

Work: R = B*L loss rows (every row an assistant token), head d x V, bf16 inputs, token-level
("dapo") mean, clip 0.2/0.2, no KL term.  Default R = 64 x 829 = 53,056 rows, d = 4096,
V = 151,552: the masked rows of one glm9b step (T_eff = 53,039).  Liger takes one advantage per
sequence; the same value is broadcast to that sequence's tokens for our call.  Prints one JSON
line: both times (CUDA events, median) and the agreement of loss / grad_hidden / grad_W.

    python tools/liger_context.py [--B 64 --L 829 --d 4096 --V 151552] [--compiled]
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_04206_b200 as ag  # noqa: E402


def timed(fn, iters):
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=64)
    ap.add_argument("--L", type=int, default=829)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--V", type=int, default=151552)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--compiled", action="store_true")
    a = ap.parse_args()
    from liger_kernel.chunked_loss import LigerFusedLinearGRPOLoss

    dev = "cuda"
    B, L, d, V = a.B, a.L, a.d, a.V
    R = B * L
    g = torch.Generator(device=dev)
    g.manual_seed(2510_04206 + 31)
    W = (torch.randn(V, d, generator=g, device=dev) * (3.0 / math.sqrt(d))).to(torch.bfloat16)
    h = torch.randn(B, L, d, generator=g, device=dev).to(torch.bfloat16)
    y = torch.randint(0, V, (B, L), generator=g, device=dev)
    adv_seq = torch.randn(B, generator=g, device=dev)
    mask = torch.ones(B, L, device=dev, dtype=torch.int64)
    # behaviour log-probs: exact log-softmax of the same logits + small noise (rho near 1)
    with torch.no_grad():
        lp = torch.empty(B, L, device=dev)
        for b in range(B):
            z = (h[b].float() @ W.float().t())
            lp[b] = torch.log_softmax(z, -1).gather(1, y[b:b + 1].t()).squeeze(1)
        old = lp + 0.08 * torch.randn(B, L, generator=g, device=dev)

    # ---- Liger
    loss_mod = LigerFusedLinearGRPOLoss(beta=0.0, compiled=a.compiled, use_ref_model=False,
                                        epsilon_low=0.2, epsilon_high=0.2, loss_type="dapo")
    hl = h.clone().requires_grad_(True)
    Wl = W.clone().requires_grad_(True)

    def liger():
        hl.grad = None
        Wl.grad = None
        out = loss_mod(hl, Wl, y, mask, adv_seq, old_per_token_logps=old)
        loss = out[0] if isinstance(out, tuple) else out
        loss.backward()
        return loss

    lg_loss = liger()
    torch.cuda.synchronize()
    t_liger = timed(liger, a.iters)
    lg_loss = float(lg_loss.item())
    lg_gh = hl.grad.float().reshape(R, d)
    lg_gw = Wl.grad.float()

    # ---- ours: agentrl_policy_loss_fwd_bwd over the same R rows
    hid = h.reshape(R, d).contiguous()
    tgt = y.reshape(R).to(torch.int32).contiguous()
    advt = adv_seq.repeat_interleave(L).contiguous()
    oldt = old.reshape(R).contiguous()
    lm = torch.ones(R, dtype=torch.uint8, device=dev)
    nglob = torch.tensor([R], dtype=torch.int64, device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    gh = torch.empty(R, d, dtype=torch.bfloat16, device=dev)
    gw = torch.empty(V, d, dtype=torch.float32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = ag.alloc_workspace(ag.agentrl_policy_loss_workspace_size(R, d, V), dev)
    args = ag.make_loss_args(R, hid, W, tgt, oldt, lm, adv_tok=advt, n_mask_global=nglob)
    out = ag.make_loss_out(loss, gh, gw)

    def ours():
        rc = ag.agentrl_policy_loss_fwd_bwd(args, out, ws, None, st)
        assert rc == 0, ag.status_string(rc)

    ours()
    torch.cuda.synchronize()
    t_ours = timed(ours, a.iters)

    def rel(x, ref):
        return float((x - ref).abs().max() / ref.abs().max())

    # plain fp32 PyTorch autograd of the same objective (small cases only): arbitrates
    ref = None
    if R * V <= 2 ** 27:
        hr = h.reshape(R, d).float().requires_grad_(True)
        Wr = W.float().requires_grad_(True)
        logp = torch.log_softmax(hr @ Wr.t(), -1).gather(1, y.reshape(R, 1)).squeeze(1)
        rho = torch.exp(logp - old.reshape(R))
        A = adv_seq.repeat_interleave(L)
        lref = -torch.minimum(rho * A, torch.clamp(rho, 0.8, 1.2) * A).mean()
        lref.backward()
        ref = {"loss": float(lref.item()),
               "ours_vs_torch": {"loss": abs(float(loss.item()) - float(lref.item())) / abs(float(lref.item())),
                                 "grad_hidden": rel(gh.float(), hr.grad), "grad_W": rel(gw, Wr.grad)},
               "liger_vs_torch": {"loss": abs(lg_loss - float(lref.item())) / abs(float(lref.item())),
                                  "grad_hidden": rel(lg_gh, hr.grad), "grad_W": rel(lg_gw, Wr.grad)}}

    res = {"case": f"R={R} (B={B} x L={L}), d={d}, V={V}, bf16, dapo token mean, clip 0.2/0.2",
           "liger_ms": t_liger, "ours_ms": t_ours, "speedup": t_liger / t_ours,
           "liger_compiled": a.compiled,
           "liger_TFLOPs_alg": 6.0 * R * V * d / (t_liger / 1e3) / 1e12,
           "ours_TFLOPs_alg": 6.0 * R * V * d / (t_ours / 1e3) / 1e12,
           "loss": {"liger": lg_loss, "ours": float(loss.item())},
           "loss_rel_diff": abs(lg_loss - float(loss.item())) / max(abs(lg_loss), 1e-12),
           "grad_hidden_maxrel": rel(gh.float(), lg_gh), "grad_W_maxrel": rel(gw, lg_gw),
           "status": int(st.item()), "fp32_torch_reference": ref}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
