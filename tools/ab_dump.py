"""A/B bitwise check between two builds of the library: run the fused step on a few configs with
the package found under ROOT (argv[1]) and save the outputs to argv[2] (.npz).  Run once per
tree, then compare the two files with --compare A.npz B.npz.  Input generation and plumbing
only."""
import os
import sys

import numpy as np


def dump(root, out, cfgs):
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    import torch
    import synth
    import paper_2510_04206_b200 as ag
    print("library", ag.LIB_PATH)
    res = {}
    for name in cfgs:
        cfg = synth.CONFIGS[name]
        b = synth.make_structure(cfg)
        hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
        dev = "cuda"
        t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)
        bf = lambda bits: torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(dev).view(torch.bfloat16)
        bd = dict(T=cfg.T, n_groups=b["n_groups"], n_tasks=b["n_tasks"],
                  traj_offsets=t(b["traj_offsets"], torch.int64), task_id=t(b["task_id"], torch.int32),
                  group_id=t(b["group_id"], torch.int32), rewards=t(b["rewards"], torch.float32),
                  loss_mask=t(b["loss_mask"], torch.uint8))
        old = t(synth.make_old_logp_free(cfg.T, 5), torch.float32)
        step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)
        step(bd, bf(hb), bf(Wb), t(y, torch.int32), old)
        torch.cuda.synchronize()
        res[name + "/loss"] = step.loss.cpu().numpy()
        res[name + "/logp"] = step.logp.cpu().numpy()
        res[name + "/gh"] = step.grad_hidden.view(torch.int16).cpu().numpy()
        res[name + "/gw"] = step.grad_W.cpu().numpy()
        res[name + "/status"] = step.status.cpu().numpy()
        del step
        torch.cuda.empty_cache()
    np.savez(out, **res)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in A.files:
        same = np.array_equal(A[k], B[k])
        if not same:
            bad += 1
            x, y = A[k].astype(np.float64), B[k].astype(np.float64)
            print("DIFF", k, "max abs", np.abs(x - y).max(), "n", int((A[k] != B[k]).sum()))
        else:
            print("same", k)
    print("bitwise identical" if bad == 0 else f"{bad} arrays differ")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        sys.exit(1 if compare(sys.argv[2], sys.argv[3]) else 0)
    dump(sys.argv[1], sys.argv[2], sys.argv[3].split(",") if len(sys.argv) > 3 else
         ["tiny", "ragged", "parity7b", "longk", "qwen7b"])
