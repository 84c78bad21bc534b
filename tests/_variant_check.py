"""Subprocess body for tests/test_gpu_variants.py: one fused step on `ragged` and `tiny` with
the library AGENTRL_LIB names (a build variant), checked against the oracle.
Exit code 0 = parity holds.  (Argument plumbing + comparison only.)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2510_04206_b200 as ag  # noqa: E402
from gpu_util import adv_close, batch_dev, bf16_dev, f64, max_abs_rel, t  # noqa: E402


def main():
    for name in ("tiny", "ragged"):
        cfg = synth.CONFIGS[name]
        b = synth.make_structure(cfg)
        hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
        h, W = f64(hb), f64(Wb)
        lp = oracle.logprob(h, W, y, b["loss_mask"])
        old = (lp + synth.make_deltas(cfg.T, 17)).astype(np.float32)
        ref = oracle.grpo_step(b, h, W, y, old.astype(np.float64))
        step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)
        step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
        torch.cuda.synchronize()
        assert adv_close(step.adv_tok.cpu().numpy(), ref["adv_tok"]), name
        N = int((b["loss_mask"] != 0).sum())
        assert abs(step.loss.item() - ref["loss"]) <= 1e-3 * max(abs(ref["loss"]), 1.0 / N) + 1e-9
        e1 = max_abs_rel(step.grad_hidden.float().cpu().numpy(), ref["grad_hidden"])
        e2 = max_abs_rel(step.grad_W.cpu().numpy(), ref["grad_W"])
        assert e1 <= 2e-2 and e2 <= 2e-2, (name, e1, e2)
    print("variant ok", ag.LIB_PATH)


if __name__ == "__main__":
    main()
