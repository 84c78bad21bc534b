"""Subprocess body for tests/test_gpu_variants.py::test_schedule_variants_bitwise: one fused
step on `ragged`, `parity7b` and `longk` with the library AGENTRL_LIB names (a build variant,
or the default build); the outputs and the throttle's wait counts are saved to the .npz named by
argv[1] for a bitwise comparison against the default build.  (Argument plumbing only.)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2510_04206_b200 as ag  # noqa: E402
from gpu_util import batch_dev, bf16_dev, t  # noqa: E402


def main(path):
    out = {}
    w0 = ag.debug_throttle_waits()
    for name in ("ragged", "parity7b", "longk"):
        cfg = synth.CONFIGS[name]
        b = synth.make_structure(cfg)
        hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
        old = synth.make_old_logp_free(cfg.T, 29)
        step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)
        step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
        torch.cuda.synchronize()
        assert int(step.status.item()) & ~ag.ST_GROUP_TOO_SMALL == 0
        out[name + "_loss"] = step.loss.cpu().numpy()
        out[name + "_adv"] = step.adv_tok.cpu().numpy()
        out[name + "_gh"] = step.grad_hidden.view(torch.int16).cpu().numpy()
        out[name + "_gw"] = step.grad_W.cpu().numpy()
    out["throttle_waits"] = np.asarray(ag.debug_throttle_waits()) - np.asarray(w0)
    np.savez(path, **out)


if __name__ == "__main__":
    main(sys.argv[1])
