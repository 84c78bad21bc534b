"""One fused step at a config (for ncu captures): python tools/one_step.py [config] [--steps n]
(input generation and plumbing only)"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "qwen7b"
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
cfg = synth.CONFIGS[name]
b = synth.make_structure(cfg)
hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
old = synth.make_old_logp_free(cfg.T, 5)
try:
    step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V,
                   max_rows=int(b["loss_mask"].astype(bool).sum()))
except TypeError:  # an older build of the binding (A/B against a previous tree)
    step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)
args = (batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
for _ in range(steps):
    step(*args)
torch.cuda.synchronize()
print(name, "status", int(step.status.item()), "loss", float(step.loss.item()))
