"""compute-sanitizer cases: one agentrl_grpo_step and one agentrl_logprob_fwd on
`tiny` and `ragged` (ragged tiles in every dimension), then the large adv-norm driver on two
adversarial layouts (standalone and in the fused step); a device sync after each; exits 0 when
every call returned OK.  Run under  compute-sanitizer --tool {memcheck,racecheck,synccheck}.
(Input generation and plumbing only.)"""
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


def main():
    for name in ("tiny", "ragged"):
        cfg = synth.CONFIGS[name]
        b = synth.make_structure(cfg)
        hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
        old = synth.make_old_logp_free(cfg.T, 3)
        T_eff = int(b["loss_mask"].astype(bool).sum())
        step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V,
                       max_rows=T_eff)
        step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
        torch.cuda.synchronize()
        st = int(step.status.item())
        ws = ag.alloc_workspace(ag.agentrl_logprob_workspace_size(cfg.T, cfg.d, cfg.V))
        lp = torch.empty(cfg.T, device="cuda")
        ent = torch.empty(cfg.T, device="cuda")
        s2 = torch.zeros(1, dtype=torch.int32, device="cuda")
        rc = ag.agentrl_logprob_fwd(cfg.T, bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32),
                                    t(b["loss_mask"], torch.uint8), lp, ent, ws, s2)
        torch.cuda.synchronize()
        assert rc == 0, ag.status_string(rc)
        print(name, "grpo_step status", st, "loss", float(step.loss.item()),
              "logprob status", int(s2.item()), "launches", ag.last_launch_count(), flush=True)
    # the large adv-norm driver (> 2,048 trajectories): popcount, cooperative statistics and
    # the programmatic dependent apply, on a contiguous-group layout (no member lists) and a
    # shuffled one (member lists), standalone and inside the fused step (compaction)
    import _adv_layout_check as lay
    for kind in ("contig", "bigtraj"):
        b = lay.layout(kind, 2510_04206 + 900)
        T, n_traj = b["T"], len(b["task_id"])
        ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                        b["n_tasks"]))
        adv = torch.empty(T, dtype=torch.float32, device="cuda")
        ts = torch.empty(b["n_tasks"], 3, dtype=torch.float64, device="cuda")
        nm = torch.empty(1, dtype=torch.int64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        rc = ag.agentrl_task_adv_norm(ag.make_batch(batch_dev(b)), 1e-6, adv, ts, nm, ws, None, st)
        torch.cuda.synchronize()
        assert rc == 0, ag.status_string(rc)
        d, V = 64, 512
        rng = np.random.default_rng(3)
        hb = synth.to_bf16_bits(rng.standard_normal((T, d)).astype(np.float32))
        Wb = synth.to_bf16_bits((rng.standard_normal((V, d)) * 3 / np.sqrt(d)).astype(np.float32))
        y = rng.integers(0, V, T).astype(np.int32)
        old = synth.make_old_logp_free(T, 5)
        step = ag.Step(T, n_traj, b["n_groups"], b["n_tasks"], d, V)
        step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
        torch.cuda.synchronize()
        print(kind, "adv_norm n_mask", int(nm.item()), "status", int(st.item()),
              "fused status", int(step.status.item()), flush=True)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
