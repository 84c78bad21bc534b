"""Helpers for the GPU tests: move synth batches to the device, call the C ABI, and
compare with the oracle.  (Argument plumbing only.)"""
import numpy as np
import torch

import synth

DEV = "cuda"


def t(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV, dt)


def bf16_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(DEV).view(torch.bfloat16)


def batch_dev(b):
    return dict(T=int(b["T"]), n_groups=int(b["n_groups"]), n_tasks=int(b["n_tasks"]),
                traj_offsets=t(b["traj_offsets"], torch.int64),
                task_id=t(b["task_id"], torch.int32), group_id=t(b["group_id"], torch.int32),
                rewards=t(b["rewards"], torch.float32), loss_mask=t(b["loss_mask"], torch.uint8))


def f64(bits):
    return synth.bf16_bits_to_f32(bits).astype(np.float64)


def adv_close(got, want):
    """north_star: <= 1e-5 relative on advantages (absolute floor 1e-6)."""
    return np.all(np.abs(got - want) <= 1e-5 * np.abs(want) + 1e-6)


def max_abs_rel(got, want):
    """north_star gradient metric: max|got - want| / max|want| per tensor."""
    den = np.abs(want).max()
    return float(np.abs(got - want).max() / den) if den > 0 else float(np.abs(got).max())


def loss_tol(ref_loss, terms_scale):
    """<= 1e-3 relative on the loss, relative to max(|L|, (1/N) sum |term|)."""
    return 1e-3 * max(abs(ref_loss), terms_scale)
