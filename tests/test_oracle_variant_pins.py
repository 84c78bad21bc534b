"""Pins for the loss-variant oracle (oracle/oracle_variants.c): KL penalty (k3 estimator,
P:1103 / P:1119) and sequence-level aggregation (GRPO's 1/K).  Anchors: PyTorch CPU
fp64 autograd of the same objective, finite differences, closed forms, and reduction to the
base oracle (an independently pinned function) at beta = 0 with token-mean weights."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def _inputs(seed=0, T=300, d=24, V=96, sigma=0.2):
    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    mask = b["loss_mask"][:T].copy()
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((T, d))
    W = rng.standard_normal((V, d)) * (2.0 / math.sqrt(d))
    y = rng.integers(0, V, size=T).astype(np.int32)
    A = rng.standard_normal(T)
    lp = oracle.logprob(h, W, y, mask)
    old = lp + synth.make_deltas(T, seed + 1, sigma=sigma)
    ref = lp + rng.normal(0.0, 0.3, size=T)
    return mask, h, W, y, A, old, ref


def _torch(h, W, y, A, old, ref, mask, w, beta, eps=(0.2, 0.2)):
    ht = torch.tensor(h, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    logp = torch.log_softmax(ht @ Wt.T, -1).gather(1, torch.tensor(y).long()[:, None])[:, 0]
    rho = torch.exp(logp - torch.tensor(old))
    At = torch.tensor(A)
    term = torch.minimum(rho * At, torch.clamp(rho, 1 - eps[0], 1 + eps[1]) * At)
    r = torch.tensor(ref) - logp
    kl = torch.exp(r) - r - 1
    mk = torch.tensor(mask != 0)
    loss = (torch.tensor(w) * (-term + beta * kl) * mk).sum()
    loss.backward()
    return loss.item(), ht.grad.numpy(), Wt.grad.numpy()


def test_reduces_to_base_oracle():
    mask, h, W, y, A, old, ref = _inputs()
    N = int(mask.sum())
    a = oracle.policy_loss_ex(h, W, y, A, old, mask, N)
    b = oracle.policy_loss_fwd_bwd(h, W, y, A, old, mask, N)
    assert abs(a["loss"] - b["loss"]) < 1e-13
    np.testing.assert_allclose(a["grad_hidden"], b["grad_hidden"], atol=1e-14)
    np.testing.assert_allclose(a["grad_W"], b["grad_W"], atol=1e-14)
    np.testing.assert_array_equal(a["loss_stats"][:4], b["loss_stats"])


@pytest.mark.parametrize("beta", [0.0, 0.05, 0.5])
@pytest.mark.parametrize("agg", ["token", "seq"])
def test_matches_torch_autograd(beta, agg):
    mask, h, W, y, A, old, ref = _inputs(seed=3)
    T = len(mask)
    N = int(mask.sum())
    if agg == "token":
        w = np.where(mask != 0, 1.0 / N, 0.0)
        weights = None
    else:
        cfg = synth.CONFIGS["ragged"]
        b = synth.make_structure(cfg)
        off = b["traj_offsets"]
        keep = int(np.searchsorted(off, T, side="right")) - 1
        bb = dict(T=T, traj_offsets=np.concatenate([off[:keep + 1], [T]]) if off[keep] < T
                  else off[:keep + 1], loss_mask=mask)
        weights, _ = oracle.seq_mean_weights(bb)
        w = weights
    out = oracle.policy_loss_ex(h, W, y, A, old, mask, N, kl_beta=beta, ref_logp=ref,
                                weights=weights)
    tl, tgh, tgw = _torch(h, W, y, A, old, ref, mask, w, beta)
    assert abs(out["loss"] - tl) < 1e-12
    np.testing.assert_allclose(out["grad_hidden"], tgh, atol=1e-13)
    np.testing.assert_allclose(out["grad_W"], tgw, atol=1e-13)
    assert out["loss_stats"][4] >= 0.0  # k3 KL is non-negative


def test_kl_zero_at_reference():
    """ref = logp -> KL_t = 0 and its gradient vanishes: beta has no effect."""
    mask, h, W, y, A, old, _ = _inputs(seed=5)
    N = int(mask.sum())
    lp = oracle.logprob(h, W, y, mask)
    a = oracle.policy_loss_ex(h, W, y, A, old, mask, N, kl_beta=0.7, ref_logp=lp)
    b = oracle.policy_loss_ex(h, W, y, A, old, mask, N)
    assert abs(a["loss"] - b["loss"]) < 1e-13 and a["loss_stats"][4] < 1e-15
    np.testing.assert_allclose(a["grad_W"], b["grad_W"], atol=1e-14)


def test_seq_mean_closed_forms():
    """On-policy (rho = 1): loss = -(1/n_seq) sum_g mean_{t in g} A_t; with equal lengths
    n_g the sequence mean equals the token mean."""
    cfg = synth.CONFIGS["micro"]
    b = synth.make_structure(cfg)
    w, n_seq = oracle.seq_mean_weights(b)
    off, mask = b["traj_offsets"], b["loss_mask"]
    assert n_seq == sum(int(mask[off[g]:off[g + 1]].sum() > 0) for g in range(len(off) - 1))
    assert abs(w.sum() - 1.0) < 1e-14
    rng = np.random.default_rng(1)
    h = rng.standard_normal((cfg.T, cfg.d))
    W = rng.standard_normal((cfg.V, cfg.d))
    y = rng.integers(0, cfg.V, size=cfg.T).astype(np.int32)
    A = rng.standard_normal(cfg.T)
    lp = oracle.logprob(h, W, y, mask)
    out = oracle.policy_loss_ex(h, W, y, A, lp, mask, int(mask.sum()), weights=w)
    ref = 0.0
    for g in range(len(off) - 1):
        m = mask[off[g]:off[g + 1]] != 0
        if m.any():
            ref += A[off[g]:off[g + 1]][m].mean()
    assert abs(out["loss"] - (-ref / n_seq)) < 1e-13
    # equal lengths: tokens 4 per trajectory of 6, all masked the same way
    eq = dict(T=12, traj_offsets=np.asarray([0, 6, 12]), loss_mask=np.asarray(
        [0, 1, 1, 0, 1, 1] * 2, np.uint8))
    w2, _ = oracle.seq_mean_weights(eq)
    np.testing.assert_allclose(w2[eq["loss_mask"] != 0], 1.0 / 8.0, atol=1e-15)


def test_finite_differences_with_kl_and_seq_weights():
    cfg = synth.CONFIGS["micro"]
    b = synth.make_structure(cfg)
    rng = np.random.default_rng(9)
    h = rng.standard_normal((cfg.T, cfg.d))
    W = rng.standard_normal((cfg.V, cfg.d))
    y = rng.integers(0, cfg.V, size=cfg.T).astype(np.int32)
    mask = b["loss_mask"]
    A = rng.standard_normal(cfg.T)
    lp = oracle.logprob(h, W, y, mask)
    old = lp + synth.make_deltas(cfg.T, 6, sigma=0.15, margin=0.05)
    ref = lp + rng.normal(0, 0.2, size=cfg.T)
    w, _ = oracle.seq_mean_weights(b)
    N = int(mask.sum())

    def L(hh, WW):
        return oracle.policy_loss_ex(hh, WW, y, A, old, mask, N, kl_beta=0.3, ref_logp=ref,
                                     weights=w, grads=False)["loss"]

    out = oracle.policy_loss_ex(h, W, y, A, old, mask, N, kl_beta=0.3, ref_logp=ref, weights=w)
    e = 1e-5
    worst = 0.0
    for arr, g in ((h, out["grad_hidden"]), (W, out["grad_W"])):
        for ij in np.ndindex(arr.shape):
            a1, a2 = arr.copy(), arr.copy()
            a1[ij] += e
            a2[ij] -= e
            fd = ((L(a1, W) - L(a2, W)) if arr is h else (L(h, a1) - L(h, a2))) / (2 * e)
            sc = max(abs(fd), abs(g[ij]), 1e-8)
            worst = max(worst, abs(fd - g[ij]) / sc if sc > 1e-6 else abs(fd - g[ij]))
    assert worst <= 1e-4, worst
