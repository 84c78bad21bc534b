"""Pins for the loss-variant oracle (oracle/oracle_variants.c): KL penalty (k3 estimator,
P:1103 / P:1119) and the GRPO group-level aggregation (E_{i,j} 1/K_{i,j} sum_g).  Anchors: PyTorch CPU
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
        cut = off[keep] < T
        bb = dict(T=T, traj_offsets=np.concatenate([off[:keep + 1], [T]]) if cut
                  else off[:keep + 1], loss_mask=mask, n_groups=b["n_groups"],
                  group_id=b["group_id"][:keep + 1] if cut else b["group_id"][:keep])
        weights, _ = oracle.grpo_group_weights(bb)
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


def test_grpo_group_weights_hand_example(golden_dir):
    """Hand-worked case with unequal K_{i,j}, an empty member and an empty group id
    (tests/golden/grpo_group_weights.json): weights and the on-policy loss."""
    import json
    import os
    g = json.load(open(os.path.join(golden_dir, "grpo_group_weights.json")))
    b = dict(T=g["T"], traj_offsets=np.asarray(g["traj_offsets"], np.int64),
             group_id=np.asarray(g["group_id"], np.int32), n_groups=g["n_groups"],
             loss_mask=np.asarray(g["loss_mask"], np.uint8))
    w, G = oracle.grpo_group_weights(b)
    assert G == g["G"]
    np.testing.assert_allclose(w, g["weights"], rtol=1e-15, atol=0)
    T, d, V = g["T"], 3, 5
    rng = np.random.default_rng(3)
    h = rng.standard_normal((T, d))
    W = rng.standard_normal((V, d))
    y = rng.integers(0, V, size=T).astype(np.int32)
    lp = oracle.logprob(h, W, y, b["loss_mask"])  # old = logp: rho = 1
    out = oracle.policy_loss_ex(h, W, y, np.asarray(g["adv_tok"]), lp, b["loss_mask"],
                                int(b["loss_mask"].sum()), weights=w)
    assert abs(out["loss"] - g["on_policy_loss"]) < 1e-15


def _variable_k_batch(seed):
    """Groups of 1..6 members, some members without masked tokens, one declared-empty id."""
    rng = np.random.default_rng(seed)
    sizes = [int(k) for k in rng.integers(1, 7, size=7)]
    gid, off, mask = [], [0], []
    for j, k in enumerate(sizes):
        for _ in range(k):
            L = int(rng.integers(1, 9))
            m = (rng.uniform(size=L) < 0.5).astype(np.uint8)
            if rng.uniform() < 0.25:
                m[:] = 0
            gid.append(j + (j >= 3))  # id 3 is declared but never used
            mask += m.tolist()
            off.append(off[-1] + L)
    return dict(T=off[-1], traj_offsets=np.asarray(off, np.int64),
                group_id=np.asarray(gid, np.int32), n_groups=len(sizes) + 1,
                loss_mask=np.asarray(mask, np.uint8))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_grpo_group_mean_closed_form(seed):
    """On policy, the weighted loss equals the paper's group-level form evaluated directly
    from the batch structure: -(1/G) sum_j (1/K_j) sum_{g in j} mean_{t in g} A_t
    (P:1247-1256), with empty members contributing 0 but counting in K_j."""
    b = _variable_k_batch(seed)
    w, G = oracle.grpo_group_weights(b)
    off, mask, gid = b["traj_offsets"], b["loss_mask"], b["group_id"]
    T = b["T"]
    rng = np.random.default_rng(seed + 10)
    h = rng.standard_normal((T, 4))
    W = rng.standard_normal((6, 4))
    y = rng.integers(0, 6, size=T).astype(np.int32)
    A = rng.standard_normal(T)
    lp = oracle.logprob(h, W, y, mask)
    out = oracle.policy_loss_ex(h, W, y, A, lp, mask, max(int(mask.sum()), 1), weights=w)
    groups = sorted(set(gid.tolist()))
    assert G == len(groups)
    obj = 0.0
    for j in groups:
        members = [g for g in range(len(gid)) if gid[g] == j]
        s = 0.0
        for g in members:
            m = mask[off[g]:off[g + 1]] != 0
            if m.any():
                s += A[off[g]:off[g + 1]][m].mean()
        obj += s / len(members)
    assert abs(out["loss"] - (-obj / len(groups))) < 1e-13
    # equal K and every member masked: the group mean is the mean over trajectories
    eq = dict(T=12, traj_offsets=np.asarray([0, 3, 6, 9, 12]), group_id=np.asarray([0, 0, 1, 1]),
              n_groups=2, loss_mask=np.asarray([1, 1, 0, 1, 0, 0, 1, 1, 1, 0, 1, 1], np.uint8))
    w2, _ = oracle.grpo_group_weights(eq)
    np.testing.assert_allclose(w2[[0, 1, 3, 6, 7, 8, 10, 11]],
                               [1 / 8, 1 / 8, 1 / 4, 1 / 12, 1 / 12, 1 / 12, 1 / 8, 1 / 8],
                               rtol=1e-15)


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
    w, _ = oracle.grpo_group_weights(b)
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
