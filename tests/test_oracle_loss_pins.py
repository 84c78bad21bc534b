"""Pins for the oracle's loss / log-prob / gradient (steps 6-7).

Independent anchors: brute-force log-sum-exp in extended precision, W=0
closed forms, hand values of the PPO-clip term (tests/golden/ppo_terms.json),
finite differences, and PyTorch CPU fp64 autograd of the
same objective (a library derivative, not a retyped one).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth


def _rand_head(T, d, V, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((T, d)) * scale
    W = rng.standard_normal((V, d)) / math.sqrt(d) * 3.0
    y = rng.integers(0, V, size=T).astype(np.int32)
    return h, W, y


def test_logprob_bruteforce_longdouble():
    """log p_y = z_y - log sum_v exp(z_v), computed directly (no max shift) in
    numpy longdouble with Python-summed exponentials."""
    T, d, V = 16, 8, 512
    h, W, y = _rand_head(T, d, V, 11)
    got = oracle.logprob(h, W, y, np.ones(T, np.uint8), logit_scale=1.25)
    for t in range(T):
        z = [np.longdouble(1.25) * sum(np.longdouble(h[t, k]) * np.longdouble(W[v, k])
                                        for k in range(d)) for v in range(V)]
        se = sum(np.exp(zz) for zz in z)
        ref = z[y[t]] - np.log(se)
        assert abs(float(ref) - got[t]) < 1e-12


def test_logprob_W_zero_is_minus_log_V():
    T, d, V = 5, 4, 512
    h, _, y = _rand_head(T, d, V, 2)
    got = oracle.logprob(h, np.zeros((V, d)), y, np.ones(T, np.uint8))
    np.testing.assert_allclose(got, -math.log(V), rtol=0, atol=1e-14)
    assert abs(got[0] - (-6.238324625039508)) < 1e-12


def test_softmax_sums_to_one():
    d, V = 6, 64
    h, W, _ = _rand_head(1, d, V, 5, scale=3.0)
    hs = np.repeat(h, V, axis=0)
    lp = oracle.logprob(hs, W, np.arange(V, dtype=np.int32), np.ones(V, np.uint8))
    assert abs(np.exp(lp).sum() - 1.0) < 1e-13


def test_ppo_term_golden(golden_dir):
    with open(os.path.join(golden_dir, "ppo_terms.json")) as f:
        g = json.load(f)
    d, V = 4, 8
    h, W, y = _rand_head(1, d, V, 9)
    lp = oracle.logprob(h, W, y, np.ones(1, np.uint8))
    for c in g["terms"]:
        old = lp - math.log(c["rho"])  # so that exp(logp - old) = rho
        r = oracle.policy_loss_rows(h, W, y, [c["A"]], old, 1, c["eps_lo"], c["eps_hi"])
        assert abs(r["rho"][0] - c["rho"]) < 1e-12
        assert abs(r["term"][0] - c["term"]) < 1e-12, c["source"]
    tt = g["two_token_grpo"]
    h2, W2, y2 = _rand_head(2, d, V, 10)
    lp2 = oracle.logprob(h2, W2, y2, np.ones(2, np.uint8))
    old2 = lp2 - np.log(tt["rho"])
    out = oracle.policy_loss_fwd_bwd(h2, W2, y2, tt["A"], old2, np.ones(2, np.uint8), 2,
                                     tt["eps"], tt["eps"], grads=False)
    # loss = -J with the token-level mean over N=2 (R7, R8)
    assert abs(out["loss"] - (-tt["objective"])) < 1e-12


def test_on_policy_loss_is_minus_mean_adv_and_zero_after_eq1():
    """north_star: old = new -> rho = 1 and loss = -mean_mask(A); with A from the
    same batch's Eq.1 every task's token mean is 0, so the loss is 0."""
    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    h = synth.bf16_bits_to_f32(hb).astype(np.float64)
    W = synth.bf16_bits_to_f32(Wb).astype(np.float64)
    an = oracle.task_adv_norm(b)
    lp = oracle.logprob(h, W, y, b["loss_mask"])
    out = oracle.policy_loss_fwd_bwd(h, W, y, an["adv_tok"], lp, b["loss_mask"], an["n_mask"],
                                     grads=False)
    m = b["loss_mask"] != 0
    assert abs(out["loss"] - (-an["adv_tok"][m].mean())) < 1e-12
    assert abs(out["loss"]) < 1e-12
    assert out["loss_stats"][0] == 0.0 and abs(out["loss_stats"][1] - 1.0) < 1e-12
    # arbitrary advantages: still -mean(A)
    A = np.random.default_rng(0).standard_normal(cfg.T)
    out2 = oracle.policy_loss_fwd_bwd(h, W, y, A, lp, b["loss_mask"], an["n_mask"], grads=False)
    assert abs(out2["loss"] - (-A[m].mean())) < 1e-12


def _torch_loss(h, W, y, A, old, mask, N, eps_lo, eps_hi, s):
    """PyTorch fp64 CPU autograd of -(1/N) sum_mask min(rho A, clamp(rho) A)."""
    ht = torch.tensor(h, dtype=torch.float64, requires_grad=True)
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    z = s * ht @ Wt.T
    logp = torch.log_softmax(z, dim=-1).gather(1, torch.tensor(y, dtype=torch.long)[:, None])[:, 0]
    rho = torch.exp(logp - torch.tensor(old))
    At = torch.tensor(A)
    term = torch.minimum(rho * At, torch.clamp(rho, 1 - eps_lo, 1 + eps_hi) * At)
    mk = torch.tensor(mask != 0)
    loss = -(term * mk).sum() / N
    loss.backward()
    return loss.item(), ht.grad.numpy(), Wt.grad.numpy(), logp.detach().numpy()


@pytest.mark.parametrize("eps", [(0.2, 0.2), (0.2, 0.28)])
@pytest.mark.parametrize("s", [1.0, 1.0 / 0.8])
def test_grads_match_torch_autograd(eps, s):
    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    T = 400
    mask = b["loss_mask"][:T].copy()
    h, W, y = _rand_head(T, 48, 200, 21)
    A = np.random.default_rng(4).standard_normal(T)
    lp = oracle.logprob(h, W, y, mask, logit_scale=s)
    old = lp + synth.make_deltas(T, 5, eps[0], eps[1], sigma=0.25)
    N = int(mask.sum())
    out = oracle.policy_loss_fwd_bwd(h, W, y, A, old, mask, N, eps[0], eps[1], s)
    tl, tgh, tgw, tlp = _torch_loss(h, W, y, A, old, mask, N, eps[0], eps[1], s)
    assert abs(out["loss"] - tl) < 1e-12
    np.testing.assert_allclose(out["logp"][mask != 0], tlp[mask != 0], atol=1e-12)
    np.testing.assert_allclose(out["grad_hidden"], tgh, atol=1e-13)
    np.testing.assert_allclose(out["grad_W"], tgw, atol=1e-13)
    assert 0.0 < out["loss_stats"][0] < 1.0  # some, not all, tokens clipped


def test_finite_differences_micro():
    """SPEC S:225 / S:607: central differences, h=1e-5, max rel err <= 1e-4 over
    all 128 parameters of the micro config (hidden 24x4 = 96, W 8x4 = 32)."""
    cfg = synth.CONFIGS["micro"]
    b = synth.make_structure(cfg)
    rng = np.random.default_rng(77)
    h = rng.standard_normal((cfg.T, cfg.d))
    W = rng.standard_normal((cfg.V, cfg.d))
    y = rng.integers(0, cfg.V, size=cfg.T).astype(np.int32)
    an = oracle.task_adv_norm(b)
    mask = b["loss_mask"]
    lp = oracle.logprob(h, W, y, mask)
    old = lp + synth.make_deltas(cfg.T, 6, sigma=0.15, margin=0.05)
    N = an["n_mask"]

    def L(hh, WW):
        return oracle.policy_loss_fwd_bwd(hh, WW, y, an["adv_tok"], old, mask, N,
                                          grads=False)["loss"]

    out = oracle.policy_loss_fwd_bwd(h, W, y, an["adv_tok"], old, mask, N)
    eps = 1e-5
    worst = 0.0
    for arr, grad in ((h, out["grad_hidden"]), (W, out["grad_W"])):
        for ij in np.ndindex(arr.shape):
            a1 = arr.copy()
            a1[ij] += eps
            a2 = arr.copy()
            a2[ij] -= eps
            fd = (L(a1, W) - L(a2, W)) / (2 * eps) if arr is h else \
                (L(h, a1) - L(h, a2)) / (2 * eps)
            an_ = grad[ij]
            scale = max(abs(an_), abs(fd), 1e-8)
            worst = max(worst, abs(fd - an_) / scale if scale > 1e-6 else abs(fd - an_))
    assert worst <= 1e-4, worst
    # unmasked rows have zero gradient
    assert np.all(out["grad_hidden"][mask == 0] == 0.0)


def test_W_zero_closed_form():
    """W = 0: p = 1/V, grad_h = 0 and grad_W_v = s sum_t c_t (1/V - [y_t = v]) h_t,
    with rho from logp = -ln V (no exponentials of logits at all)."""
    T, d, V, s = 40, 8, 16, 1.3
    rng = np.random.default_rng(8)
    h = rng.standard_normal((T, d))
    y = rng.integers(0, V, size=T).astype(np.int32)
    mask = (rng.uniform(size=T) < 0.6).astype(np.uint8)
    A = rng.standard_normal(T)
    old = -math.log(V) + synth.make_deltas(T, 9, sigma=0.3)
    N = int(mask.sum())
    out = oracle.policy_loss_fwd_bwd(h, np.zeros((V, d)), y, A, old, mask, N, 0.2, 0.2, s)
    assert np.all(out["grad_hidden"] == 0.0)
    rho = V ** -1.0 / np.exp(old)  # exp(-ln V - old)
    clipped = ((A > 0) & (rho > 1.2)) | ((A < 0) & (rho < 0.8))
    c = np.where(clipped, 0.0, rho * A / N) * (mask != 0)
    ref = np.zeros((V, d))
    for t in range(T):
        for v in range(V):
            ref[v] += s * c[t] * ((1.0 / V) - (1.0 if y[t] == v else 0.0)) * h[t]
    np.testing.assert_allclose(out["grad_W"], ref, atol=1e-14)


def test_fully_clipped_batch_has_zero_gradient():
    T, d, V = 30, 8, 32
    h, W, y = _rand_head(T, d, V, 12)
    mask = np.ones(T, np.uint8)
    lp = oracle.logprob(h, W, y, mask)
    A = np.where(np.arange(T) % 2 == 0, 1.0, -1.0)
    # A>0: rho = 1.5 > 1+eps ; A<0: rho = 0.5 < 1-eps  -> every token strictly clipped
    rho = np.where(A > 0, 1.5, 0.5)
    old = lp - np.log(rho)
    out = oracle.policy_loss_fwd_bwd(h, W, y, A, old, mask, T)
    assert out["loss_stats"][0] == 1.0
    assert np.all(out["grad_hidden"] == 0.0) and np.all(out["grad_W"] == 0.0)
    # loss = -(1/N) sum clip(rho) A = -(1/T) sum (1.2 * 1 + 0.8 * -1)
    assert abs(out["loss"] - (-(1.2 * 15 - 0.8 * 15) / T)) < 1e-12


def test_on_policy_gradient_closed_form():
    """on-policy grad = -(1/N) sum_t A_t grad logp_t, i.e. the
    cross-entropy gradient (p - onehot) scaled by A_t/N."""
    T, d, V = 20, 6, 24
    h, W, y = _rand_head(T, d, V, 14)
    mask = np.ones(T, np.uint8)
    A = np.random.default_rng(1).standard_normal(T)
    lp = oracle.logprob(h, W, y, mask)
    out = oracle.policy_loss_fwd_bwd(h, W, y, A, lp, mask, T)
    z = h @ W.T
    p = np.exp(z - z.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    G = p.copy()
    G[np.arange(T), y] -= 1.0
    G *= (A / T)[:, None]
    np.testing.assert_allclose(out["grad_hidden"], G @ W, atol=1e-13)
    np.testing.assert_allclose(out["grad_W"], G.T @ h, atol=1e-13)


def test_spot_rows_match_full():
    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    h = synth.bf16_bits_to_f32(hb).astype(np.float64)
    W = synth.bf16_bits_to_f32(Wb).astype(np.float64)
    an = oracle.task_adv_norm(b)
    lp = oracle.logprob(h, W, y, b["loss_mask"])
    old = lp + synth.make_deltas(cfg.T, 3)
    full = oracle.policy_loss_fwd_bwd(h, W, y, an["adv_tok"], old, b["loss_mask"], an["n_mask"])
    rows = an["idx"][::37]
    r = oracle.policy_loss_rows(h[rows], W, y[rows], an["adv_tok"][rows], old[rows],
                                an["n_mask"])
    np.testing.assert_allclose(r["logp"], full["logp"][rows], atol=1e-12)
    np.testing.assert_allclose(r["grad_hidden"], full["grad_hidden"][rows], atol=1e-14)


def test_bad_target_and_empty():
    h, W, y = _rand_head(4, 4, 8, 0)
    y[1] = 8
    out = oracle.policy_loss_fwd_bwd(h, W, y, np.ones(4), np.zeros(4), np.ones(4, np.uint8), 4)
    assert out["status"] & oracle.S_BAD_TARGET
    y[1] = 0
    out = oracle.policy_loss_fwd_bwd(h, W, y, np.ones(4), np.zeros(4), np.zeros(4, np.uint8), 0)
    assert out["status"] & oracle.S_NO_TOKENS and out["loss"] == 0.0


def test_grpo_step_composes():
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    h = synth.bf16_bits_to_f32(hb).astype(np.float64)
    W = synth.bf16_bits_to_f32(Wb).astype(np.float64)
    lp = oracle.logprob(h, W, y, b["loss_mask"])
    old = lp + synth.make_deltas(cfg.T, 4)
    st = oracle.grpo_step(b, h, W, y, old)
    an = oracle.task_adv_norm(b)
    sep = oracle.policy_loss_fwd_bwd(h, W, y, an["adv_tok"], old, b["loss_mask"], an["n_mask"])
    assert st["loss"] == sep["loss"]
    np.testing.assert_array_equal(st["grad_W"], sep["grad_W"])
    np.testing.assert_array_equal(st["adv_tok"], an["adv_tok"])


# --------------------------------------------------------------------------- entropy
def test_entropy_uniform_is_log_V():
    T, d, V = 6, 4, 512
    h, _, y = _rand_head(T, d, V, 31)
    lp, H = oracle.logprob_entropy(h, np.zeros((V, d)), y, np.ones(T, np.uint8))
    np.testing.assert_allclose(H, math.log(V), rtol=0, atol=1e-12)
    np.testing.assert_allclose(lp, -math.log(V), rtol=0, atol=1e-12)


def test_entropy_two_logit_closed_form():
    """d=1, W=[[1],[0]], h=[x]: z=(s x, 0), p = sigmoid(s x), H = binary entropy."""
    xs = np.linspace(-6, 6, 13)
    h = xs[:, None]
    W = np.asarray([[1.0], [0.0]])
    y = np.zeros(len(xs), np.int32)
    for s in (1.0, 1.25):
        lp, H = oracle.logprob_entropy(h, W, y, np.ones(len(xs), np.uint8), logit_scale=s)
        p = 1.0 / (1.0 + np.exp(-s * xs))
        np.testing.assert_allclose(H, -(p * np.log(p) + (1 - p) * np.log(1 - p)), atol=1e-13)
        np.testing.assert_allclose(lp, np.log(p), atol=1e-13)


def test_entropy_bruteforce_and_bounds():
    T, d, V = 10, 8, 64
    h, W, y = _rand_head(T, d, V, 33, scale=2.0)
    mask = (np.arange(T) % 3 != 0).astype(np.uint8)
    lp, H = oracle.logprob_entropy(h, W, y, mask)
    for t in range(T):
        if not mask[t]:
            assert H[t] == 0.0 and lp[t] == 0.0
            continue
        z = [sum(np.longdouble(h[t, k]) * np.longdouble(W[v, k]) for k in range(d))
             for v in range(V)]
        Z = sum(np.exp(zz) for zz in z)
        ref = -sum((np.exp(zz) / Z) * (zz - np.log(Z)) for zz in z)
        assert abs(float(ref) - H[t]) < 1e-12
        assert 0.0 <= H[t] <= math.log(V) + 1e-12
    np.testing.assert_allclose(lp, oracle.logprob(h, W, y, mask), atol=1e-13)
