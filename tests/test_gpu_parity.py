"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle.

Bars (north_star): integers bit-exact; advantages <= 1e-5
relative (+1e-6 absolute floor); loss <= 1e-3 relative to max(|L|, (1/N) sum|term|);
grad_hidden / grad_W max|diff| / max|ref| <= 2e-2 per tensor; logp <= 1e-3 absolute.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

from gpu_util import (adv_close, batch_dev, bf16_dev, f64, loss_tol, max_abs_rel,  # noqa: E402
                      t)


@pytest.fixture(scope="module")
def ag():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_04206_b200 as m
    return m


def run_adv(ag, b, eps_std=1e-6, mask_offset=0):
    bd = batch_dev(b)
    if mask_offset:
        buf = torch.zeros(b["T"] + mask_offset, dtype=torch.uint8, device="cuda")
        buf[mask_offset:] = bd["loss_mask"]
        bd["loss_mask"] = buf[mask_offset:]
    T = b["T"]
    n_traj = len(b["task_id"])
    ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                    b["n_tasks"]))
    adv = torch.full((max(T, 1),), float("nan"), dtype=torch.float32, device="cuda")
    ts = torch.zeros(b["n_tasks"], 3, dtype=torch.float64, device="cuda")
    nm = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = ag.agentrl_task_adv_norm(ag.make_batch(bd), eps_std, adv, ts, nm, ws, None, st)
    assert rc == 0, ag.status_string(rc)
    torch.cuda.synchronize()
    return adv[:T].cpu().numpy(), ts.cpu().numpy(), int(nm.item()), int(st.item())


@pytest.mark.parametrize("cfg", ["tiny", "ragged", "parity7b", "qwen7b", "glm9b", "skew14b"])
def test_adv_norm_parity(ag, cfg):
    b = synth.make_structure(synth.CONFIGS[cfg])
    ref = oracle.task_adv_norm(b)
    adv, ts, nm, st = run_adv(ag, b)
    assert st == (ref["status"] & ~oracle.S_NO_TOKENS)
    assert nm == ref["n_mask"]  # integer, bit-exact
    np.testing.assert_array_equal(ts[:, 0], ref["task_stats"][:, 0])  # N_i exact
    np.testing.assert_allclose(ts[:, 1], ref["task_stats"][:, 1], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ts[:, 2], ref["task_stats"][:, 2], rtol=1e-9, atol=1e-12)
    assert adv_close(adv, ref["adv_tok"])
    assert np.all(adv[b["loss_mask"] == 0] == 0.0)


@pytest.mark.parametrize("cfg", ["tiny", "ragged", "qwen7b", "glm9b", "skew14b", "qwen32b"])
def test_bookkeeping_bitexact(ag, cfg):
    """n_g, K_j, the local masked count and the fused step's stable compaction idx, bit-exact
    against the oracle (north_star: integer bookkeeping; token set P:557-569, groups
    P:1214-1218).  Part 1 alone, then the fused step with a small head (d=64, V=512) so the
    compaction is written."""
    b = synth.make_structure(synth.CONFIGS[cfg])
    ref = oracle.task_adv_norm(b)
    T, n_traj = b["T"], len(b["task_id"])
    bd = batch_dev(b)
    ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                    b["n_tasks"]))
    adv = torch.empty(T, dtype=torch.float32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert ag.agentrl_task_adv_norm(ag.make_batch(bd), 1e-6, adv, None, None, ws, None, st) == 0
    n_g, K, _, rows = ag.bookkeeping(ws, T, n_traj, b["n_groups"], b["n_tasks"])
    np.testing.assert_array_equal(n_g, ref["n_g"])
    np.testing.assert_array_equal(K, ref["K_j"])
    assert rows == ref["n_mask"]
    d, V = 64, 512
    step = ag.Step(T, n_traj, b["n_groups"], b["n_tasks"], d, V)
    step(bd, torch.zeros(T, d, dtype=torch.bfloat16, device="cuda"),
         torch.zeros(V, d, dtype=torch.bfloat16, device="cuda"),
         torch.zeros(T, dtype=torch.int32, device="cuda"),
         torch.full((T,), -6.0, dtype=torch.float32, device="cuda"))
    n_g, K, idx, rows = ag.bookkeeping(step.ws, T, n_traj, b["n_groups"], b["n_tasks"])
    np.testing.assert_array_equal(n_g, ref["n_g"])
    np.testing.assert_array_equal(K, ref["K_j"])
    assert rows == ref["n_mask"]
    np.testing.assert_array_equal(idx, ref["idx"])


def test_adv_norm_misaligned_and_ragged_T(ag):
    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    # cut to a T that is not a multiple of 16 / 4096 and mis-align the mask pointer
    off = b["traj_offsets"]
    keep = int(np.searchsorted(off, 1203, side="right")) - 1
    T = int(off[keep])
    grp_keep = sorted(set(b["group_id"][:keep].tolist()))
    b2 = dict(T=T, traj_offsets=off[:keep + 1], task_id=b["task_id"][:keep],
              group_id=b["group_id"][:keep], rewards=b["rewards"][:keep],
              loss_mask=b["loss_mask"][:T], n_groups=max(grp_keep) + 1, n_tasks=b["n_tasks"])
    ref = oracle.task_adv_norm(b2)
    for mo in (0, 1, 3):
        adv, ts, nm, st = run_adv(ag, b2, mask_offset=mo)
        assert nm == ref["n_mask"]
        assert adv_close(adv, ref["adv_tok"])


def test_adv_norm_status_bits(ag):
    base = dict(T=8, traj_offsets=np.asarray([0, 2, 4, 6, 8]), task_id=np.asarray([0, 0, 1, 1]),
                group_id=np.asarray([0, 0, 1, 1]), rewards=np.asarray([1, 0, 1, 0], np.float32),
                loss_mask=np.asarray([1, 1, 0, 1, 0, 1, 1, 0], np.uint8), n_groups=2, n_tasks=2)
    adv, ts, nm, st = run_adv(ag, base)
    assert st == 0 and nm == 5
    ref = oracle.task_adv_norm(base)
    assert adv_close(adv, ref["adv_tok"])
    _, _, _, st = run_adv(ag, dict(base, task_id=np.asarray([0, 1, 1, 1])))
    assert st & ag.ST_GROUP_SPANS_TASKS
    _, _, _, st = run_adv(ag, dict(base, group_id=np.asarray([0, 1, 2, 2]), n_groups=3))
    assert st & ag.ST_GROUP_TOO_SMALL
    _, _, _, st = run_adv(ag, dict(base, traj_offsets=np.asarray([0, 2, 4, 6, 7])))
    assert st & ag.ST_BAD_OFFSETS
    adv, _, nm, st = run_adv(ag, dict(base, loss_mask=np.zeros(8, np.uint8)))
    assert st & ag.ST_NO_TOKENS and nm == 0 and np.all(adv == 0)


def _loss_inputs(cfg_name, seed_delta=17, eps=(0.2, 0.2), sigma=0.08):
    cfg = synth.CONFIGS[cfg_name]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    h, W = f64(hb), f64(Wb)
    lp = oracle.logprob(h, W, y, b["loss_mask"])
    old = (lp + synth.make_deltas(cfg.T, seed_delta, eps[0], eps[1], sigma=sigma)).astype(np.float32)
    return cfg, b, hb, Wb, y, h, W, old


def _check_loss(ref, loss, logp, gh, gw, mask):
    N = max(int((mask != 0).sum()), 1)
    assert abs(loss - ref["loss"]) <= loss_tol(ref["loss"], 1.0 / N) + 1e-9, (loss, ref["loss"])
    m = mask != 0
    assert np.abs(logp[m] - ref["logp"][m]).max() <= 1e-3
    assert np.all(logp[~m] == 0.0)
    e1 = max_abs_rel(gh, ref["grad_hidden"])
    e2 = max_abs_rel(gw, ref["grad_W"])
    assert e1 <= 2e-2, e1
    assert e2 <= 2e-2, e2
    assert np.all(gh[~m] == 0.0)
    return e1, e2


@pytest.mark.parametrize("cfg_name,eps,scale", [("tiny", (0.2, 0.2), 1.0),
                                                ("ragged", (0.2, 0.2), 1.0),
                                                ("ragged", (0.2, 0.28), 1.0 / 0.8)])
def test_policy_loss_parity(ag, cfg_name, eps, scale):
    cfg, b, hb, Wb, y, h, W, old = _loss_inputs(cfg_name, eps=eps)
    if scale != 1.0:
        lp = oracle.logprob(h, W, y, b["loss_mask"], logit_scale=scale)
        old = (lp + synth.make_deltas(cfg.T, 3, eps[0], eps[1])).astype(np.float32)
    an = oracle.task_adv_norm(b)
    adv32 = an["adv_tok"].astype(np.float32)
    ref = oracle.policy_loss_fwd_bwd(h, W, y, adv32.astype(np.float64), old.astype(np.float64),
                                     b["loss_mask"], an["n_mask"], eps[0], eps[1], scale)
    T, d, V = cfg.T, cfg.d, cfg.V
    hidden, Wd = bf16_dev(hb), bf16_dev(Wb)
    mask = t(b["loss_mask"], torch.uint8)
    ws = ag.alloc_workspace(ag.agentrl_policy_loss_workspace_size(T, d, V))
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    logp = torch.full((T,), float("nan"), device="cuda")
    gh = torch.full((T, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    gw = torch.full((V, d), float("nan"), device="cuda")
    stats = torch.zeros(5, dtype=torch.float64, device="cuda")
    nm = torch.tensor([an["n_mask"]], dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = ag.make_loss_args(T, hidden, Wd, t(y, torch.int32), t(old, torch.float32), mask,
                             adv_tok=t(adv32, torch.float32), n_mask_global=nm, eps_low=eps[0],
                             eps_high=eps[1], logit_scale=scale)
    out = ag.make_loss_out(loss, gh, gw, logp, stats)
    rc = ag.agentrl_policy_loss_fwd_bwd(args, out, ws, None, st)
    assert rc == 0, ag.status_string(rc)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    _check_loss(ref, loss.item(), logp.cpu().numpy(), gh.float().cpu().numpy(),
                gw.cpu().numpy(), b["loss_mask"])
    s = stats.cpu().numpy()
    assert abs(s[0] - ref["loss_stats"][0]) < 1e-9 + 2.0 / an["n_mask"]  # clip fraction
    assert s[3] == an["n_mask"]


def test_onehot_cancellation_rows(ag):
    """Rows with p_y -> 1 at large |z| (z_y ~ 20..32, 1 - p_y ~ 1e-9 .. 1e-4) and a large
    unclipped coefficient (A < 0, rho = e^3): grad_hidden = c sum_v (p_v - [v=y]) W_v is a
    difference of nearly equal terms.  Checked per ROW against the oracle (the tensor-level
    metric would hide it).  Two failure modes this pins: an lse rounded to the ulp of z_y
    (~2e-6) loses all of 1 - p_y; an fp16 P~ flushes the target tile's other entries
    (exp(z - z_y) < 6e-8) to zero.  The range stops at 1 - p_y ~ 1e-9: below ~1e-12 the fp64
    oracle's own p_y - 1 = exp(z_y - lse) - 1 cancels (4% at 8e-14, checked against 80-bit
    long double), so it would no longer be the arbiter."""
    rng = np.random.default_rng(2510_04206 + 77)
    T, d, V = 256, 64, 512
    Wf = rng.standard_normal((V, d)).astype(np.float32) / np.float32(np.sqrt(d))
    Wb = synth.to_bf16_bits(Wf)
    W = f64(Wb)
    y = rng.integers(0, V, T).astype(np.int32)
    a = rng.uniform(20.0, 32.0, T)  # target logit
    wy = W[y]
    h = a[:, None] * wy / (wy * wy).sum(1, keepdims=True) + 0.05 * rng.standard_normal((T, d))
    hb = synth.to_bf16_bits(h.astype(np.float32))
    h = f64(hb)
    mask = np.ones(T, np.uint8)
    lp = oracle.logprob(h, W, y, mask)
    assert lp.max() < -1e-10 and lp.min() > -1e-3  # p_y near 1 on every row, within fp64 reach
    old = (lp - 3.0).astype(np.float32)  # rho = e^3 > 1 + eps, A < 0: not clipped
    adv = np.full(T, -1.0, np.float32)
    ref = oracle.policy_loss_rows(h, W, y, adv.astype(np.float64), old.astype(np.float64), T)
    assert not ref["clipped"].any()
    ws = ag.alloc_workspace(ag.agentrl_policy_loss_workspace_size(T, d, V))
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    logp = torch.full((T,), float("nan"), device="cuda")
    gh = torch.full((T, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    gw = torch.full((V, d), float("nan"), device="cuda")
    nm = torch.tensor([T], dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = ag.make_loss_args(T, bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32),
                             t(old, torch.float32), t(mask, torch.uint8),
                             adv_tok=t(adv, torch.float32), n_mask_global=nm)
    rc = ag.agentrl_policy_loss_fwd_bwd(args, ag.make_loss_out(loss, gh, gw, logp), ws, None, st)
    assert rc == 0, ag.status_string(rc)
    torch.cuda.synchronize()
    got = gh.float().cpu().numpy()
    want = ref["grad_hidden"]
    row_err = np.abs(got - want).max(1) / np.abs(want).max(1)
    assert row_err.max() <= 2e-2, (row_err.max(), -lp[np.argmax(row_err)])


def _run_step(ag, cfg, b, hb, Wb, y, old, eps=(0.2, 0.2), scale=1.0):
    step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V,
                   eps_low=eps[0], eps_high=eps[1], logit_scale=scale)
    step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
    torch.cuda.synchronize()
    return step


def test_longk_full_tensor_parity(ag):
    """Long reduction loops compared element by element with the oracle (the full-size configs
    only get spot checks): grad_W's K = T_eff ~ 26.6K rows (416 k-blocks) and grad_hidden's
    K = V = 8192 (128 k-blocks), both beyond the default backward progress-throttle lead (96
    k-blocks), with grad_hidden in two waves of CTA-pair tiles; default schedule.  The
    throttle's wait episodes during this call are reported (a lead-1 lockstep build that must
    wait is the bitwise schedule variant in tests/test_gpu_variants.py)."""
    cfg, b, hb, Wb, y, h, W, old = _loss_inputs("longk")
    ref = oracle.grpo_step(b, h, W, y, old.astype(np.float64))
    w0 = ag.debug_throttle_waits()
    step = _run_step(ag, cfg, b, hb, Wb, y, old)
    w1 = ag.debug_throttle_waits()
    print("throttle wait episodes (fwd, grad_W, grad_hidden):", [b_ - a_ for a_, b_ in zip(w0, w1)])
    assert int(step.status.item()) & ~ag.ST_GROUP_TOO_SMALL == 0
    assert adv_close(step.adv_tok.cpu().numpy(), ref["adv_tok"])
    e1, e2 = _check_loss(ref, step.loss.item(), step.logp.cpu().numpy(),
                         step.grad_hidden.float().cpu().numpy(), step.grad_W.cpu().numpy(),
                         b["loss_mask"])
    print("longk max-abs-rel grad_hidden %.3e grad_W %.3e" % (e1, e2))


@pytest.mark.parametrize("cfg_name", ["tiny", "ragged"])
def test_grpo_step_parity(ag, cfg_name):
    cfg, b, hb, Wb, y, h, W, old = _loss_inputs(cfg_name)
    ref = oracle.grpo_step(b, h, W, y, old.astype(np.float64))
    step = _run_step(ag, cfg, b, hb, Wb, y, old)
    assert int(step.status.item()) & ~ag.ST_GROUP_TOO_SMALL == ref["status"] & ~oracle.S_GROUP_TOO_SMALL
    assert adv_close(step.adv_tok.cpu().numpy(), ref["adv_tok"])
    np.testing.assert_array_equal(step.task_stats.cpu().numpy()[:, 0], ref["task_stats"][:, 0])
    _check_loss(ref, step.loss.item(), step.logp.cpu().numpy(),
                step.grad_hidden.float().cpu().numpy(), step.grad_W.cpu().numpy(),
                b["loss_mask"])


@pytest.mark.slow
def test_grpo_step_parity7b(ag):
    """Real Qwen2.5-7B head dims (d=3584, V=152064), full-tensor parity."""
    cfg, b, hb, Wb, y, h, W, old = _loss_inputs("parity7b")
    ref = oracle.grpo_step(b, h, W, y, old.astype(np.float64))
    step = _run_step(ag, cfg, b, hb, Wb, y, old)
    assert adv_close(step.adv_tok.cpu().numpy(), ref["adv_tok"])
    _check_loss(ref, step.loss.item(), step.logp.cpu().numpy(),
                step.grad_hidden.float().cpu().numpy(), step.grad_W.cpu().numpy(),
                b["loss_mask"])


def test_on_policy_loss_is_zero(ag):
    """old = logp (oracle) -> rho = 1 -> loss = -mean(A_tilde) = 0 (north_star)."""
    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    lp = oracle.logprob(f64(hb), f64(Wb), y, b["loss_mask"]).astype(np.float32)
    step = _run_step(ag, cfg, b, hb, Wb, y, lp)
    an = oracle.task_adv_norm(b)
    scale = np.abs(an["adv_tok"]).sum() / an["n_mask"]
    assert abs(step.loss.item()) <= 1e-3 * scale
    s = step.loss_stats.cpu().numpy()
    assert s[0] == 0.0 and abs(s[1] - 1.0) < 1e-4


def test_determinism(ag):
    cfg, b, hb, Wb, y, h, W, old = _loss_inputs("ragged")
    s1 = _run_step(ag, cfg, b, hb, Wb, y, old)
    r1 = [x.clone() for x in (s1.loss, s1.adv_tok, s1.grad_hidden, s1.grad_W, s1.logp)]
    s1(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
    torch.cuda.synchronize()
    for a, bb in zip(r1, (s1.loss, s1.adv_tok, s1.grad_hidden, s1.grad_W, s1.logp)):
        assert torch.equal(a, bb)


def _full_size_case(ag, cfg_name, n_spot=24, shard_of=None):
    """shard_of = (world, rank): the rank's LPT shard of the global batch, run as
    one single-GPU batch -- the per-rank problem size of the multi-GPU configs"""
    import dataclasses
    cfg = synth.CONFIGS[cfg_name]
    b = synth.make_structure(cfg)
    if shard_of is not None:
        world, rank = shard_of
        off = b["traj_offsets"]
        cs = np.concatenate([[0], np.cumsum(b["loss_mask"].astype(np.int64))])
        ng = cs[off[1:]] - cs[off[:-1]]
        rog = synth.shard_groups_lpt(np.bincount(b["group_id"], weights=ng,
                                                 minlength=b["n_groups"]), world)
        b = {k: v for k, v in synth.shard_batch(b, rog, rank).items() if k != "token_index"}
        cfg = dataclasses.replace(cfg, T=int(b["T"]))
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    old = synth.make_old_logp_free(cfg.T, 99)
    step = _run_step(ag, cfg, b, hb, Wb, y, old)
    an = oracle.task_adv_norm(b)
    assert int(step.status.item()) & ~ag.ST_GROUP_TOO_SMALL == 0
    assert adv_close(step.adv_tok.cpu().numpy(), an["adv_tok"])
    logp = step.logp.cpu().numpy()
    gh = step.grad_hidden.float().cpu().numpy()
    rng = np.random.default_rng(5)
    rows = rng.choice(an["idx"], size=n_spot, replace=False)
    # always include rows where p_y is close to 1 (planted: |h| far above the bulk), the
    # onehot-cancellation case
    hn = np.abs(f64(hb[an["idx"]])).max(1)
    planted = an["idx"][np.argsort(-hn)[:4]]
    rows = np.unique(np.concatenate([rows, planted]))
    Wf = f64(Wb)
    h_rows = f64(hb[rows])
    r = oracle.policy_loss_rows(h_rows, Wf, y[rows], an["adv_tok"][rows].astype(np.float32)
                                .astype(np.float64), old[rows].astype(np.float64), an["n_mask"])
    # skip rows whose ratio sits within 1e-4 of a clip boundary (decision ill-conditioned)
    near = (np.abs(r["rho"] - 0.8) < 1e-4) | (np.abs(r["rho"] - 1.2) < 1e-4)
    ok = ~near
    assert np.abs(logp[rows][ok] - r["logp"][ok]).max() <= 1e-3
    # grad_hidden rows: per-row max-abs-rel against the row's own scale and the tensor scale
    gref = r["grad_hidden"][ok]
    err = np.abs(gh[rows][ok] - gref).max() / max(np.abs(gref).max(), 1e-30)
    assert err <= 2e-2, err
    # every masked row's log-prob and the loss against an INDEPENDENT full-size computation:
    # plain fp32 torch (matmul + logsumexp on the same bf16 inputs, chunked; no TF32) for the
    # log-probs and the oracle's advantages -- the loss is not recomputed from the GPU's logp
    m = b["loss_mask"] != 0
    assert not torch.backends.cuda.matmul.allow_tf32
    Wt = bf16_dev(Wb).float()
    hdev = bf16_dev(hb)
    lp_ref = np.empty(len(an["idx"]), dtype=np.float64)
    with torch.no_grad():
        for s0 in range(0, len(an["idx"]), 4096):
            ii = torch.from_numpy(an["idx"][s0:s0 + 4096].astype(np.int64)).cuda()
            z = hdev[ii].float() @ Wt.T
            yy = torch.from_numpy(y[an["idx"][s0:s0 + 4096]].astype(np.int64)).cuda()
            lp = z.gather(1, yy[:, None])[:, 0] - torch.logsumexp(z, dim=1)
            lp_ref[s0:s0 + len(ii)] = lp.double().cpu().numpy()
    del Wt
    assert np.abs(logp[an["idx"]] - lp_ref).max() <= 1e-3
    A = an["adv_tok"][an["idx"]].astype(np.float32).astype(np.float64)
    rho = np.exp(lp_ref - old[an["idx"]])
    term = np.minimum(rho * A, np.clip(rho, 0.8, 1.2) * A)
    L = -term.sum() / an["n_mask"]
    assert abs(step.loss.item() - L) <= 1e-3 * max(abs(L), np.abs(term).sum() / an["n_mask"])
    gw = step.grad_W
    # sum_v G_tv = 0  =>  column sums of grad_W vanish (relative to the row scale)
    colsum = gw.double().sum(0).abs().max().item()
    assert colsum <= 2e-2 * gw.abs().max().item() * math.sqrt(cfg.V)
    # <grad_hidden, hidden> = <grad_W, W> = s * sum G o Z
    hd, Wd = bf16_dev(hb).double(), bf16_dev(Wb).double()
    lhs = (step.grad_hidden.double() * hd).sum().item()
    rhs = (gw.double() * Wd).sum().item()
    assert abs(lhs - rhs) <= 2e-2 * max(abs(lhs), abs(rhs), 1e-12) + 1e-6
    return step


@pytest.mark.slow
def test_full_size_qwen7b_spot_rows(ag):
    _full_size_case(ag, "qwen7b")


@pytest.mark.slow
def test_full_size_glm9b_spot_rows(ag):
    _full_size_case(ag, "glm9b", n_spot=16)


@pytest.mark.slow
@pytest.mark.parametrize("cfg_name", ["qwen32b", "skew14b"])
def test_full_size_rank_shard_spot_rows(ag, cfg_name):
    """the 8-GPU configs at their per-rank size and head dims (d=5120, V=152064)"""
    _full_size_case(ag, cfg_name, n_spot=12, shard_of=(8, 0))
