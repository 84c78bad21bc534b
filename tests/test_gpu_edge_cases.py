"""Edge cases of part 2 and of the fused step on the GPU (SURVEY 8(b) error contract):
data-dependent problems raise bits in the device status word and still produce defined
outputs; host-checkable problems return error codes before any launch.
  - a masked token's target outside [0, V)      -> ST_BAD_TARGET (S:221 analogue)
  - non-finite behaviour log-prob               -> ST_NONFINITE ("abort")
  - no loss-masked token at all                 -> ST_NO_TOKENS, loss 0, zero grads (R16)
  - an empty batch (T = 0)                      -> ST_NO_TOKENS, loss 0, zero grad_W
  - d % 64 != 0, clip eps outside [0, 1), a workspace one byte short -> SHAPE / INVALID_ARG /
    WORKSPACE return codes
  - a workspace sized by max_rows: = T_eff gives the T-sized result bit for bit; below T_eff
    -> ST_ROWS_OVERFLOW, only the first max_rows masked tokens are processed, no fault."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402

from gpu_util import batch_dev, bf16_dev, t  # noqa: E402


@pytest.fixture(scope="module")
def ag():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_04206_b200 as m
    return m


def _inputs(T=512, d=64, V=512, seed=3):
    rng = np.random.default_rng(seed)
    hb = synth.to_bf16_bits(rng.standard_normal((T, d)).astype(np.float32))
    Wb = synth.to_bf16_bits((rng.standard_normal((V, d)) / np.sqrt(d)).astype(np.float32))
    y = rng.integers(0, V, T).astype(np.int32)
    old = np.full(T, -6.0, np.float32)
    adv = rng.standard_normal(T).astype(np.float32)
    mask = (rng.random(T) < 0.5).astype(np.uint8)
    return hb, Wb, y, old, adv, mask


def _loss(ag, hb, Wb, y, old, adv, mask, ws_bytes=None, **kw):
    T, d = hb.shape
    V = Wb.shape[0]
    need = ag.agentrl_policy_loss_workspace_size(T, d, V, kw.get("max_rows", 0))
    ws = ag.alloc_workspace(need if ws_bytes is None else ws_bytes)
    loss = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    gh = torch.full((max(T, 1), d), float("nan"), dtype=torch.bfloat16, device="cuda")
    gw = torch.full((V, d), float("nan"), device="cuda")
    nm = torch.tensor([int((mask != 0).sum())], dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = ag.make_loss_args(T, bf16_dev(hb) if T else torch.empty(0, d, dtype=torch.bfloat16,
                                                                       device="cuda"),
                             bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32),
                             t(mask, torch.uint8), adv_tok=t(adv, torch.float32),
                             n_mask_global=nm, **kw)
    rc = ag.agentrl_policy_loss_fwd_bwd(args, ag.make_loss_out(loss, gh, gw), ws, None, st)
    torch.cuda.synchronize()
    return rc, loss.item(), gh[:T].float().cpu().numpy(), gw.cpu().numpy(), int(st.item())


def test_bad_target_sets_status(ag):
    hb, Wb, y, old, adv, mask = _inputs()
    i = int(np.nonzero(mask)[0][3])
    y[i] = Wb.shape[0] + 5
    rc, loss, gh, gw, st = _loss(ag, hb, Wb, y, old, adv, mask)
    assert rc == 0 and st & ag.ST_BAD_TARGET


def test_unmasked_bad_target_is_ignored(ag):
    hb, Wb, y, old, adv, mask = _inputs()
    i = int(np.nonzero(mask == 0)[0][0])
    y[i] = -7  # never read: the token is not a loss token
    rc, loss, gh, gw, st = _loss(ag, hb, Wb, y, old, adv, mask)
    assert rc == 0 and st == 0 and np.isfinite(loss)
    assert np.all(gh[mask == 0] == 0)


def test_nonfinite_old_logp_sets_status(ag):
    hb, Wb, y, old, adv, mask = _inputs()
    old[int(np.nonzero(mask)[0][0])] = np.nan
    rc, loss, gh, gw, st = _loss(ag, hb, Wb, y, old, adv, mask)
    assert rc == 0 and st & ag.ST_NONFINITE


def test_all_unmasked_batch(ag):
    hb, Wb, y, old, adv, mask = _inputs()
    mask[:] = 0
    rc, loss, gh, gw, st = _loss(ag, hb, Wb, y, old, adv, mask)
    assert rc == 0 and st & ag.ST_NO_TOKENS
    assert loss == 0.0 and np.all(gh == 0) and np.all(gw == 0)


def test_fused_step_empty_and_unmasked(ag):
    """the fused step with no loss tokens: adv 0, loss 0, grads 0, ST_NO_TOKENS"""
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_structure(cfg)
    b["loss_mask"] = np.zeros_like(b["loss_mask"])
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    old = np.full(cfg.T, -6.0, np.float32)
    step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)
    step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
    torch.cuda.synchronize()
    assert int(step.status.item()) & ag.ST_NO_TOKENS
    assert step.loss.item() == 0.0
    assert torch.all(step.adv_tok == 0) and torch.all(step.grad_hidden == 0)
    assert torch.all(step.grad_W == 0)


def test_zero_length_batch(ag):
    """T = 0 (no tokens, no trajectories): defined outputs, no launch error"""
    d, V = 64, 512
    b = dict(T=0, traj_offsets=np.zeros(1, np.int64), task_id=np.zeros(0, np.int32),
             group_id=np.zeros(0, np.int32), rewards=np.zeros(0, np.float32),
             loss_mask=np.zeros(0, np.uint8), n_groups=1, n_tasks=1)
    bd = batch_dev(b)
    step = ag.Step(0, 0, 1, 1, d, V)
    Wb = _inputs(d=d, V=V)[1]
    empty_h = torch.empty(0, d, dtype=torch.bfloat16, device="cuda")
    step(bd, empty_h, bf16_dev(Wb), torch.empty(0, dtype=torch.int32, device="cuda"),
         torch.empty(0, dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    assert int(step.status.item()) & ag.ST_NO_TOKENS
    assert step.loss.item() == 0.0 and torch.all(step.grad_W == 0)


def test_host_checked_errors(ag):
    hb, Wb, y, old, adv, mask = _inputs()
    # d not a multiple of 64
    rc = _loss(ag, hb[:, :48].copy(), Wb[:, :48].copy(), y, old, adv, mask)[0]
    assert rc == ag.ERR_SHAPE
    # clip epsilon outside [0, 1)
    rc = _loss(ag, hb, Wb, y, old, adv, mask, eps_low=1.5)[0]
    assert rc == ag.ERR_INVALID_ARG
    # workspace one byte short
    need = ag.agentrl_policy_loss_workspace_size(hb.shape[0], hb.shape[1], Wb.shape[0])
    rc = _loss(ag, hb, Wb, y, old, adv, mask, ws_bytes=need - 1)[0]
    assert rc == ag.ERR_WORKSPACE


def test_max_rows_workspace(ag):
    """max_rows = T_eff: the same bits as the T-sized workspace with a far smaller buffer;
    max_rows < T_eff: ST_ROWS_OVERFLOW and the first max_rows rows only (defined outputs)."""
    hb, Wb, y, old, adv, mask = _inputs(T=1500, d=128, V=1000, seed=8)
    T, d = hb.shape
    V = Wb.shape[0]
    n = int(mask.sum())
    assert ag.agentrl_policy_loss_workspace_size(T, d, V, n) < \
        ag.agentrl_policy_loss_workspace_size(T, d, V) * 0.75
    rc0, l0, gh0, gw0, st0 = _loss(ag, hb, Wb, y, old, adv, mask)
    rc1, l1, gh1, gw1, st1 = _loss(ag, hb, Wb, y, old, adv, mask, max_rows=n)
    assert rc0 == rc1 == 0 and st0 == st1 == 0
    assert l0 == l1 and np.array_equal(gh0, gh1) and np.array_equal(gw0, gw1)
    cut = n - 200  # the first `cut` masked tokens (token order) are processed
    rc2, l2, gh2, gw2, st2 = _loss(ag, hb, Wb, y, old, adv, mask, max_rows=cut)
    assert rc2 == 0 and st2 & ag.ST_ROWS_OVERFLOW
    keep = np.zeros(T, np.uint8)
    keep[np.nonzero(mask)[0][:cut]] = 1
    # same as a batch whose mask holds only those tokens, with the full N in the mean
    args_n = n
    ws = ag.alloc_workspace(ag.agentrl_policy_loss_workspace_size(T, d, V))
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    gh = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    gw = torch.empty(V, d, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    a = ag.make_loss_args(T, bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32),
                          t(keep, torch.uint8), adv_tok=t(adv, torch.float32),
                          n_mask_global=torch.tensor([args_n], dtype=torch.int64, device="cuda"))
    assert ag.agentrl_policy_loss_fwd_bwd(a, ag.make_loss_out(loss, gh, gw), ws, None, st) == 0
    torch.cuda.synchronize()
    assert abs(loss.item() - l2) <= 1e-12 * max(abs(l2), 1e-30)
    assert np.array_equal(gh.float().cpu().numpy(), gh2)
    assert np.array_equal(gw.cpu().numpy(), gw2)
