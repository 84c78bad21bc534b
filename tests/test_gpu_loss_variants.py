"""GPU parity of the objective variants against the variant oracle
(oracle/oracle_variants.c): the k3 KL penalty with reference log-probs (P:1103 / P:1119),
caller-supplied per-token weights, and the GRPO group-level aggregation
E_{i,j}[1/K_{i,j} sum_g ...] in the fused step, on batches with unequal K_{i,j}
and members without masked tokens.  Same bars as tests/test_gpu_parity.py."""
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


def _inputs(cfg_name):
    cfg = synth.CONFIGS[cfg_name]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    h, W = f64(hb), f64(Wb)
    lp = oracle.logprob(h, W, y, b["loss_mask"])
    old = (lp + synth.make_deltas(cfg.T, 41)).astype(np.float32)
    ref = (lp + np.random.default_rng(42).normal(0, 0.3, cfg.T)).astype(np.float32)
    return cfg, b, hb, Wb, y, h, W, old, ref


def _check(ref, loss, gh, gw, mask, scale):
    assert abs(loss - ref["loss"]) <= 1e-3 * max(abs(ref["loss"]), scale) + 1e-9, (loss, ref["loss"])
    assert max_abs_rel(gh, ref["grad_hidden"]) <= 2e-2
    assert max_abs_rel(gw, ref["grad_W"]) <= 2e-2
    assert np.all(gh[mask == 0] == 0)


@pytest.mark.parametrize("beta,weighted", [(0.1, False), (0.0, True), (0.25, True)])
def test_standalone_kl_and_weights(ag, beta, weighted):
    cfg, b, hb, Wb, y, h, W, old, ref_lp = _inputs("ragged")
    an = oracle.task_adv_norm(b)
    adv32 = an["adv_tok"].astype(np.float32)
    mask = b["loss_mask"]
    wts = None
    if weighted:  # arbitrary positive per-token weights (caller-defined aggregation)
        wts = (np.random.default_rng(7).uniform(0.5, 2.0, cfg.T) / an["n_mask"]).astype(np.float32)
    ref = oracle.policy_loss_ex(h, W, y, adv32.astype(np.float64), old.astype(np.float64), mask,
                                an["n_mask"], kl_beta=beta, ref_logp=ref_lp.astype(np.float64),
                                weights=None if wts is None else wts.astype(np.float64))
    T, d, V = cfg.T, cfg.d, cfg.V
    ws = ag.alloc_workspace(ag.agentrl_policy_loss_workspace_size(T, d, V))
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    gh = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    gw = torch.empty(V, d, device="cuda")
    stats = torch.zeros(5, dtype=torch.float64, device="cuda")
    nm = torch.tensor([an["n_mask"]], dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = ag.make_loss_args(T, bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32),
                             t(old, torch.float32), t(mask, torch.uint8),
                             adv_tok=t(adv32, torch.float32), n_mask_global=nm, kl_beta=beta,
                             ref_logp=t(ref_lp, torch.float32),
                             tok_weight=None if wts is None else t(wts, torch.float32))
    rc = ag.agentrl_policy_loss_fwd_bwd(args, ag.make_loss_out(loss, gh, gw, None, stats), ws,
                                        None, st)
    assert rc == 0, ag.status_string(rc)
    torch.cuda.synchronize()
    _check(ref, loss.item(), gh.float().cpu().numpy(), gw.cpu().numpy(), mask, 1.0 / an["n_mask"])
    s = stats.cpu().numpy()
    assert abs(s[4] - ref["loss_stats"][4]) <= 1e-3 * max(ref["loss_stats"][4], 1e-3)


def test_standalone_seq_agg_needs_weights(ag):
    cfg, b, hb, Wb, y, h, W, old, ref_lp = _inputs("tiny")
    T, d, V = cfg.T, cfg.d, cfg.V
    ws = ag.alloc_workspace(ag.agentrl_policy_loss_workspace_size(T, d, V))
    args = ag.make_loss_args(T, bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32),
                             t(old, torch.float32), t(b["loss_mask"], torch.uint8),
                             adv_tok=t(np.zeros(T, np.float32), torch.float32),
                             n_mask_global=torch.ones(1, dtype=torch.int64, device="cuda"),
                             loss_agg=1)
    out = ag.make_loss_out(torch.zeros(1, dtype=torch.float64, device="cuda"),
                           torch.empty(T, d, dtype=torch.bfloat16, device="cuda"),
                           torch.empty(V, d, device="cuda"))
    rc = ag.agentrl_policy_loss_fwd_bwd(args, out, ws, None,
                                        torch.zeros(1, dtype=torch.int32, device="cuda"))
    assert rc == ag.ERR_INVALID_ARG


@pytest.mark.parametrize("cfg_name,beta,kr", [("tiny", 0.0, None), ("ragged", 0.0, (2, 7)),
                                             ("ragged", 0.2, (2, 7)), ("parity7b", 0.0, (1, 3))])
def test_fused_group_mean(ag, cfg_name, beta, kr):
    cfg, b, hb, Wb, y, h, W, old, ref_lp = _inputs(cfg_name)
    if kr:  # unequal group sizes (K = 1 included for parity7b), members without masked tokens
        b = synth.make_variable_k(b, seed=5 + cfg.index, k_range=kr)
        ks = np.bincount(b["group_id"])
        assert ks.min() != ks.max()
    an = oracle.task_adv_norm(b)
    w, G = oracle.grpo_group_weights(b)
    ref = oracle.policy_loss_ex(h, W, y, an["adv_tok"], old.astype(np.float64), b["loss_mask"],
                                an["n_mask"], kl_beta=beta, ref_logp=ref_lp.astype(np.float64),
                                weights=w)
    step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V,
                   kl_beta=beta, loss_agg=1)
    step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32),
         ref_logp=t(ref_lp, torch.float32))
    torch.cuda.synchronize()
    assert int(step.status.item()) & ~ag.ST_GROUP_TOO_SMALL == 0
    assert adv_close(step.adv_tok.cpu().numpy(), an["adv_tok"])
    _check(ref, step.loss.item(), step.grad_hidden.float().cpu().numpy(),
           step.grad_W.cpu().numpy(), b["loss_mask"], 1.0 / max(an["n_mask"], 1))
