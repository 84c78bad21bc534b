"""fp64 CPU oracle for the AgentRL hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It wraps
``oracle/agentrl_oracle.c`` (plain C, fp64, OpenMP across independent outputs)
through ctypes and shares nothing with ``paper_2510_04206_b200`` (the CUDA
path): no imports, no headers, no helpers.

Each wrapper cites the PAPER.md passage the C function follows; the C file
header lists them all.  See DESIGN.md section "Readings" for R1..R18.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "agentrl_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "oracle_variants.c")]
_LIB = os.path.join(_HERE, "liboracle.so")

# data-dependent status bits
S_BAD_TARGET = 1
S_NONFINITE = 2
S_BAD_OFFSETS = 4
S_GROUP_SPANS_TASKS = 8
S_GROUP_TOO_SMALL = 16
S_NO_TOKENS = 32


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB) or any(
            os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", *_SRCS, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64, i32, f64 = C.c_int64, C.c_int32, C.c_double
        L.oracle_validate.argtypes = [i64, i32, i32, i32, P, P, P]
        L.oracle_task_adv_norm.argtypes = [i64, i32, i32, i32, P, P, P, P, P, f64,
                                           P, P, P, P, P, P, P, P]
        L.oracle_group_advantage.argtypes = [i32, i32, P, P, f64, P]
        L.oracle_task_moments.argtypes = [i32, i32, P, P, P, P]
        L.oracle_apply.argtypes = [i64, i32, P, P, P, P, P, f64, P, P, P, P]
        L.oracle_policy_loss_fwd_bwd.argtypes = [i64, i32, i32, P, P, P, P, P, P, f64, f64, f64,
                                                 i64, P, P, P, P, P]
        L.oracle_policy_loss_rows.argtypes = [i32, i32, P, P, P, P, P, i64, f64, f64, f64, i64,
                                              P, P]
        L.oracle_logprob.argtypes = [i64, i32, i32, P, P, P, P, f64, P]
        L.oracle_grpo_step.argtypes = [i64, i32, i32, i32, P, P, P, P, P, f64, i32, i32, P, P, P,
                                       P, f64, f64, f64, P, P, P, P, P, P, P]
        L.oracle_logprob_entropy.argtypes = [i64, i32, i32, P, P, P, P, f64, P, P]
        L.oracle_grpo_group_weights.argtypes = [i64, i32, i32, P, P, P, P]
        L.oracle_grpo_group_weights.restype = i64
        L.oracle_policy_loss_ex.argtypes = [i64, i32, i32, P, P, P, P, P, P, f64, f64, f64, i64,
                                            f64, P, P, P, P, P, P, P]
        L.oracle_num_threads.restype = C.c_int
        L.oracle_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def validate(T, traj_offsets, task_id, group_id, n_groups, n_tasks) -> int:
    off = _c(traj_offsets, np.int64)
    tid = _c(task_id, np.int32)
    gid = _c(group_id, np.int32)
    return lib().oracle_validate(int(T), len(tid), int(n_groups), int(n_tasks), _p(off), _p(tid),
                                 _p(gid))


def group_advantage(group_id, rewards, n_groups, eps_std=1e-6):
    """GRPO A_hat per trajectory (R1 population std, R2 exact-equal -> 0)."""
    gid = _c(group_id, np.int32)
    r = _c(rewards, np.float32)
    out = np.zeros(len(gid), np.float64)
    lib().oracle_group_advantage(len(gid), int(n_groups), _p(gid), _p(r), float(eps_std), _p(out))
    return out


def task_moments(task_id, n_g, adv_hat, n_tasks):
    """Per-task (N_i, mu_i, sigma_i) over the token set A_i^tok."""
    tid = _c(task_id, np.int32)
    ng = _c(n_g, np.int64)
    ah = _c(adv_hat, np.float64)
    out = np.zeros(3 * int(n_tasks), np.float64)
    lib().oracle_task_moments(len(tid), int(n_tasks), _p(tid), _p(ng), _p(ah), _p(out))
    return out.reshape(int(n_tasks), 3)


def task_adv_norm(b, eps_std=1e-6):
    """Steps 1-5 (Eq.1 after P:1263).  ``b`` is a dict with
    T, traj_offsets, task_id, group_id, rewards, loss_mask, n_groups, n_tasks."""
    T = int(b["T"])
    off = _c(b["traj_offsets"], np.int64)
    tid = _c(b["task_id"], np.int32)
    gid = _c(b["group_id"], np.int32)
    rw = _c(b["rewards"], np.float32)
    mk = _c(b["loss_mask"], np.uint8)
    n_traj, n_groups, n_tasks = len(tid), int(b["n_groups"]), int(b["n_tasks"])
    n_g = np.zeros(n_traj, np.int64)
    K_j = np.zeros(max(n_groups, 1), np.int32)
    ah = np.zeros(n_traj, np.float64)
    at = np.zeros(n_traj, np.float64)
    ts = np.zeros(3 * n_tasks, np.float64)
    adv = np.zeros(T, np.float64)
    idx = np.zeros(max(T, 1), np.int64)
    nm = np.zeros(1, np.int64)
    st = lib().oracle_task_adv_norm(T, n_traj, n_groups, n_tasks, _p(off), _p(tid), _p(gid),
                                    _p(rw), _p(mk), float(eps_std), _p(n_g), _p(K_j), _p(ah),
                                    _p(at), _p(ts), _p(adv), _p(idx), _p(nm))
    n = int(nm[0])
    return dict(status=st, n_g=n_g, K_j=K_j[:n_groups], adv_hat=ah, adv_tilde=at,
                task_stats=ts.reshape(n_tasks, 3), adv_tok=adv, idx=idx[:n], n_mask=n)


def policy_loss_fwd_bwd(hidden, W, target, adv_tok, old_logp, loss_mask, n_mask_global,
                        eps_lo=0.2, eps_hi=0.2, logit_scale=1.0, grads=True):
    """Loss, logp, grad_hidden, grad_W (R7-R10).
    hidden [T,d] and W [V,d] are taken as fp64 (pass bf16-rounded values)."""
    h = _c(hidden, np.float64)
    w = _c(W, np.float64)
    T, d = h.shape
    V = w.shape[0]
    tg = _c(target, np.int32)
    adv = _c(adv_tok, np.float64)
    old = _c(old_logp, np.float64)
    mk = _c(loss_mask, np.uint8)
    loss = np.zeros(1, np.float64)
    logp = np.zeros(T, np.float64)
    gh = np.zeros((T, d), np.float64) if grads else None
    gw = np.zeros((V, d), np.float64) if grads else None
    stats = np.zeros(4, np.float64)
    st = lib().oracle_policy_loss_fwd_bwd(T, d, V, _p(h), _p(w), _p(tg), _p(adv), _p(old), _p(mk),
                                          float(eps_lo), float(eps_hi), float(logit_scale),
                                          int(n_mask_global), _p(loss), _p(logp), _p(gh), _p(gw),
                                          _p(stats))
    return dict(status=st, loss=float(loss[0]), logp=logp, grad_hidden=gh, grad_W=gw,
                loss_stats=stats)


def policy_loss_rows(hidden_rows, W, target_rows, adv_rows, old_rows, n_mask_global,
                     eps_lo=0.2, eps_hi=0.2, logit_scale=1.0, grad_rows=True):
    """Spot rows: per token (lse, logp, rho, term, coef, clipped) and grad_hidden row."""
    h = _c(hidden_rows, np.float64)
    w = _c(W, np.float64)
    n, d = h.shape
    V = w.shape[0]
    out = np.zeros((n, 6), np.float64)
    gh = np.zeros((n, d), np.float64) if grad_rows else None
    st = lib().oracle_policy_loss_rows(d, V, _p(h), _p(w), _p(_c(target_rows, np.int32)),
                                       _p(_c(adv_rows, np.float64)), _p(_c(old_rows, np.float64)),
                                       n, float(eps_lo), float(eps_hi), float(logit_scale),
                                       int(n_mask_global), _p(out), _p(gh))
    if st != 0:
        raise ValueError(f"oracle_policy_loss_rows status {st}")
    return dict(lse=out[:, 0], logp=out[:, 1], rho=out[:, 2], term=out[:, 3], coef=out[:, 4],
                clipped=out[:, 5].astype(bool), grad_hidden=gh)


def logprob(hidden, W, target, loss_mask, logit_scale=1.0):
    h = _c(hidden, np.float64)
    w = _c(W, np.float64)
    T, d = h.shape
    out = np.zeros(T, np.float64)
    st = lib().oracle_logprob(T, d, w.shape[0], _p(h), _p(w), _p(_c(target, np.int32)),
                              _p(_c(loss_mask, np.uint8)), float(logit_scale), _p(out))
    if st != 0:
        raise ValueError(f"oracle_logprob status {st}")
    return out


def grpo_group_weights(b):
    """w_t = 1/(G K_j n_g(t)) of the GRPO group-level aggregation (reading R7b).
    Returns (w [T], G = number of groups with at least one trajectory)."""
    T = int(b["T"])
    off = _c(b["traj_offsets"], np.int64)
    gid = _c(b["group_id"], np.int32)
    w = np.zeros(T, np.float64)
    G = lib().oracle_grpo_group_weights(T, len(off) - 1, int(b["n_groups"]), _p(off), _p(gid),
                                        _p(_c(b["loss_mask"], np.uint8)), _p(w))
    if G < 0:
        raise ValueError("group id outside [0, n_groups)")
    return w, int(G)


def policy_loss_ex(hidden, W, target, adv_tok, old_logp, loss_mask, n_mask_global,
                   eps_lo=0.2, eps_hi=0.2, logit_scale=1.0, kl_beta=0.0, ref_logp=None,
                   weights=None, grads=True):
    """Loss variants (oracle_variants.c): KL penalty (k3) and per-token
    weights (token mean by default; GRPO group mean via grpo_group_weights)."""
    h = _c(hidden, np.float64)
    w = _c(W, np.float64)
    T, d = h.shape
    V = w.shape[0]
    loss = np.zeros(1, np.float64)
    logp = np.zeros(T, np.float64)
    gh = np.zeros((T, d), np.float64) if grads else None
    gw = np.zeros((V, d), np.float64) if grads else None
    stats = np.zeros(5, np.float64)
    ref = None if ref_logp is None else _c(ref_logp, np.float64)
    wt = None if weights is None else _c(weights, np.float64)
    st = lib().oracle_policy_loss_ex(T, d, V, _p(h), _p(w), _p(_c(target, np.int32)),
                                     _p(_c(adv_tok, np.float64)), _p(_c(old_logp, np.float64)),
                                     _p(_c(loss_mask, np.uint8)), float(eps_lo), float(eps_hi),
                                     float(logit_scale), int(n_mask_global), float(kl_beta),
                                     _p(ref), _p(wt), _p(loss), _p(logp), _p(gh), _p(gw),
                                     _p(stats))
    return dict(status=st, loss=float(loss[0]), logp=logp, grad_hidden=gh, grad_W=gw,
                loss_stats=stats)


def logprob_entropy(hidden, W, target, loss_mask, logit_scale=1.0):
    """(logp, entropy) of every masked token; plain definitions."""
    h = _c(hidden, np.float64)
    w = _c(W, np.float64)
    T, d = h.shape
    lp = np.zeros(T, np.float64)
    ent = np.zeros(T, np.float64)
    st = lib().oracle_logprob_entropy(T, d, w.shape[0], _p(h), _p(w), _p(_c(target, np.int32)),
                                      _p(_c(loss_mask, np.uint8)), float(logit_scale), _p(lp),
                                      _p(ent))
    if st != 0:
        raise ValueError(f"oracle_logprob_entropy status {st}")
    return lp, ent


def grpo_step(b, hidden, W, target, old_logp, eps_std=1e-6, eps_lo=0.2, eps_hi=0.2,
              logit_scale=1.0, grads=True):
    """Fused steps 1-7 on one (global) batch."""
    T = int(b["T"])
    off = _c(b["traj_offsets"], np.int64)
    tid = _c(b["task_id"], np.int32)
    gid = _c(b["group_id"], np.int32)
    rw = _c(b["rewards"], np.float32)
    mk = _c(b["loss_mask"], np.uint8)
    n_tasks = int(b["n_tasks"])
    h = _c(hidden, np.float64)
    w = _c(W, np.float64)
    d = h.shape[1]
    V = w.shape[0]
    adv = np.zeros(T, np.float64)
    ts = np.zeros(3 * n_tasks, np.float64)
    loss = np.zeros(1, np.float64)
    logp = np.zeros(T, np.float64)
    gh = np.zeros((T, d), np.float64) if grads else None
    gw = np.zeros((V, d), np.float64) if grads else None
    stats = np.zeros(4, np.float64)
    st = lib().oracle_grpo_step(T, len(tid), int(b["n_groups"]), n_tasks, _p(off), _p(tid),
                                _p(gid), _p(rw), _p(mk), float(eps_std), d, V, _p(h), _p(w),
                                _p(_c(target, np.int32)), _p(_c(old_logp, np.float64)),
                                float(eps_lo), float(eps_hi), float(logit_scale), _p(adv), _p(ts),
                                _p(loss), _p(logp), _p(gh), _p(gw), _p(stats))
    return dict(status=st, adv_tok=adv, task_stats=ts.reshape(n_tasks, 3), loss=float(loss[0]),
                logp=logp, grad_hidden=gh, grad_W=gw, loss_stats=stats)
