"""Seeded synthetic rollout batches shaped like the paper's workloads.

INPUT GENERATION ONLY -- this module holds none of the method's arithmetic
(no advantages, no logits, no losses).  It is the one piece both the oracle
tests and the CUDA path's tests/bench use, and it imports neither.

Recipe:
  * tasks in order ALFWorld, DB, KG, OS, WebShop; groups of G=8
    rollouts ("sampling eight times per rollout");
  * trajectory lengths lognormal(sigma=0.5) apportioned to sum exactly to T
    (largest remainder);
  * t_g turns per trajectory, uniform in a per-task range (KG capped at 15,
    P:1525; the other ranges are invented);
  * each turn = observation span (mask 0) then assistant span (mask 1); the
    assistant fraction per task 0.30/0.45/0.40/0.45/0.40, +-0.1 per trajectory;
  * rewards: -0.2 w.p. p_abn (Task-Limit rates), else 1 w.p.
    p_succ (Qwen2.5-14B prompting success), else 0 (reward scheme
    P:1333-1335);
  * hidden ~ N(0,1), W ~ N(0, (3/sqrt(d))^2), both rounded to bf16; 5% of
    masked tokens "planted" so that p_y is close to 1;
  * target ~ U[0,V); behaviour-log-prob offsets delta ~ N(0, 0.08^2) kept
    at least `margin` away from the clip boundaries.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 2510_04206

TASKS = ("alfworld", "db", "kg", "os", "webshop")
TURN_RANGE = {"alfworld": (5, 24), "db": (1, 5), "kg": (2, 15), "os": (1, 8), "webshop": (3, 15)}
ASSIST_FRAC = {"alfworld": 0.30, "db": 0.45, "kg": 0.40, "os": 0.45, "webshop": 0.40}
P_ABN = {"alfworld": 0.68, "db": 0.043, "kg": 0.213, "os": 0.444, "webshop": 0.275}
P_SUCC = {"alfworld": 0.087, "db": 0.484, "kg": 0.353, "os": 0.260, "webshop": 0.176}


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n_tasks: int
    groups_per_task: tuple  # groups of each task
    rollouts: int  # trajectories per group (K)
    T: int  # packed tokens (global)
    d: int
    V: int
    task_token_share: tuple | None = None  # None = proportional to #trajectories
    assist_scale: float = 1.0  # multiplies the per-task assistant fraction
    index: int = 0


def _cfg(name, n_tasks, gpt, K, T, d, V, share=None, assist_scale=1.0, index=0):
    return Config(name, n_tasks, tuple(gpt), K, T, d, V, share, assist_scale, index)


CONFIGS = {
    # BASELINE.json configs[0]: 2 tasks x 2 groups x 4 rollouts, 48 tok/rollout, d=64, V=512
    "tiny": _cfg("tiny", 2, (2, 2), 4, 768, 64, 512, index=0),
    # configs[1]: Qwen2.5-7B head, 5 tasks x 8 groups x 8 rollouts, 32K tokens, 1 GPU
    "qwen7b": _cfg("qwen7b", 5, (8,) * 5, 8, 32768, 3584, 152064, index=1),
    # configs[2]: GLM-4-9B head, 5 tasks (16 groups each), ~40% assistant, 128K tokens
    "glm9b": _cfg("glm9b", 5, (16,) * 5, 8, 131072, 4096, 151552, index=2),
    # configs[3]: Qwen2.5-32B head, 5 x 32 x 8, 512K tokens over 8 GPUs
    "qwen32b": _cfg("qwen32b", 5, (32,) * 5, 8, 524288, 5120, 152064, index=3),
    # configs[4]: 5 tasks with 20:1 token imbalance (geometric shares), 14B head, 256K
    "skew14b": _cfg("skew14b", 5, (16,) * 5, 8, 262144, 5120, 152064,
                    share=(20.0, 9.46, 4.47, 2.11, 1.0), index=4),
    # added parity cases: real Qwen2.5-7B head dims, few tokens
    "parity7b": _cfg("parity7b", 5, (1,) * 5, 4, 384, 3584, 152064, index=5),
    # ragged tiles: V not a multiple of 256, T_eff not a multiple of 128, d = 3*64
    "ragged": _cfg("ragged", 3, (2, 3, 2), 4, 1536, 192, 2000, index=6),
    # finite-difference case: 2 tasks x 1 group x 2 rollouts x 6 tokens, d=4, V=8
    "micro": _cfg("micro", 2, (1, 1), 2, 24, 4, 8, index=7),
    # long reduction loops at oracle-affordable cost (full-tensor gradient parity): T_eff ~ 26.6K
    # rows = 416 k-blocks in grad_W, V = 8192 = 128 k-blocks in grad_hidden, both longer than
    # the backward progress-throttle lead (96 k-blocks), 104 x 1 grad_hidden tiles (> 74 CTA
    # pairs: two waves)
    "longk": _cfg("longk", 5, (4,) * 5, 8, 65536, 256, 8192, index=8),
}


# ----------------------------------------------------------------------------
# bf16 helpers (a storage format, not method arithmetic)
# ----------------------------------------------------------------------------
def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 -> bf16 (round to nearest even); return uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ----------------------------------------------------------------------------
# batch structure
# ----------------------------------------------------------------------------
def _apportion(weights: np.ndarray, total: int, minimum: int = 1) -> np.ndarray:
    """Integer parts >= minimum summing exactly to total (largest remainder)."""
    n = len(weights)
    assert total >= n * minimum
    w = np.asarray(weights, np.float64)
    w = w / w.sum()
    free = total - n * minimum
    raw = w * free
    base = np.floor(raw).astype(np.int64)
    rem = free - int(base.sum())
    order = np.argsort(-(raw - base), kind="stable")
    base[order[:rem]] += 1
    return base + minimum


def make_structure(cfg: Config, seed: int | None = None, hand_rewards: bool | None = None):
    """Batch descriptor arrays: traj_offsets, task_id, group_id, rewards, loss_mask."""
    rng = np.random.default_rng(SEED_BASE + cfg.index if seed is None else seed)
    K = cfg.rollouts
    task_of_traj, group_of_traj = [], []
    gid = 0
    for i in range(cfg.n_tasks):
        for _ in range(cfg.groups_per_task[i]):
            task_of_traj += [i] * K
            group_of_traj += [gid] * K
            gid += 1
    task_id = np.asarray(task_of_traj, np.int32)
    group_id = np.asarray(group_of_traj, np.int32)
    n_traj = len(task_id)

    # trajectory lengths: lognormal, optionally per-task token shares (skew)
    w = rng.lognormal(0.0, 0.5, size=n_traj)
    if cfg.task_token_share is not None:
        share = np.asarray(cfg.task_token_share, np.float64)
        share = share / share.sum()
        for i in range(cfg.n_tasks):
            sel = task_id == i
            w[sel] = w[sel] / w[sel].sum() * share[i]
    if cfg.name == "tiny":
        lengths = np.full(n_traj, cfg.T // n_traj, np.int64)
    else:
        lengths = _apportion(w, cfg.T, minimum=2)
    offsets = np.zeros(n_traj + 1, np.int64)
    offsets[1:] = np.cumsum(lengths)
    assert offsets[-1] == cfg.T

    mask = np.zeros(cfg.T, np.uint8)
    for g in range(n_traj):
        name = TASKS[task_id[g] % len(TASKS)]
        L = int(lengths[g])
        lo, hi = TURN_RANGE[name]
        if cfg.name == "tiny":
            turns = 3
        else:
            turns = int(rng.integers(lo, hi + 1))
        turns = max(1, min(turns, L // 2))
        if cfg.name == "tiny":
            # 3 turns, assistant spans of 4..12 tokens (SURVEY 8(d) tiny)
            a_sp = rng.integers(4, 13, size=turns)
        else:
            frac = ASSIST_FRAC[name] * cfg.assist_scale + rng.uniform(-0.1, 0.1)
            frac = min(max(frac, 0.05), 1.0)
            A = min(max(int(round(frac * L)), turns), L - turns)
            a_sp = _apportion(rng.uniform(0.5, 1.5, size=turns), A, minimum=1)
        O = L - int(a_sp.sum())
        o_sp = _apportion(rng.uniform(0.5, 1.5, size=turns), O, minimum=1) if O >= turns else \
            np.asarray([O] + [0] * (turns - 1), np.int64)
        pos = int(offsets[g])
        for k in range(turns):  # observation span, then assistant span (an action a_t)
            pos += int(o_sp[k])
            mask[pos:pos + int(a_sp[k])] = 1
            pos += int(a_sp[k])
        assert pos <= offsets[g + 1]

    if hand_rewards is None:
        hand_rewards = cfg.name in ("tiny", "micro")
    if hand_rewards and cfg.name == "tiny":
        # one mixed group, one all-0 group, one all-(-0.2) group, one mixed with -0.2
        rewards = np.asarray([1, 0, 0, 1, 0, 0, 0, 0, -0.2, -0.2, -0.2, -0.2, 1, -0.2, 0, 1],
                             np.float32)
    elif hand_rewards and cfg.name == "micro":
        rewards = np.asarray([1, 0, 0, 1], np.float32)
    else:
        rewards = np.zeros(n_traj, np.float32)
        u = rng.uniform(size=n_traj)
        v = rng.uniform(size=n_traj)
        for g in range(n_traj):
            name = TASKS[task_id[g] % len(TASKS)]
            if u[g] < P_ABN[name]:
                rewards[g] = -0.2
            elif v[g] < P_SUCC[name]:
                rewards[g] = 1.0
    return dict(T=cfg.T, traj_offsets=offsets, task_id=task_id, group_id=group_id,
                rewards=rewards, loss_mask=mask, n_groups=int(gid), n_tasks=cfg.n_tasks)


# ----------------------------------------------------------------------------
# model-side inputs
# ----------------------------------------------------------------------------
def make_head(cfg: Config, seed: int | None = None, plant_frac: float = 0.05,
              mask: np.ndarray | None = None, planted_logit: float = 24.0,
              target_tokens: int | None = None):
    """hidden bf16 bits [T,d], W bf16 bits [V,d], target i32 [T].

    hidden ~ N(0,1), W ~ N(0,(3/sqrt d)^2) -> logits std ~ 3.  A fraction of
    masked tokens gets hidden = a * W_y/|W_y| + 0.5 noise with a chosen so that
    the target logit is ~planted_logit above the bulk (p_y close to 1).
    """
    rng = np.random.default_rng(SEED_BASE + 1000 + cfg.index if seed is None else seed)
    T = cfg.T if target_tokens is None else target_tokens
    d, V = cfg.d, cfg.V
    W = (rng.standard_normal((V, d), dtype=np.float32) * np.float32(3.0 / math.sqrt(d)))
    W_bits = to_bf16_bits(W)
    del W
    Wf = bf16_bits_to_f32(W_bits).reshape(V, d)
    hidden = rng.standard_normal((T, d), dtype=np.float32)
    target = rng.integers(0, V, size=T).astype(np.int32)
    if plant_frac > 0 and mask is not None:
        cand = np.nonzero(mask[:T])[0]
        n_plant = int(round(plant_frac * len(cand)))
        if n_plant > 0:
            rows = rng.choice(cand, size=n_plant, replace=False)
            wy = Wf[target[rows]]
            nrm = np.linalg.norm(wy, axis=1, keepdims=True).astype(np.float32)
            # h = a W_y with a = planted/|W_y|^2 -> z_y ~ planted (+ noise, std ~1.5)
            a = np.float32(planted_logit) / (nrm * nrm)
            hidden[rows] = a * wy + np.float32(0.5) * hidden[rows]
    h_bits = to_bf16_bits(hidden).reshape(T, d)
    return h_bits, W_bits.reshape(V, d), target


def make_deltas(n: int, seed: int, eps_lo=0.2, eps_hi=0.2, sigma=0.08, margin=0.02):
    """delta ~ N(0, sigma^2) for old_logp = logp_ref + delta, rejecting draws that
    put rho = exp(-delta) within `margin` of 1-eps_lo or 1+eps_hi."""
    rng = np.random.default_rng(seed)
    out = np.empty(n, np.float64)
    filled = 0
    while filled < n:
        x = rng.normal(0.0, sigma, size=max(16, 2 * (n - filled)))
        rho = np.exp(-x)
        ok = (np.abs(rho - (1 - eps_lo)) >= margin) & (np.abs(rho - (1 + eps_hi)) >= margin)
        x = x[ok][: n - filled]
        out[filled:filled + len(x)] = x
        filled += len(x)
    return out


def make_old_logp_free(T: int, seed: int, mean=-9.0, sd=3.0):
    """Behaviour log-probs drawn without reference to any model (full-size cases
    where no oracle forward over every token is affordable)."""
    rng = np.random.default_rng(seed)
    return np.minimum(rng.normal(mean, sd, size=T), -1e-3).astype(np.float32)



def make_variable_k(b: dict, seed: int, k_range=(2, 7), empty_frac=0.15):
    """Re-group a batch structure into groups of unequal size K_{i,j} (K_{i,j} is per
    sample) within each task, and clear the loss mask of a fraction of the trajectories (members
    without assistant tokens).  Offsets, task ids and rewards are kept; group ids are re-densified
    in trajectory order.  Structure only: no method arithmetic."""
    rng = np.random.default_rng(seed)
    task = b["task_id"]
    gid = np.empty(len(task), np.int32)
    j = 0
    for i in range(int(b["n_tasks"])):
        members = np.nonzero(task == i)[0]
        pos = 0
        while pos < len(members):
            k = int(rng.integers(k_range[0], k_range[1] + 1))
            if len(members) - pos - k < k_range[0]:
                k = len(members) - pos
            gid[members[pos:pos + k]] = j
            j += 1
            pos += k
    mask = b["loss_mask"].copy()
    off = b["traj_offsets"]
    for g in np.nonzero(rng.uniform(size=len(task)) < empty_frac)[0]:
        mask[off[g]:off[g + 1]] = 0
    return dict(b, group_id=gid, n_groups=int(j), loss_mask=mask)

def make_sweep_structure(T: int, tok_per_traj: int = 400, K: int = 8, n_tasks: int = 5,
                         seed: int = SEED_BASE + 99):
    """Vectorised batch structure for the adv-norm bandwidth sweep (~400
    tokens/trajectory, 5 tasks, G=8): fixed-length trajectories of 5 turns, each turn an
    observation span then an assistant span (~40% assistant), rewards {1, 0, -0.2}."""
    rng = np.random.default_rng(seed)
    n_traj = max(K, (T // tok_per_traj) // K * K)
    lens = np.full(n_traj, T // n_traj, np.int64)
    lens[: T - int(lens.sum())] += 1
    off = np.zeros(n_traj + 1, np.int64)
    off[1:] = np.cumsum(lens)
    n_groups = n_traj // K
    group_id = np.repeat(np.arange(n_groups), K).astype(np.int32)
    task_id = (group_id % n_tasks).astype(np.int32)
    pos = np.arange(T, dtype=np.int64)
    traj = np.repeat(np.arange(n_traj), lens)
    rel = (pos - off[traj]) * 5 // lens[traj]              # turn index 0..4
    within = (pos - off[traj]) - rel * lens[traj] // 5      # position inside the turn
    turn_len = lens[traj] // 5
    mask = (within >= (turn_len * 6) // 10).astype(np.uint8)  # last 40% of each turn
    rewards = rng.choice(np.asarray([1.0, 0.0, -0.2], np.float32), size=n_traj)
    return dict(T=int(T), traj_offsets=off, task_id=task_id, group_id=group_id,
                rewards=rewards, loss_mask=mask, n_groups=int(n_groups), n_tasks=n_tasks)


def shard_groups_lpt(group_tokens: np.ndarray, world: int) -> np.ndarray:
    """Deterministic LPT bin-packing of whole groups onto ranks:
    largest masked-token count first (ties: lower group id) to the least-loaded
    rank (ties: lower rank).  Returns rank_of_group [n_groups]."""
    order = sorted(range(len(group_tokens)), key=lambda j: (-int(group_tokens[j]), j))
    load = [0] * world
    out = np.zeros(len(group_tokens), np.int32)
    for j in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[j] = r
        load[r] += int(group_tokens[j])
    return out


def shard_batch(b: dict, rank_of_group: np.ndarray, rank: int):
    """Packed local stream of one rank: the trajectories of its groups in global
    order; group ids re-densified locally (task ids stay global)."""
    off = b["traj_offsets"]
    sel = [g for g in range(len(b["task_id"])) if rank_of_group[b["group_id"][g]] == rank]
    groups = sorted({int(b["group_id"][g]) for g in sel})
    remap = {j: k for k, j in enumerate(groups)}
    lens = np.asarray([off[g + 1] - off[g] for g in sel], np.int64)
    loff = np.zeros(len(sel) + 1, np.int64)
    loff[1:] = np.cumsum(lens)
    tok = np.concatenate([np.arange(off[g], off[g + 1]) for g in sel]) if sel else \
        np.zeros(0, np.int64)
    return dict(T=int(loff[-1]), traj_offsets=loff,
                task_id=b["task_id"][sel].astype(np.int32),
                group_id=np.asarray([remap[int(b["group_id"][g])] for g in sel], np.int32),
                rewards=b["rewards"][sel].astype(np.float32),
                loss_mask=b["loss_mask"][tok].astype(np.uint8),
                n_groups=len(groups), n_tasks=b["n_tasks"], token_index=tok)
