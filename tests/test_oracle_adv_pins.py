"""Pins for the oracle's task advantage normalization (steps 1-5).

Pinned against values the paper / SPEC fix (tests/golden/*.json, each with its
citation), closed forms and invariants -- never against the oracle itself.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# GRPO group advantage
# --------------------------------------------------------------------------
def test_grpo_golden(golden_dir):
    g = _load(golden_dir, "grpo_group_advantage.json")
    for case in g["cases"]:
        r = np.asarray(case["rewards"], np.float32)
        got = oracle.group_advantage(np.zeros(len(r), np.int32), r, 1)
        # rewards are given to the oracle as f32 (the ABI type); the hand values
        # were computed from the decimal rewards, so allow the f32 rounding of -0.2
        np.testing.assert_allclose(got, case["adv"], rtol=1e-6, atol=1e-7, err_msg=case["source"])


def test_grpo_all_equal_is_exact_zero():
    for val in (0.1, -0.2, 1.0, 0.0, 0.3):
        for K in (2, 3, 8):
            got = oracle.group_advantage(np.zeros(K, np.int32), np.full(K, val, np.float32), 1)
            assert np.all(got == 0.0), (val, K, got)


def test_grpo_invariants():
    rng = np.random.default_rng(1)
    for _ in range(50):
        K = int(rng.integers(2, 12))
        r = rng.choice(np.asarray([1.0, 0.0, -0.2], np.float32), size=K)
        if r.max() == r.min():
            r[0] = 1.0 if r[0] != 1.0 else 0.0
        a = oracle.group_advantage(np.zeros(K, np.int32), r, 1)
        assert abs(a.sum()) < 1e-9
        # population std of A_hat is 1 (floor not binding)
        assert abs(np.sqrt(np.mean(a * a)) - 1.0) < 1e-9
        # shift invariance with an exactly representable shift
        a2 = oracle.group_advantage(np.zeros(K, np.int32), (r.astype(np.float64) + 0.5)
                                    .astype(np.float32), 1)
        np.testing.assert_allclose(a2, a, atol=1e-6)
        # positive scale invariance (power of two: exact in f32)
        a3 = oracle.group_advantage(np.zeros(K, np.int32), r * np.float32(4.0), 1)
        np.testing.assert_allclose(a3, a, atol=1e-12)


def test_grpo_groups_independent_and_unordered():
    # interleaved membership must not matter
    gid = np.asarray([0, 1, 0, 1, 0, 1], np.int32)
    r = np.asarray([1, 0, 0, 1, 1, 1], np.float32)
    a = oracle.group_advantage(gid, r, 2)
    a0 = oracle.group_advantage(np.zeros(3, np.int32), r[gid == 0], 1)
    a1 = oracle.group_advantage(np.zeros(3, np.int32), r[gid == 1], 1)
    np.testing.assert_array_equal(a[gid == 0], a0)
    np.testing.assert_array_equal(a[gid == 1], a1)


# --------------------------------------------------------------------------
# task normalization (Eq.1)
# --------------------------------------------------------------------------
def _one_token_batch(task, adv_hat, n):
    """Trajectory g has n[g] masked tokens; apply Eq.1 through oracle_apply."""
    task = np.asarray(task, np.int32)
    n = np.asarray(n, np.int64)
    n_tasks = int(task.max()) + 1
    st = oracle.task_moments(task, n, np.asarray(adv_hat, np.float64), n_tasks)
    return st


def test_task_norm_golden(golden_dir):
    g = _load(golden_dir, "task_adv_norm.json")
    for case in g["cases"]:
        task = np.asarray(case["task"], np.int32)
        n = np.asarray(case["n"], np.int64)
        ah = np.asarray(case["adv_hat"], np.float64)
        n_tasks = int(task.max()) + 1
        st = oracle.task_moments(task, n, ah, n_tasks)
        # run the full apply step over a packed stream of fully-masked trajectories
        off = np.zeros(len(n) + 1, np.int64)
        off[1:] = np.cumsum(n)
        T = int(off[-1])
        mask = np.ones(T, np.uint8)
        lib = oracle.lib()
        at = np.zeros(len(n), np.float64)
        adv = np.zeros(T, np.float64)
        idx = np.zeros(T, np.int64)
        nm = np.zeros(1, np.int64)
        ts = np.ascontiguousarray(st.reshape(-1))
        lib.oracle_apply(T, len(n), oracle._p(off), oracle._p(task), oracle._p(mask),
                         oracle._p(ah), oracle._p(ts), 1e-6, oracle._p(at), oracle._p(adv),
                         oracle._p(idx), oracle._p(nm))
        if "adv_tilde" in case:
            np.testing.assert_allclose(at, case["adv_tilde"], rtol=1e-12, atol=1e-12,
                                       err_msg=case["source"])
        if "mu" in case:
            assert abs(st[0, 1] - case["mu"]) < 1e-12
            assert abs(st[0, 2] - case["sigma"]) < 1e-12
        if "uniform_group_adv_tilde" in case:
            np.testing.assert_allclose(at[4:], case["uniform_group_adv_tilde"], rtol=1e-12)
        # broadcast: every token of trajectory g carries A_tilde_g
        np.testing.assert_array_equal(adv, np.repeat(at, n))


@pytest.mark.parametrize("cfg", ["tiny", "ragged", "parity7b", "qwen7b"])
def test_task_norm_zero_mean_unit_std(cfg):
    """per task the token-level advantages have zero mean, unit variance."""
    b = synth.make_structure(synth.CONFIGS[cfg])
    r = oracle.task_adv_norm(b)
    assert r["status"] & ~oracle.S_GROUP_TOO_SMALL == 0
    mask = b["loss_mask"] != 0
    tok_task = np.repeat(b["task_id"], np.diff(b["traj_offsets"]))
    for i in range(b["n_tasks"]):
        sel = mask & (tok_task == i)
        a = r["adv_tok"][sel]
        if len(a) == 0:
            continue
        if r["task_stats"][i, 2] > 1e-6:
            assert abs(a.mean()) < 1e-9
            assert abs(a.std() - 1.0) < 1e-9
        else:
            assert np.all(a == 0.0)
    assert np.all(r["adv_tok"][~mask] == 0.0)


def test_counts_and_compaction_bruteforce():
    for cfg in ("tiny", "ragged", "qwen7b"):
        b = synth.make_structure(synth.CONFIGS[cfg])
        r = oracle.task_adv_norm(b)
        off, mk = b["traj_offsets"], b["loss_mask"]
        ng = [int((mk[off[g]:off[g + 1]] != 0).sum()) for g in range(len(b["task_id"]))]
        np.testing.assert_array_equal(r["n_g"], ng)
        np.testing.assert_array_equal(r["K_j"], np.bincount(b["group_id"],
                                                            minlength=b["n_groups"]))
        np.testing.assert_array_equal(r["idx"], np.nonzero(mk)[0])
        assert r["n_mask"] == int((mk != 0).sum())
        tok_task = np.repeat(b["task_id"], np.diff(off))
        for i in range(b["n_tasks"]):
            assert r["task_stats"][i, 0] == float(((mk != 0) & (tok_task == i)).sum())


def test_task_norm_monotone_and_scale_invariant():
    rng = np.random.default_rng(7)
    b = synth.make_structure(synth.CONFIGS["ragged"])
    r = oracle.task_adv_norm(b)
    ng = r["n_g"]
    for i in range(b["n_tasks"]):
        sel = b["task_id"] == i
        ah = rng.standard_normal(sel.sum())
        st = oracle.task_moments(np.zeros(sel.sum(), np.int32), ng[sel], ah, 1)
        at = (ah - st[0, 1]) / st[0, 2]
        order = np.argsort(ah)
        assert np.all(np.diff(at[order]) > 0)  # S:230 strictly monotone
        st2 = oracle.task_moments(np.zeros(sel.sum(), np.int32), ng[sel], 3.5 * ah, 1)
        at2 = (3.5 * ah - st2[0, 1]) / st2[0, 2]
        np.testing.assert_allclose(at2, at, atol=1e-12)


def test_equal_length_closed_form():
    """Equal n for every trajectory -> mu_i = 0 and A_tilde = A_hat / sqrt(f_i),
    f_i = fraction of the task's trajectories in non-uniform groups (closed form)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        n_groups = int(rng.integers(2, 6))
        K = int(rng.integers(2, 6))
        gid = np.repeat(np.arange(n_groups), K).astype(np.int32)
        r = rng.choice(np.asarray([1.0, 0.0, -0.2], np.float32), size=n_groups * K)
        ah = oracle.group_advantage(gid, r, n_groups)
        mixed = np.asarray([r[gid == j].max() != r[gid == j].min() for j in range(n_groups)])
        if not mixed.any():
            continue
        f = mixed.sum() / n_groups
        st = oracle.task_moments(np.zeros(len(gid), np.int32), np.full(len(gid), 5, np.int64),
                                 ah, 1)
        assert abs(st[0, 1]) < 1e-12
        np.testing.assert_allclose((ah - st[0, 1]) / st[0, 2], ah / np.sqrt(f), atol=1e-9)


def test_empty_task_and_validation():
    # task 1 has no masked tokens -> stats (0,0,0), no error (R16)
    b = dict(T=8, traj_offsets=np.asarray([0, 2, 4, 6, 8]), task_id=np.asarray([0, 0, 1, 1]),
             group_id=np.asarray([0, 0, 1, 1]), rewards=np.asarray([1, 0, 1, 0], np.float32),
             loss_mask=np.asarray([1, 1, 0, 1, 0, 0, 0, 0], np.uint8), n_groups=2, n_tasks=2)
    r = oracle.task_adv_norm(b)
    assert r["status"] == 0
    np.testing.assert_array_equal(r["task_stats"][1], [0, 0, 0])
    # group spanning tasks
    b2 = dict(b, task_id=np.asarray([0, 1, 1, 1]))
    assert oracle.task_adv_norm(b2)["status"] & oracle.S_GROUP_SPANS_TASKS
    # group of size 1
    b3 = dict(b, group_id=np.asarray([0, 1, 2, 2]), n_groups=3)
    assert oracle.task_adv_norm(b3)["status"] & oracle.S_GROUP_TOO_SMALL
    # bad offsets
    b4 = dict(b, traj_offsets=np.asarray([0, 2, 1, 6, 8]))
    assert oracle.task_adv_norm(b4)["status"] & oracle.S_BAD_OFFSETS
    # no masked tokens at all
    b5 = dict(b, loss_mask=np.zeros(8, np.uint8))
    assert oracle.task_adv_norm(b5)["status"] & oracle.S_NO_TOKENS


def test_sharded_stats_equal_global():
    """Sharding whole groups over ranks and summing (N_i, sum n A_hat, sum n A_hat^2)
    reproduces the global mu_i, sigma_i (the decomposition the multi-GPU path uses)."""
    b = synth.make_structure(synth.CONFIGS["qwen7b"])
    g = oracle.task_adv_norm(b)
    gtok = np.bincount(b["group_id"], weights=g["n_g"], minlength=b["n_groups"])
    for world in (2, 3, 8):
        rog = synth.shard_groups_lpt(gtok, world)
        N = np.zeros(b["n_tasks"])
        S = np.zeros(b["n_tasks"])
        Q = np.zeros(b["n_tasks"])
        for rank in range(world):
            sb = synth.shard_batch(b, rog, rank)
            loc = oracle.task_adv_norm(sb)
            for i in range(b["n_tasks"]):
                sel = sb["task_id"] == i
                N[i] += loc["n_g"][sel].sum()
                S[i] += (loc["n_g"][sel] * loc["adv_hat"][sel]).sum()
                Q[i] += (loc["n_g"][sel] * loc["adv_hat"][sel] ** 2).sum()
        mu = S / N
        sd = np.sqrt(np.maximum(Q / N - mu * mu, 0))
        np.testing.assert_array_equal(N, g["task_stats"][:, 0])
        np.testing.assert_allclose(mu, g["task_stats"][:, 1], atol=1e-12)
        np.testing.assert_allclose(sd, g["task_stats"][:, 2], rtol=1e-10)
