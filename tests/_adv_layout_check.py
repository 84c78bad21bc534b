"""Subprocess body for tests/test_gpu_adv_layouts.py: part 1 (and the fused step's compaction,
through the loss and gradients) on adversarial batch layouts, with the library AGENTRL_LIB
names (the default build or an adv-norm driver variant), against the oracle.  Layouts (seeded, synthetic):
  short    trajectories of 0..5 tokens (empty ones included): > 32 trajectory starts per
           512-token chunk, many per lane
  long     few trajectories of ~40K tokens: every trajectory spans many chunks and blocks
  shuffled group ids not contiguous in trajectory order, groups of 2..20 members (both sides
           of the 16-member register path), a task with no masked tokens
  bigtraj  > 2048 trajectories (the large driver), mixed lengths
  contig   > 2048 trajectories in contiguous groups of 2..16 (the large driver's fast path
           without member lists), mixed lengths with empty trajectories
  huge     16M tokens in 1,500 trajectories (small driver): with a -DADV_KC_CAP=64 build every
           block stages several windows and trajectories cross window boundaries
  glm9b    the BASELINE glm9b batch structure (synth), under whichever driver the build picks
The integer bookkeeping (n_g, K_j, the local masked count and the fused step's compaction idx)
is compared bit-exactly (agentrl_debug_bookkeeping).
Exit code 0 = parity holds.  (Input generation, plumbing and comparison only.)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2510_04206_b200 as ag  # noqa: E402
from gpu_util import adv_close, batch_dev, bf16_dev, f64, max_abs_rel, t  # noqa: E402


def layout(kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "short":
        n_traj = 1600
        lens = rng.integers(0, 6, n_traj)
    elif kind == "long":
        n_traj = 24
        lens = rng.integers(30000, 50000, n_traj)
    elif kind == "huge":
        n_traj = 1500
        lens = rng.integers(4000, 18000, n_traj)
    elif kind == "shuffled":
        n_traj = 900
        lens = rng.integers(1, 200, n_traj)
    else:  # bigtraj, contig
        n_traj = 5000 if kind == "bigtraj" else 6000
        lens = np.where(rng.random(n_traj) < 0.5, rng.integers(0, 8, n_traj),
                        rng.integers(100, 600, n_traj))
    # groups of 2..20 members, ids shuffled over trajectories, one task per group
    sizes = []
    left = n_traj
    while left > 0:
        k = int(min(left, rng.integers(2, 17 if kind == "contig" else 21)))
        if left - k == 1:  # no group of one
            k = k + 1 if (kind != "contig" or k < 16) else k - 1
        sizes.append(k)
        left -= k
    n_groups = len(sizes)
    n_tasks = 5
    gid = np.repeat(np.arange(n_groups), sizes)
    if kind not in ("long", "huge", "contig"):
        rng.shuffle(gid)
    gtask = rng.integers(0, n_tasks - 1, n_groups)  # task n_tasks-1 has no trajectories
    tid = gtask[gid]
    rew = rng.choice(np.asarray([1.0, 0.0, -0.2], np.float32), n_traj)
    off = np.zeros(n_traj + 1, np.int64)
    off[1:] = np.cumsum(lens)
    T = int(off[-1])
    mask = (rng.random(T) < 0.4).astype(np.uint8)
    mask[mask == 1] = rng.integers(1, 256, int(mask.sum()))  # any nonzero byte (R18)
    return dict(T=T, traj_offsets=off, task_id=tid.astype(np.int32),
                group_id=gid.astype(np.int32), rewards=rew, loss_mask=mask,
                n_groups=n_groups, n_tasks=n_tasks)


def run_adv(b, mask_offset=0, out_offset=0):
    """out_offset / mask_offset: the output / mask pointers start that many elements into
    their buffers (not 16-byte aligned: the scalar store and direct-load paths)"""
    bd = batch_dev(b)
    T, n_traj = b["T"], len(b["task_id"])
    if mask_offset:
        mbuf = torch.zeros(T + mask_offset, dtype=torch.uint8, device="cuda")
        mbuf[mask_offset:] = bd["loss_mask"]
        bd["loss_mask"] = mbuf[mask_offset:]
    ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                    b["n_tasks"]))
    # NaN canaries before (out_offset) and after (64) the output: no write may land there
    buf = torch.full((max(T, 1) + out_offset + 64,), float("nan"), dtype=torch.float32,
                     device="cuda")
    adv = buf[out_offset:out_offset + max(T, 1)]
    ts = torch.zeros(b["n_tasks"], 3, dtype=torch.float64, device="cuda")
    nm = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = ag.agentrl_task_adv_norm(ag.make_batch(bd), 1e-6, adv, ts, nm, ws, None, st)
    assert rc == 0, ag.status_string(rc)
    torch.cuda.synchronize()
    bk = ag.bookkeeping(ws, T, n_traj, b["n_groups"], b["n_tasks"])
    canary = torch.cat([buf[:out_offset], buf[out_offset + max(T, 1):]])
    assert bool(torch.isnan(canary).all()), "adv_tok write outside [0, T)"
    return adv[:T].cpu().numpy(), ts.cpu().numpy(), int(nm.item()), int(st.item()), bk


def check_bookkeeping(kind, ref, bk, with_idx):
    n_g, K, idx, rows = bk
    np.testing.assert_array_equal(n_g, ref["n_g"], err_msg=kind)
    np.testing.assert_array_equal(K, ref["K_j"], err_msg=kind)
    assert rows == ref["n_mask"], (kind, rows, ref["n_mask"])
    if with_idx:
        np.testing.assert_array_equal(idx, ref["idx"], err_msg=kind)


def check_idx(kind, b, ref, d=64, V=512):
    """the fused step's compaction, bit-exact (a small head: only part 1's output matters)"""
    T = b["T"]
    hidden = torch.zeros(T, d, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(V, d, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(T, dtype=torch.int32, device="cuda")
    old = torch.full((T,), -6.0, dtype=torch.float32, device="cuda")
    step = ag.Step(T, len(b["task_id"]), b["n_groups"], b["n_tasks"], d, V)
    step(batch_dev(b), hidden, W, y, old)
    torch.cuda.synchronize()
    check_bookkeeping(kind, ref, ag.bookkeeping(step.ws, T, len(b["task_id"]), b["n_groups"],
                                                b["n_tasks"]), True)


def check_adv(kind, b):
    ref = oracle.task_adv_norm(b)
    adv, ts, nm, st, bk = run_adv(b)
    check_bookkeeping(kind, ref, bk, False)
    assert st == (ref["status"] & ~oracle.S_NO_TOKENS), (kind, st, ref["status"])
    assert nm == ref["n_mask"], (kind, nm, ref["n_mask"])
    np.testing.assert_array_equal(ts[:, 0], ref["task_stats"][:, 0])
    np.testing.assert_allclose(ts[:, 1:], ref["task_stats"][:, 1:], rtol=1e-9, atol=1e-12)
    assert adv_close(adv, ref["adv_tok"]), kind
    assert np.all(adv[b["loss_mask"] == 0] == 0.0), kind


def check_step(kind, b, d=64, V=512):
    """the fused step consumes part 1's compaction: loss and grads pin it"""
    rng = np.random.default_rng(7)
    T = b["T"]
    hb = synth.to_bf16_bits(rng.standard_normal((T, d)).astype(np.float32))
    Wb = synth.to_bf16_bits((rng.standard_normal((V, d)) * 3 / np.sqrt(d)).astype(np.float32))
    y = rng.integers(0, V, T).astype(np.int32)
    h, W = f64(hb), f64(Wb)
    lp = oracle.logprob(h, W, y, b["loss_mask"])
    old = (lp + synth.make_deltas(T, 17)).astype(np.float32)
    ref = oracle.grpo_step(b, h, W, y, old.astype(np.float64))
    step = ag.Step(T, len(b["task_id"]), b["n_groups"], b["n_tasks"], d, V)
    step(batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
    torch.cuda.synchronize()
    assert adv_close(step.adv_tok.cpu().numpy(), ref["adv_tok"]), kind
    N = int((b["loss_mask"] != 0).sum())
    assert abs(step.loss.item() - ref["loss"]) <= 1e-3 * max(abs(ref["loss"]), 1.0 / N) + 1e-9, kind
    e1 = max_abs_rel(step.grad_hidden.float().cpu().numpy(), ref["grad_hidden"])
    e2 = max_abs_rel(step.grad_W.cpu().numpy(), ref["grad_W"])
    assert e1 <= 2e-2 and e2 <= 2e-2, (kind, e1, e2)


def main():
    for i, kind in enumerate(("short", "long", "shuffled", "bigtraj", "huge", "contig")):
        b = layout(kind, 2510_04206 + 500 + i)
        check_adv(kind, b)
        if kind != "huge":
            check_idx(kind, b, oracle.task_adv_norm(b))
        if kind in ("short", "shuffled"):
            check_step(kind, b)
        if kind in ("short", "bigtraj", "contig"):  # T % 512 != 0; misaligned pointers
            ref = oracle.task_adv_norm(b)
            adv, _, nm, _, _ = run_adv(b, mask_offset=3, out_offset=1)
            assert nm == ref["n_mask"] and adv_close(adv, ref["adv_tok"]), kind + " misaligned"
    # a BASELINE config's real batch structure (glm9b: 131,072 tokens, 640 trajectories, ~40%
    # assistant tokens): the small driver in the default build, the large one under advlarge
    b = synth.make_structure(synth.CONFIGS["glm9b"])
    b = {k: v for k, v in b.items() if k != "token_index"}
    check_adv("glm9b", b)
    check_idx("glm9b", b, oracle.task_adv_norm(b))
    print("adv layouts ok", ag.LIB_PATH)


if __name__ == "__main__":
    main()
