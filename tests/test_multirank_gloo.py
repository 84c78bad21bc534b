"""World-size-2 CPU (gloo) test of the multi-GPU protocol the library implements:
whole groups per rank (LPT partition), C1 = all-reduce of per-task (N_i, S_i, Q_i),
C2 = all-reduce of the loss, C3 = all-reduce of grad_W.  Each rank runs the oracle on
its shard with the exchanged global statistics; the result must equal the oracle on the
global batch (R6: "current batch" = global batch)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["ragged"]
    gb = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=gb["loss_mask"])
    h = synth.bf16_bits_to_f32(hb).astype(np.float64)
    W = synth.bf16_bits_to_f32(Wb).astype(np.float64)
    old = synth.make_old_logp_free(cfg.T, 3).astype(np.float64)
    # partition whole groups by masked tokens
    off = gb["traj_offsets"]
    cs = np.concatenate([[0], np.cumsum(gb["loss_mask"].astype(np.int64))])
    ng = cs[off[1:]] - cs[off[:-1]]
    rog = synth.shard_groups_lpt(np.bincount(gb["group_id"], weights=ng,
                                             minlength=gb["n_groups"]), world)
    lb = synth.shard_batch(gb, rog, rank)
    tok = lb["token_index"]
    loc = oracle.task_adv_norm(lb)
    # C1: per-task raw moments
    nt = lb["n_tasks"]
    stats = torch.zeros(3 * nt, dtype=torch.float64)
    for i in range(nt):
        sel = lb["task_id"] == i
        n = loc["n_g"][sel].astype(np.float64)
        a = loc["adv_hat"][sel]
        stats[3 * i:3 * i + 3] = torch.tensor([n.sum(), (n * a).sum(), (n * a * a).sum()])
    dist.all_reduce(stats)
    s = stats.numpy().reshape(nt, 3)
    mu = s[:, 1] / np.maximum(s[:, 0], 1)
    sd = np.sqrt(np.maximum(s[:, 2] / np.maximum(s[:, 0], 1) - mu * mu, 0))
    N = int(s[:, 0].sum())
    adv = np.zeros(lb["T"])
    oracle.lib().oracle_apply(lb["T"], len(lb["task_id"]), oracle._p(lb["traj_offsets"]),
                              oracle._p(np.ascontiguousarray(lb["task_id"], np.int32)),
                              oracle._p(lb["loss_mask"]), oracle._p(loc["adv_hat"]),
                              oracle._p(np.ascontiguousarray(np.stack([s[:, 0], mu, sd], 1)
                                                             .reshape(-1))),
                              1e-6, oracle._p(np.zeros(len(lb["task_id"]))), oracle._p(adv),
                              None, oracle._p(np.zeros(1, np.int64)))
    out = oracle.policy_loss_fwd_bwd(h[tok], W, y[tok], adv, old[tok], lb["loss_mask"], N)
    # C2, C3
    loss = torch.tensor([out["loss"]], dtype=torch.float64)
    dist.all_reduce(loss)
    gw_local = torch.from_numpy(out["grad_W"])
    # C3 as a reduce-scatter (grad_W_mode 2, FSDP-style row shard): block `rank` of the rows
    shard = torch.empty(gw_local.shape[0] // world, gw_local.shape[1], dtype=gw_local.dtype)
    dist.reduce_scatter_tensor(shard, gw_local.clone())
    gw = gw_local.clone()
    dist.all_reduce(gw)
    np.save(os.path.join(out_dir, f"shard{rank}.npy"), shard.numpy())
    if rank == 0:
        ref = oracle.grpo_step(gb, h, W, y, old)
        np.save(os.path.join(out_dir, "gw_ref.npy"), ref["grad_W"])
        np.save(os.path.join(out_dir, "res.npy"),
                np.asarray([loss.item(), ref["loss"],
                            float(np.abs(gw.numpy() - ref["grad_W"]).max()),
                            float(np.abs(ref["grad_W"]).max()), N, int(gb["loss_mask"].sum())]))
        # per-token advantages and grad_hidden rows of rank 0's tokens
        np.save(os.path.join(out_dir, "adv.npy"), np.stack([adv, ref["adv_tok"][tok]]))
        np.save(os.path.join(out_dir, "gh.npy"),
                np.stack([out["grad_hidden"], ref["grad_hidden"][tok]]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_protocol_matches_global(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r = np.load(tmp_path / "res.npy")
    loss, ref_loss, gw_err, gw_max, N, N_ref = r
    assert N == N_ref
    assert abs(loss - ref_loss) <= 1e-12 * max(abs(ref_loss), 1.0)
    assert gw_err <= 1e-12 * max(gw_max, 1.0)
    adv = np.load(tmp_path / "adv.npy")
    np.testing.assert_allclose(adv[0], adv[1], atol=1e-12)
    gh = np.load(tmp_path / "gh.npy")
    np.testing.assert_allclose(gh[0], gh[1], atol=1e-14)
    # reduce-scatter shards tile the global grad_W
    shards = np.concatenate([np.load(tmp_path / f"shard{k}.npy") for k in range(2)])
    ref = np.load(tmp_path / "gw_ref.npy")
    assert np.abs(shards - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1.0)
