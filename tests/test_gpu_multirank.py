"""Two ranks on one GPU: the sharded data path of the library (split cooperative adv-norm
launches around the statistics all-reduce, the loss all-reduce, the grad_W all-reduce on the
side stream) against the fp64 oracle on the GLOBAL batch (R6).  NCCL cannot place two ranks
on one device, so the ranks use the callback communicator with a gloo all-reduce; the
library-side collective placement is the same as with NCCL."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out_dir, cfg_name, mode=1, p2p=False):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    import paper_2510_04206_b200 as ag
    from gpu_util import batch_dev, bf16_dev, f64, t

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = synth.CONFIGS[cfg_name]
    gb = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=gb["loss_mask"])
    h, W = f64(hb), f64(Wb)
    lp = oracle.logprob(h, W, y, gb["loss_mask"])
    old = (lp + synth.make_deltas(cfg.T, 23)).astype(np.float32)
    off = gb["traj_offsets"]
    cs = np.concatenate([[0], np.cumsum(gb["loss_mask"].astype(np.int64))])
    ng = cs[off[1:]] - cs[off[:-1]]
    rog = synth.shard_groups_lpt(np.bincount(gb["group_id"], weights=ng,
                                             minlength=gb["n_groups"]), world)
    lb = synth.shard_batch(gb, rog, rank)
    tok = lb["token_index"]
    def poison(*a):  # the fused path must not fall back to the collective reduce-scatter
        raise RuntimeError("collective reduce-scatter called on the p2p path")
    rs = (poison if p2p else ag.gloo_reduce_scatter_fn(world, rank)) if mode == 2 else None
    comm = ag.CallbackComm(world, rank, ag.gloo_allreduce_fn(), rs_fn=rs)
    if p2p:  # grad_W reduce-scatter fused into the GEMM epilogue over IPC peer memory
        comm.enable_peer_window(cfg.V * cfg.d * 4)
    step = ag.Step(lb["T"], len(lb["task_id"]), lb["n_groups"], lb["n_tasks"], cfg.d, cfg.V,
                   comm=comm, grad_W_mode=mode)
    inputs = (batch_dev(lb), bf16_dev(hb[tok]), bf16_dev(Wb), t(y[tok], torch.int32),
              t(old[tok], torch.float32))
    step(*inputs)
    torch.cuda.synchronize()
    if p2p:  # a second epoch (exercises the consumed-slot guard): bitwise the same shard
        sh = slice(rank * cfg.V // world, (rank + 1) * cfg.V // world)
        first = step.grad_W[sh].clone()
        step(*inputs)
        torch.cuda.synchronize()
        assert torch.equal(first, step.grad_W[sh])
    res = dict(loss=step.loss.item(), adv=step.adv_tok.cpu().numpy(),
               gh=step.grad_hidden.float().cpu().numpy(), gw=step.grad_W.cpu().numpy(),
               ts=step.task_stats.cpu().numpy(), st=int(step.status.item()), tok=tok)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **res)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def test_nccl_world1_matches_no_comm():
    """The real NCCL communicator (dlopen'd libnccl, unique id, init, all-reduces incl. the
    grad_W one on the side stream) at world size 1 gives bitwise the single-GPU result."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import synth
    import paper_2510_04206_b200 as ag
    from gpu_util import batch_dev, bf16_dev, t

    cfg = synth.CONFIGS["ragged"]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    old = synth.make_old_logp_free(cfg.T, 5)
    args = (batch_dev(b), bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32))
    s0 = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)
    s0(*args)
    comm = ag.Comm(1, 0, ag.Comm.unique_id())
    s1 = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V, comm=comm)
    s1(*args)
    # grad_W_mode 2: ncclReduceScatter in place (world 1: the whole buffer is rank 0's shard)
    s2 = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V, comm=comm,
                 grad_W_mode=2)
    s2(*args)
    torch.cuda.synchronize()
    for s in (s1, s2):
        for a, c in ((s0.loss, s.loss), (s0.adv_tok, s.adv_tok), (s0.grad_W, s.grad_W),
                     (s0.grad_hidden, s.grad_hidden), (s0.task_stats, s.task_stats)):
            assert torch.equal(a, c)
    comm.destroy()


@pytest.mark.parametrize("cfg_name,mode,p2p", [("tiny", 1, False), ("ragged", 1, False),
                                               ("ragged", 2, False), ("ragged", 2, True),
                                               ("tiny", 2, True)])
def test_two_ranks_one_gpu_match_global_oracle(tmp_path, cfg_name, mode, p2p):
    """mode 1: grad_W all-reduced (replicated head); mode 2: reduce-scattered (FSDP-style row
    shard): each rank's rows [r V/2, (r+1) V/2) hold the global sum.  p2p: the
    reduce-scatter fused into the grad_W GEMM epilogue over CUDA-IPC peer memory (the two
    processes map each other's windows on the one device)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import oracle
    import synth
    from gpu_util import adv_close, f64, max_abs_rel

    mp.spawn(_rank, args=(2, _port(), str(tmp_path), cfg_name, mode, p2p), nprocs=2, join=True)
    cfg = synth.CONFIGS[cfg_name]
    gb = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=gb["loss_mask"])
    h, W = f64(hb), f64(Wb)
    lp = oracle.logprob(h, W, y, gb["loss_mask"])
    old = (lp + synth.make_deltas(cfg.T, 23)).astype(np.float32)
    ref = oracle.grpo_step(gb, h, W, y, old.astype(np.float64))
    r = [dict(np.load(tmp_path / f"r{k}.npz")) for k in range(2)]
    N = int((gb["loss_mask"] != 0).sum())
    for k in range(2):
        assert r[k]["st"] & ~16 == 0
        # global (all-reduced) results are identical on both ranks
        assert abs(r[k]["loss"] - ref["loss"]) <= 1e-3 * max(abs(ref["loss"]), 1.0 / N) + 1e-9
        if mode == 1:
            assert max_abs_rel(r[k]["gw"], ref["grad_W"]) <= 2e-2
        else:
            sh = slice(k * cfg.V // 2, (k + 1) * cfg.V // 2)
            gmax = np.abs(ref["grad_W"]).max()
            assert np.abs(r[k]["gw"][sh] - ref["grad_W"][sh]).max() <= 2e-2 * gmax
        np.testing.assert_array_equal(r[k]["ts"][:, 0], ref["task_stats"][:, 0])
        np.testing.assert_allclose(r[k]["ts"][:, 1:], ref["task_stats"][:, 1:], rtol=1e-9,
                                   atol=1e-12)
        # rank-local rows
        tok = r[k]["tok"]
        assert adv_close(r[k]["adv"], ref["adv_tok"][tok])
    if mode == 1:
        np.testing.assert_array_equal(r[0]["gw"], r[1]["gw"])
    gh = np.zeros_like(ref["grad_hidden"])
    for k in range(2):
        gh[r[k]["tok"]] = r[k]["gh"]
    assert max_abs_rel(gh, ref["grad_hidden"]) <= 2e-2


def test_nccl_world1_large_driver_matches_no_comm():
    """The large adv-norm driver (more than 2,048 trajectories: popcount launch, cooperative
    statistics, apply launch) with a real NCCL communicator at world size 1 -- the all-reduce of
    (N, S, Q, G) between the statistics and the apply launches -- gives bitwise the result of
    the call without a communicator, and both match the fp64 oracle."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import synth
    import paper_2510_04206_b200 as ag
    from gpu_util import adv_close, batch_dev

    b = synth.make_sweep_structure(1 << 20)  # 2,621 trajectories: the large driver
    assert len(b["task_id"]) > 2048
    T, n_traj = int(b["T"]), len(b["task_id"])
    bd = batch_dev(b)

    def run(comm):
        ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                        b["n_tasks"]))
        adv = torch.full((T,), float("nan"), dtype=torch.float32, device="cuda")
        ts = torch.zeros(b["n_tasks"], 3, dtype=torch.float64, device="cuda")
        nm = torch.zeros(1, dtype=torch.int64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        rc = ag.agentrl_task_adv_norm(ag.make_batch(bd), 1e-6, adv, ts, nm, ws,
                                      comm.handle if comm else None, st)
        assert rc == 0, ag.status_string(rc)
        torch.cuda.synchronize()
        return adv.cpu().numpy(), ts.cpu().numpy(), int(nm.item()), int(st.item())

    a0, t0, n0, s0 = run(None)
    comm = ag.Comm(1, 0, ag.Comm.unique_id())
    a1, t1, n1, s1 = run(comm)
    comm.destroy()
    np.testing.assert_array_equal(a0, a1)
    np.testing.assert_array_equal(t0, t1)
    assert n0 == n1 and s0 == s1
    ref = oracle.task_adv_norm(b)
    assert n0 == ref["n_mask"]
    np.testing.assert_array_equal(t0[:, 0], ref["task_stats"][:, 0])
    np.testing.assert_allclose(t0[:, 1:], ref["task_stats"][:, 1:], rtol=1e-9, atol=1e-12)
    assert adv_close(a0, ref["adv_tok"])
