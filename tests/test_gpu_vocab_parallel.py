"""Vocabulary-parallel head (grad_W_mode = 3) on one GPU: two ranks share
cuda:0 through gloo and the callback communicator (NCCL cannot place two ranks on one device;
the library's collective placement is the same).  Every rank holds the same token rows and
half of W_head's rows.  Checked against the fp64 oracle on the whole head:
  loss, logp, loss statistics     identical on both ranks and equal to the global oracle
  grad_hidden                     the full gradient on both ranks (summed inside the call)
  grad_W                          each rank's complete shard = the oracle's rows of that shard
Also: world size 1 gives the single-GPU (mode 0) result."""
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


def _inputs(cfg_name):
    import oracle
    import synth
    from gpu_util import f64
    cfg = synth.CONFIGS[cfg_name]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    lp = oracle.logprob(f64(hb), f64(Wb), y, b["loss_mask"])
    old = (lp + synth.make_deltas(cfg.T, 29)).astype(np.float32)
    adv = oracle.task_adv_norm(b)["adv_tok"].astype(np.float32)
    return cfg, b, hb, Wb, y, old, adv


def _run_vp(ag, comm, world, rank, cfg, b, hb, Wb, y, old, adv, mode=3):
    import torch
    from gpu_util import bf16_dev, t
    T, d, V = cfg.T, cfg.d, cfg.V
    Vs = V // world if mode == 3 else V
    Wsh = np.ascontiguousarray(Wb[rank * Vs:(rank + 1) * Vs]) if mode == 3 else Wb
    need = (ag.agentrl_policy_loss_workspace_size_vp(T, d, Vs, world) if mode == 3
            else ag.agentrl_policy_loss_workspace_size(T, d, V))
    ws = ag.alloc_workspace(need)
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    logp = torch.full((T,), float("nan"), device="cuda")
    gh = torch.full((T, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    gw = torch.full((Vs, d), float("nan"), device="cuda")
    stats = torch.zeros(5, dtype=torch.float64, device="cuda")
    nm = torch.tensor([int((b["loss_mask"] != 0).sum())], dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = ag.make_loss_args(T, bf16_dev(hb), bf16_dev(Wsh), t(y, torch.int32),
                             t(old, torch.float32), t(b["loss_mask"], torch.uint8),
                             adv_tok=t(adv, torch.float32), n_mask_global=nm, grad_W_mode=mode)
    rc = ag.agentrl_policy_loss_fwd_bwd(args, ag.make_loss_out(loss, gh, gw, logp, stats), ws,
                                        comm.handle if comm else None, st)
    assert rc == 0, ag.status_string(rc)
    torch.cuda.synchronize()
    return dict(loss=loss.item(), logp=logp.cpu().numpy(), gh=gh.float().cpu().numpy(),
                gw=gw.cpu().numpy(), stats=stats.cpu().numpy(), st=int(st.item()))


def _rank(rank, world, port, out_dir, cfg_name):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import paper_2510_04206_b200 as ag

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg, b, hb, Wb, y, old, adv = _inputs(cfg_name)
    comm = ag.CallbackComm(world, rank, ag.gloo_allreduce_fn())
    res = _run_vp(ag, comm, world, rank, cfg, b, hb, Wb, y, old, adv)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **res)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["tiny", "ragged"])
def test_vocab_parallel_two_ranks(tmp_path, cfg_name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import oracle
    from gpu_util import f64, max_abs_rel

    mp.spawn(_rank, args=(2, _port(), str(tmp_path), cfg_name), nprocs=2, join=True)
    cfg, b, hb, Wb, y, old, adv = _inputs(cfg_name)
    m = b["loss_mask"] != 0
    N = int(m.sum())
    ref = oracle.policy_loss_fwd_bwd(f64(hb), f64(Wb), y, adv.astype(np.float64),
                                     old.astype(np.float64), b["loss_mask"], N)
    r = [dict(np.load(tmp_path / f"r{k}.npz")) for k in range(2)]
    for k in range(2):
        assert int(r[k]["st"]) == 0
        assert abs(float(r[k]["loss"]) - ref["loss"]) <= 1e-3 * max(abs(ref["loss"]), 1.0 / N)
        assert np.abs(r[k]["logp"][m] - ref["logp"][m]).max() <= 1e-3
        assert max_abs_rel(r[k]["gh"], ref["grad_hidden"]) <= 2e-2
        sh = slice(k * cfg.V // 2, (k + 1) * cfg.V // 2)
        assert np.abs(r[k]["gw"] - ref["grad_W"][sh]).max() <= 2e-2 * np.abs(ref["grad_W"]).max()
    # replicated results: bitwise equal on both ranks
    for key in ("loss", "logp", "gh", "stats"):
        np.testing.assert_array_equal(r[0][key], r[1][key])


def test_vocab_parallel_world1_matches_mode0():
    """one rank holding the whole head: the same result as the single-GPU path (the row
    statistics then come from one slot; grad_hidden via the fp32 partial + scatter)"""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_04206_b200 as ag
    from gpu_util import max_abs_rel

    cfg, b, hb, Wb, y, old, adv = _inputs("ragged")
    comm = ag.CallbackComm(1, 0, lambda *a: None)
    vp = _run_vp(ag, comm, 1, 0, cfg, b, hb, Wb, y, old, adv, mode=3)
    base = _run_vp(ag, None, 1, 0, cfg, b, hb, Wb, y, old, adv, mode=0)
    comm.destroy()
    assert vp["st"] == 0 and base["st"] == 0
    assert abs(vp["loss"] - base["loss"]) <= 1e-6 * max(abs(base["loss"]), 1e-6)
    assert np.abs(vp["logp"] - base["logp"]).max() <= 1e-5
    assert max_abs_rel(vp["gh"], base["gh"]) <= 1e-2
    np.testing.assert_array_equal(vp["gw"], base["gw"])
