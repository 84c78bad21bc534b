"""Two ranks on two GPUs over NCCL (skipped unless two devices are visible; the driver's
multi-GPU runs and any 2-GPU lease execute it): the real communicator at world 2 -- the split
cooperative adv-norm launches around the NCCL all-reduce of the per-task (N, S, Q), the loss
all-reduce, the grad_W all-reduce (mode 1), ncclReduceScatter (mode 2) and the reduce-scatter
fused into the grad_W GEMM epilogue as NVLink peer stores across devices (mode 2 + peer window)
-- against the fp64 oracle on the GLOBAL batch (reading R6)."""
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.gpu2]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out_dir, cfg_name, mode, p2p):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    import paper_2510_04206_b200 as ag
    from gpu_util import batch_dev, bf16_dev, f64

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
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
    comm = ag.Comm.from_process_group()
    if p2p:
        comm.enable_peer_window(cfg.V * cfg.d * 4)

    def td(x, dt):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev, dt)

    bd = {k: (td(v, {"traj_offsets": torch.int64, "rewards": torch.float32,
                     "loss_mask": torch.uint8}.get(k, torch.int32))
              if isinstance(v, np.ndarray) else v) for k, v in lb.items() if k != "token_index"}
    step = ag.Step(lb["T"], len(lb["task_id"]), lb["n_groups"], lb["n_tasks"], cfg.d, cfg.V,
                   device=dev, comm=comm, grad_W_mode=mode,
                   max_rows=int(lb["loss_mask"].astype(bool).sum()))
    hid = torch.from_numpy(np.ascontiguousarray(hb[tok]).view(np.int16)).to(dev).view(torch.bfloat16)
    Wd = torch.from_numpy(np.ascontiguousarray(Wb).view(np.int16)).to(dev).view(torch.bfloat16)
    inputs = (bd, hid, Wd, td(y[tok], torch.int32), td(old[tok], torch.float32))
    step(*inputs)
    torch.cuda.synchronize()
    if p2p:  # a second epoch (the consumed-slot guard across devices): bitwise the same shard
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


@pytest.mark.parametrize("cfg_name,mode,p2p", [("ragged", 1, False), ("ragged", 2, False),
                                               ("ragged", 2, True), ("parity7b", 2, True)])
def test_two_gpus_nccl_match_global_oracle(tmp_path, cfg_name, mode, p2p):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
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
        assert adv_close(r[k]["adv"], ref["adv_tok"][r[k]["tok"]])
    if mode == 1:
        np.testing.assert_array_equal(r[0]["gw"], r[1]["gw"])
    gh = np.zeros_like(ref["grad_hidden"])
    for k in range(2):
        gh[r[k]["tok"]] = r[k]["gh"]
    assert max_abs_rel(gh, ref["grad_hidden"]) <= 2e-2
