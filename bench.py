#!/usr/bin/env python
"""Benchmark: fused task-normalized GRPO LM-head loss fwd+bwd (agentrl_grpo_step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config glm9b] [--impl reference]

One "step" = one agentrl_grpo_step over one synthetic batch (all section-8(a) rows:
task advantage normalization, LM-head forward with the softmax epilogue, loss, grad_W,
grad_hidden).  Rank 0 prints ONE JSON line.  For N > 1 launch with torchrun; each rank
holds whole groups (LPT-balanced on masked tokens) of the same global batch (strong
scaling) and the library all-reduces task statistics, the loss and grad_W over NCCL.

value   = global packed tokens T / step time (max over ranks), inputs resident in HBM
e2e     = same metric through the C ABI with the step's inputs copied from pinned host
          memory each step and the loss/stats read back (copies inside the timed region)
roofline: the dominant kernel's algorithmic FLOPs per launch / its CUDA-event duration
          (recorded by the library on the launching stream during the timed region)
cpu_baseline: the fp64 CPU oracle (test infrastructure) timed on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "fused GRPO loss fwd+bwd tokens/s"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="glm9b", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--all-masked", action="store_true",
                    help="every token a loss token (SURVEY 8(d): the compute upper bound)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=j.get("hbm_gbs", 6650.0), bf16=j.get("bf16_tflops", 1590.0),
                    bf16_sus=j.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for k, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- inputs
def build_inputs(cfg, rank, world, all_masked=False):
    """Global batch structure; this rank's shard (whole groups, LPT on masked tokens)."""
    b = synth.make_structure(cfg)
    if all_masked:
        b["loss_mask"] = np.ones_like(b["loss_mask"])
    if world > 1:
        ng = np.zeros(len(b["task_id"]), np.int64)
        off = b["traj_offsets"]
        cs = np.concatenate([[0], np.cumsum(b["loss_mask"].astype(np.int64))])
        ng = cs[off[1:]] - cs[off[:-1]]  # masked tokens per trajectory (input bookkeeping)
        gtok = np.bincount(b["group_id"], weights=ng, minlength=b["n_groups"])
        rog = synth.shard_groups_lpt(gtok, world)
        lb = synth.shard_batch(b, rog, rank)
    else:
        lb = dict(b)
    return b, lb


def main():
    args = parse()
    cfg = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    return run_native(args, cfg, world, rank, local_rank)


def run_native(args, cfg, world, rank, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2510_04206_b200 as ag

    # AGENTRL_BENCH_SHARED_GPU=1 (flow test only, tests/test_gpu_bench_multirank.py): every
    # rank on cuda:0 over gloo with the library's callback communicator -- NCCL cannot place
    # two ranks on one device.  The numbers of such a run are not measurements.
    shared = os.environ.get("AGENTRL_BENCH_SHARED_GPU") == "1" and world > 1
    if shared:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    comm = None
    if world > 1 and shared:
        dist.init_process_group("gloo")
        comm = ag.CallbackComm(world, rank, ag.gloo_allreduce_fn(),
                               rs_fn=ag.gloo_reduce_scatter_fn(world, rank))
    elif world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = ag.Comm.from_process_group()

    def max_over_ranks(x):
        if world == 1:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    gb, lb = build_inputs(cfg, rank, world, args.all_masked)
    # analysis mode: one GPU runs rank 0's LPT shard of an n-GPU run, no communication (the
    # per-rank compute of the scaling configuration); the line then describes that shard
    shard_of = int(os.environ.get("AGENTRL_BENCH_SHARD", "0"))
    if world == 1 and shard_of > 1:
        _, lb = build_inputs(cfg, 0, shard_of, args.all_masked)
        lb = {k: v for k, v in lb.items() if k != "token_index"}
        gb = lb
    T = int(lb["T"])
    d, V = cfg.d, cfg.V
    n_traj = len(lb["task_id"])
    # ---- device-resident weights (generated on device, seeded: not a step input)
    g = torch.Generator(device=dev)
    g.manual_seed(synth.SEED_BASE + 77)
    W = (torch.randn(V, d, generator=g, device=dev) * (3.0 / math.sqrt(d))).to(torch.bfloat16)
    # ---- this rank's step inputs on host (pinned), seeded per rank
    rng = np.random.default_rng(synth.SEED_BASE + 1000 * (rank + 1) + cfg.index)
    hid = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
    gh = torch.Generator(device=dev)
    gh.manual_seed(synth.SEED_BASE + 4242 + rank)
    hid.copy_(torch.randn(T, d, generator=gh, device=dev).to(torch.bfloat16))
    target = torch.from_numpy(rng.integers(0, V, size=T).astype(np.int32)).to(dev)
    # planted 5% of masked rows: h = a W_y / |W_y|^2 + 0.5 noise (input generation)
    mrows = np.nonzero(lb["loss_mask"])[0]
    pr = torch.from_numpy(rng.choice(mrows, size=int(0.05 * len(mrows)), replace=False)).to(dev)
    wy = W[target[pr].long()].float()
    hid[pr] = (24.0 * wy / (wy * wy).sum(1, keepdim=True) + 0.5 * hid[pr].float()).to(torch.bfloat16)
    bd = {k: (torch.from_numpy(np.ascontiguousarray(v)).to(dev) if isinstance(v, np.ndarray) else v)
          for k, v in lb.items() if k != "token_index"}
    bd["traj_offsets"] = bd["traj_offsets"].to(torch.int64)
    for k in ("task_id", "group_id"):
        bd[k] = bd[k].to(torch.int32)
    bd["rewards"] = bd["rewards"].to(torch.float32)
    bd["loss_mask"] = bd["loss_mask"].to(torch.uint8)
    # C3 as the FSDP-style reduce-scatter of grad_W rows (the paper's trainer shards the head,
    # P:1357) when V divides evenly, else the all-reduce of a replicated head
    gw_mode = (2 if V % world == 0 else 1) if comm is not None else 0
    # C3 fused into the grad_W GEMM epilogue over peer memory (CUDA IPC windows; include/
    # agentrl.h agentrl_comm_enable_peer_window), unless AGENTRL_C3_P2P=0 or the mapping fails
    c3 = {0: "none", 1: "all-reduce (collective)", 2: "reduce-scatter (collective)"}[gw_mode]
    # the host built the mask, so it knows this rank's masked-token count: the workspace's
    # T_eff x V intermediate is sized by it (max_rows), not by T
    T_eff_local = int(lb["loss_mask"].astype(bool).sum())
    step = ag.Step(T, n_traj, lb["n_groups"], lb["n_tasks"], d, V, device=dev, comm=comm,
                   grad_W_mode=gw_mode, max_rows=T_eff_local)
    # behaviour log-probs: one untimed forward (old = 0), then old = logp + delta
    old = torch.zeros(T, dtype=torch.float32, device=dev)
    step(bd, hid, W, target, old)
    torch.cuda.synchronize()
    delta = torch.from_numpy(synth.make_deltas(T, synth.SEED_BASE + 9 + rank).astype(np.float32))
    old = (step.logp + delta.to(dev)) * bd["loss_mask"].float()
    c3_check = None
    if gw_mode == 2 and os.environ.get("AGENTRL_C3_P2P", "1") != "0":
        # C3 fused into the grad_W GEMM epilogue over peer memory (CUDA IPC windows; include/
        # agentrl.h agentrl_comm_enable_peer_window).  Validated on first use: one step with the
        # collective reduce-scatter, one with the fused path; the rank's grad_W shard must agree
        # on every rank (max over ranks), else the collective path is kept.
        rows = V // world
        step(bd, hid, W, target, old)
        torch.cuda.synchronize()
        ref_shard = step.grad_W[rank * rows:(rank + 1) * rows].clone()
        err = float("inf")
        try:
            comm.enable_peer_window(V * d * 4)
            step(bd, hid, W, target, old)
            torch.cuda.synchronize()
            got = step.grad_W[rank * rows:(rank + 1) * rows]
            err = float(((got - ref_shard).abs().max() / ref_shard.abs().max().clamp_min(1e-30))
                        .item())
            if int(step.status.item()) & ag.ST_COMM_TIMEOUT:
                err = float("inf")
        except RuntimeError as e:
            print(f"peer window unavailable ({e})", file=sys.stderr)
        err = max_over_ranks(err)
        c3_check = {"max_rel_diff_vs_collective": err, "ok": err <= 1e-5}
        if err <= 1e-5:
            c3 = "reduce-scatter fused into the grad_W GEMM epilogue (P2P stores)"
        else:
            print(f"fused C3 self-check failed (max rel diff {err}); collective reduce-scatter",
                  file=sys.stderr)
            dist.barrier()
            comm.enable_peer_window(0)
        step.status.zero_()
    T_eff_global = int(gb["loss_mask"].astype(bool).sum())
    T_global = int(gb["T"])

    def barrier():
        if world > 1:
            dist.barrier()

    def one_step():
        step(bd, hid, W, target, old)

    # part 1 alone, timed before the power-heavy GEMM steps (the GPU is not yet clocked down
    # by the power cap; a latency-bound kernel scales with the SM clock)
    adv = adv_norm_timing(ag, bd, lb, dev, peaks()["hbm"]) if rank == 0 else None
    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        one_step()
    torch.cuda.synchronize()
    launches_per_step = ag.last_launch_count()

    # ---- timed region (device time, CUDA events, max over ranks)
    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.3)
    ag.profile_start(64 * max(args.steps, 1))
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        one_step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    prof = ag.profile_stop()
    clocks = clk.stop()
    status = int(step.status.item())
    ms = max_over_ranks(ms)
    value = T_global / (ms / 1e3)
    imbalance = None
    if world > 1:  # per-rank load: max / mean of the masked rows (LPT group sharding)
        mx = max_over_ranks(float(T_eff_local))
        tot = torch.tensor([float(T_eff_local)], dtype=torch.float64,
                           device="cpu" if shared else dev)
        dist.all_reduce(tot)
        imbalance = mx / (float(tot.item()) / world)

    # ---- e2e: host buffers through the C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hid_h = hid.cpu().pin_memory()
        tgt_h = target.cpu().pin_memory()
        old_h = old.cpu().pin_memory()
        meta_h = {k: bd[k].cpu().pin_memory() for k in
                  ("traj_offsets", "task_id", "group_id", "rewards", "loss_mask")}
        loss_h = torch.empty(6, dtype=torch.float64).pin_memory()
        h2d = sum(x.numel() * x.element_size() for x in [hid_h, tgt_h, old_h, *meta_h.values()])
        d2h = loss_h.numel() * loss_h.element_size()
        stats_dev = torch.empty(6, dtype=torch.float64, device=dev)
        # double-buffered device inputs: step k+1's host->device copy runs on a copy stream
        # while step k computes (every copy is still inside the timed region)
        sets = [dict(hid=hid, target=target, old=old, bd=bd),
                dict(hid=torch.empty_like(hid), target=torch.empty_like(target),
                     old=torch.empty_like(old),
                     bd={k: (v.clone() if torch.is_tensor(v) else v) for k, v in bd.items()})]
        main_s = torch.cuda.current_stream()
        copy_s = torch.cuda.Stream(device=dev)

        def copy_inputs(S):
            S["hid"].copy_(hid_h, non_blocking=True)
            S["target"].copy_(tgt_h, non_blocking=True)
            S["old"].copy_(old_h, non_blocking=True)
            for k, v in meta_h.items():
                S["bd"][k].copy_(v, non_blocking=True)

        def run_e2e(n):
            copy_s.wait_stream(main_s)
            done, ready = [None, None], [None, None]
            with torch.cuda.stream(copy_s):
                copy_inputs(sets[0])
                ready[0] = copy_s.record_event()
            for k in range(n):
                i, j = k % 2, 1 - k % 2
                if k + 1 < n:
                    with torch.cuda.stream(copy_s):
                        if done[j] is not None:
                            copy_s.wait_event(done[j])
                        copy_inputs(sets[j])
                        ready[j] = copy_s.record_event()
                main_s.wait_event(ready[i])
                S = sets[i]
                step(S["bd"], S["hid"], W, S["target"], S["old"])
                stats_dev[0:1].copy_(step.loss)
                stats_dev[1:6].copy_(step.loss_stats)
                loss_h.copy_(stats_dev, non_blocking=True)
                done[i] = main_s.record_event()

        run_e2e(2)
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        run_e2e(args.steps)
        f1.record()
        torch.cuda.synchronize()
        barrier()
        ms_e2e = f0.elapsed_time(f1) / args.steps
        ms_e2e = max_over_ranks(ms_e2e)
        e2e = {"value": T_global / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ms_e2e,
               "pipelining": "inputs double-buffered; step k+1's pinned H2D copy overlaps "
                             "step k on a copy stream; loss/stats D2H after each step"}

    # ---- roofline of the dominant kernel (events recorded by the library, same stream)
    pk = peaks()
    gemm_names = {"gemm_fwd", "gemm_grad_W", "gemm_grad_hidden"}
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    kernel_ms = {k: (v[0] / max(v[1], 1), v[1]) for k, v in prof.items() if v[1] > 0}
    if dom_name in gemm_names and dom_n > 0:
        # each GEMM does 2 T_eff V d per step, over dom_n / steps launches (row-chunked forward)
        flop = 2.0 * T_eff_local * V * d * args.steps / dom_n
        achieved = flop / (dom_ms / dom_n / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": dom_name, "achieved": achieved,
                "peak": pk["bf16_sus"], "unit": "TFLOP/s", "frac": achieved / pk["bf16_sus"],
                "peak_kind": f"{pk['src']} sustained bf16 (kernel timed inside a long step)",
                "frac_of_burst": achieved / pk["bf16"],
                "frac_of_datasheet": achieved / 2250.0,  # nominal dense bf16 per B200
                "flop_per_launch": flop, "traffic": traffic_from_profiles(args.config, dom_name)}
    else:
        roof = {"bound": "hbm", "kernel": dom_name, "achieved": None, "peak": pk["hbm"],
                "unit": "GB/s", "frac": None, "traffic": None}
    step_flop = 6.0 * T_eff_global * V * d
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": cfg.name, "T": T_global, "T_eff": T_eff_global, "d": d, "V": V,
                   "n_tasks": cfg.n_tasks, "groups": int(gb["n_groups"]),
                   "rollouts": cfg.rollouts, "parallelism": f"dp{world}",
                   "grad_W_collective": c3, "c3_self_check": c3_check,
                   "workspace_gb": round(step.ws.numel() / 1e9, 2),
                   **({"shard": f"rank 0 of {shard_of} (LPT), no communication"}
                      if world == 1 and shard_of > 1 else {}),
                   "mask": "all tokens (--all-masked)" if args.all_masked else "synthetic multi-turn (~40% assistant)",
                   "l2": "inputs larger than L2 (hidden %.2f GB, W %.2f GB, P~ %.1f GB)" % (
                       T * d * 2 / 1e9, V * d * 2 / 1e9, T_eff_local * V * 2 / 1e9)},
        "masked_tokens_per_s": T_eff_global / (ms / 1e3),
        "rank_imbalance_masked_rows": imbalance,
        "step_tflops_algorithmic": step_flop / (ms / 1e3) / 1e12,
        "clocks": clocks, "e2e": e2e,
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": roof, "adv_norm": adv, "kernel_ms": kernel_ms, "status": status,
        "loss": float(step.loss.item()), "clip_frac": float(step.loss_stats[0].item()),
    }
    if world > 1:
        dist.barrier()
    if rank == 0:
        if not args.no_cpu and world == 1:  # the oracle baseline: rank 0 at N=1 only
            result["cpu_baseline"] = cpu_baseline(cfg, gb, args.cpu_seconds)
        if shared:
            result["note"] = "AGENTRL_BENCH_SHARED_GPU flow test: all ranks on one GPU, not a measurement"
        print(json.dumps(result), flush=True)
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()


def _adv_time(ag, bd, lb, dev, iters, graph):
    """median event time (ms) of agentrl_task_adv_norm on its own stream, cold L2 (a 2 x L2
    buffer is written before every timed call); optionally replayed from a CUDA graph"""
    import torch
    T = int(lb["T"])
    n_traj = len(lb["task_id"])
    ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, lb["n_groups"],
                                                                    lb["n_tasks"]), dev)
    adv = torch.empty(T, dtype=torch.float32, device=dev)
    ts = torch.empty(lb["n_tasks"], 3, dtype=torch.float64, device=dev)
    nm = torch.empty(1, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    batch = ag.make_batch(bd)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(device=dev)
    times = []
    with torch.cuda.stream(s):
        for _ in range(3):
            if ag.agentrl_task_adv_norm(batch, 1e-6, adv, ts, nm, ws, None, st, stream=s) != 0:
                return None
        g = None
        if graph:
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                ag.agentrl_task_adv_norm(batch, 1e-6, adv, ts, nm, ws, None, st, stream=s)
        for i in range(iters):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if g is not None:
                g.replay()
            else:
                ag.agentrl_task_adv_norm(batch, 1e-6, adv, ts, nm, ws, None, st, stream=s)
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    times.sort()
    return times[len(times) // 2]


def adv_norm_timing(ag, bd, lb, dev, hbm_gbs, iters=20):
    """Part 1 alone (agentrl_task_adv_norm), single GPU, cold L2, at this rank's batch
    (launch-latency bound) and at the 2^27-token bandwidth point of the DESIGN.md sweep
    (synth.make_sweep_structure: ~400 tokens/trajectory, 5 tasks, G=8).  Algorithmic bytes:
    mask T B + adv_tok 4T B + 20 B per trajectory (offsets, ids, reward)."""
    import torch
    T = int(lb["T"])
    n_traj = len(lb["task_id"])
    ms = _adv_time(ag, bd, lb, dev, iters, False)
    if ms is None:
        return None
    try:
        gms = _adv_time(ag, bd, lb, dev, iters, True)
    except Exception:  # graph capture unavailable: report the direct number only
        gms = None
    by = 5 * T + 20 * n_traj
    out = {"latency_us": ms * 1e3, "graph_latency_us": None if gms is None else gms * 1e3,
           "alg_bytes": by, "GBps": by / (ms / 1e3) / 1e9,
           "frac_hbm": by / (ms / 1e3) / 1e9 / hbm_gbs, "cold_l2": True,
           "note": "launch-latency bound at this size (an empty cooperative launch is ~5 us, "
                   "a grid barrier ~1.5 us); bandwidth_point is the HBM-bound regime"}
    try:
        sb = synth.make_sweep_structure(1 << 27)
        sbd = {k: (torch.from_numpy(np.ascontiguousarray(v)).to(dev) if isinstance(v, np.ndarray)
                   else v) for k, v in sb.items()}
        sbd["traj_offsets"] = sbd["traj_offsets"].long()
        sbd["task_id"] = sbd["task_id"].int()
        sbd["group_id"] = sbd["group_id"].int()
        sms = _adv_time(ag, sbd, sb, dev, 10, False)
        try:
            sgms = _adv_time(ag, sbd, sb, dev, 10, True)
        except Exception:  # graph capture unavailable
            sgms = None
        sby = 5 * int(sb["T"]) + 20 * len(sb["task_id"])
        out["bandwidth_point"] = {"T": int(sb["T"]), "n_traj": len(sb["task_id"]),
                                  "latency_us": sms * 1e3, "alg_bytes": sby,
                                  "GBps": sby / (sms / 1e3) / 1e9,
                                  "frac_hbm": sby / (sms / 1e3) / 1e9 / hbm_gbs,
                                  "graph_latency_us": None if sgms is None else sgms * 1e3,
                                  "graph_frac_hbm": None if sgms is None else
                                  sby / sgms * 1e3 / 1e9 / hbm_gbs}
        del sbd
        torch.cuda.empty_cache()
    except Exception as e:  # noqa: BLE001 -- report, never fail the bench line
        out["bandwidth_point"] = {"error": str(e)[:200]}
    return out


def traffic_from_profiles(config, kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    e = j.get(config, {}).get(kernel)
    if isinstance(e, dict):  # per launch = per step / launches per step
        return e["bytes_per_step"] / max(e["launches_per_step"], 1)
    return e


# --------------------------------------------------------------------------- oracle timing
def cpu_baseline(cfg, gb, seconds=15.0, rows=None):
    """fp64 CPU oracle (as it stands) on a bounded sample: full adv-norm of the batch +
    the loss fwd+bwd of the first `rows` masked tokens at full V, d; extrapolated."""
    import oracle
    cores = oracle.num_threads()
    t0 = time.perf_counter()
    an = oracle.task_adv_norm(gb)
    t_adv = time.perf_counter() - t0
    d, V = cfg.d, cfg.V
    # per-token oracle cost ~ 3*V*d fp64 MACs; the oracle parallelises across tokens, so the
    # sample holds 4 tokens per host thread (~10 s at the paper's head sizes)
    if rows is None:
        rows = 4 * max(cores, 1)
    rng = np.random.default_rng(1)
    W = rng.standard_normal((V, d)) * (3.0 / math.sqrt(d))
    h = rng.standard_normal((rows, d))
    t1 = time.perf_counter()
    oracle.policy_loss_fwd_bwd(h, W, rng.integers(0, V, size=rows).astype(np.int32),
                               rng.standard_normal(rows), np.full(rows, -12.0),
                               np.ones(rows, np.uint8), rows)
    t_loss = time.perf_counter() - t1
    n_eff = int(an["n_mask"])
    t_step = t_adv + t_loss / rows * n_eff
    # the same oracle on ONE host thread: 2 tokens of the loss sample
    one = None
    try:
        oracle.set_num_threads(1)
        r1 = 2
        t2 = time.perf_counter()
        oracle.policy_loss_fwd_bwd(h[:r1], W, rng.integers(0, V, size=r1).astype(np.int32),
                                   rng.standard_normal(r1), np.full(r1, -12.0),
                                   np.ones(r1, np.uint8), r1)
        t_one = time.perf_counter() - t2
        one = {"value": int(gb["T"]) / (t_adv + t_one / r1 * n_eff), "cores": 1,
               "sample": f"loss fwd+bwd of {r1} masked tokens on 1 thread ({t_one:.2f} s), "
                         f"extrapolated like the multi-thread figure"}
    finally:
        oracle.set_num_threads(cores)
    cpu = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"value": int(gb["T"]) / t_step, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu, "host_cpus": os.cpu_count(),
            "sample": f"adv-norm on the full batch ({t_adv:.3f} s) + loss fwd+bwd of {rows} "
                      f"masked tokens at full V={V}, d={d} ({t_loss:.2f} s), extrapolated to "
                      f"{n_eff} masked tokens", "one_thread": one,
            "extrapolated": True, "sample_wall_s": t_adv + t_loss}


def run_reference(args, cfg, world, rank):
    """Reference arm = the fp64 CPU oracle as it stands, on this box's host cores."""
    if rank != 0:
        return 0
    gb = synth.make_structure(cfg)
    samples = []
    for i in range(max(args.warmup, 0) + args.steps):
        import oracle
        cb = cpu_baseline(cfg, gb, seconds=min(args.cpu_seconds, 10.0),
                          rows=2 * max(oracle.num_threads(), 1))
        if i >= args.warmup:
            samples.append(cb)
    v = statistics.median([s["value"] for s in samples])
    # ms_per_step is the time the oracle WOULD take for one whole step, extrapolated from the
    # bounded sample (cpu_baseline.sample); the arm itself ran sample_wall_s per step
    ms = int(gb["T"]) / v * 1e3
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference", "config": {"workload": cfg.name, "T": int(gb["T"]), "d": cfg.d,
                                           "V": cfg.V, "parallelism": "host cores"},
           "ms_per_step_extrapolated": True,
           "sample_wall_s_per_step": statistics.median([s["sample_wall_s"] for s in samples]),
           "cpu_baseline": dict(samples[-1], value=v),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
