"""The fused step (agentrl_grpo_step, single GPU) captured in a CUDA graph.

DESIGN.md §1 states that every launch configuration is independent of the data, so a step can
be captured once and replayed.  Checked here:
  - a replay gives bitwise the outputs of a direct call on the same inputs;
  - after the inputs are rewritten in place (new rewards, so new advantages; new behaviour
    log-probs; new hidden states), a replay gives bitwise the outputs of a direct call on the
    new inputs: nothing data-dependent was frozen into the graph at capture time.
Results are deterministic run to run (fixed-order reductions, fixed per-tile K loops), which
is what makes the bitwise comparison meaningful."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402

from gpu_util import batch_dev, bf16_dev, t  # noqa: E402

OUTS = ("loss", "adv_tok", "task_stats", "logp", "grad_hidden", "grad_W", "loss_stats", "status")


@pytest.fixture(scope="module")
def ag():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_04206_b200 as m
    return m


def _snap(step):
    return {k: getattr(step, k).clone() for k in OUTS}


def _same(a, b):
    for k in OUTS:
        x, y = a[k], b[k]
        assert torch.equal(x.view(torch.int16) if x.dtype == torch.bfloat16 else x,
                           y.view(torch.int16) if y.dtype == torch.bfloat16 else y), k


@pytest.mark.parametrize("cfg_name", ["ragged", "qwen7b"])
def test_grpo_step_graph_replay(ag, cfg_name):
    cfg = synth.CONFIGS[cfg_name]
    b = synth.make_structure(cfg)
    hb, Wb, y = synth.make_head(cfg, mask=b["loss_mask"])
    rng = np.random.default_rng(11)
    old = np.full(cfg.T, -6.0, np.float32) + rng.normal(0, 0.5, cfg.T).astype(np.float32)
    bd = batch_dev(b)
    h, W, yt, ot = bf16_dev(hb), bf16_dev(Wb), t(y, torch.int32), t(old, torch.float32)
    step = ag.Step(cfg.T, len(b["task_id"]), b["n_groups"], b["n_tasks"], cfg.d, cfg.V)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(bd, h, W, yt, ot, stream=s)  # warm-up: side streams and attributes set up
        s.synchronize()
        direct = _snap(step)
        assert int(direct["status"].item()) == 0
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step(bd, h, W, yt, ot, stream=s)
        for k in ("loss", "grad_W", "grad_hidden", "adv_tok"):  # poison before the replay
            getattr(step, k).fill_(float("nan"))
        g.replay()
        s.synchronize()
        _same(_snap(step), direct)

        # new inputs written into the captured buffers
        rew = synth.make_structure(cfg)["rewards"][::-1].copy()
        bd["rewards"].copy_(t(rew, torch.float32))
        ot.add_(0.03)
        h.copy_(h.flip(0))
        g.replay()
        s.synchronize()
        replayed = _snap(step)
        step(bd, h, W, yt, ot, stream=s)
        s.synchronize()
        _same(replayed, _snap(step))
        assert not torch.equal(replayed["grad_W"], direct["grad_W"])


def test_large_adv_norm_graph_replay(ag):
    """Part 1 alone with the large driver (> 2,048 trajectories: popcount, cooperative
    statistics and the apply as a programmatic dependent launch) captured in a CUDA graph:
    replays are bitwise the direct call, also after the rewards are rewritten in place, and the
    direct call matches the oracle."""
    import oracle
    from gpu_util import adv_close
    b = synth.make_sweep_structure(1 << 20)
    assert len(b["task_id"]) > 2048
    bd = batch_dev(b)
    T, n_traj = int(b["T"]), len(b["task_id"])
    ws = ag.alloc_workspace(ag.agentrl_task_adv_norm_workspace_size(T, n_traj, b["n_groups"],
                                                                    b["n_tasks"]))
    outs = dict(adv=torch.empty(T, dtype=torch.float32, device="cuda"),
                ts=torch.empty(b["n_tasks"], 3, dtype=torch.float64, device="cuda"),
                nm=torch.empty(1, dtype=torch.int64, device="cuda"),
                st=torch.zeros(1, dtype=torch.int32, device="cuda"))
    batch = ag.make_batch(bd)

    def call(s):
        rc = ag.agentrl_task_adv_norm(batch, 1e-6, outs["adv"], outs["ts"], outs["nm"], ws, None,
                                      outs["st"], stream=s)
        assert rc == 0

    def snap():
        return {k: v.clone() for k, v in outs.items()}

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call(s)
        s.synchronize()
        direct = snap()
        ref = oracle.task_adv_norm(b)
        assert int(direct["nm"].item()) == ref["n_mask"]
        assert adv_close(direct["adv"].cpu().numpy(), ref["adv_tok"])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call(s)
        for v in outs.values():
            v.zero_()
        g.replay()
        s.synchronize()
        for k in outs:
            assert torch.equal(outs[k], direct[k]), k
        # new rewards in place: the replay follows the data
        rng = np.random.default_rng(5)
        bd["rewards"].copy_(torch.from_numpy(
            rng.choice(np.asarray([1.0, 0.0, -0.2], np.float32), n_traj)).cuda())
        call(s)
        s.synchronize()
        direct2 = snap()
        assert not torch.equal(direct2["adv"], direct["adv"])
        g.replay()
        s.synchronize()
        for k in outs:
            assert torch.equal(outs[k], direct2[k]), k
