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
