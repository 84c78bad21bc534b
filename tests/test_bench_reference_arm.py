"""bench.py's reference arm (the fp64 oracle on the host cores) keeps the driver's JSON
contract: one line with the metric, value, unit, impl, cpu_baseline and a zero-copy e2e; under
a multi-rank launch only rank 0 prints, the other ranks exit 0 without work.  CPU only (tiny)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = [sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "1",
        "--warmup", "0"]


def _run(extra_env, extra_args=()):
    env = dict(os.environ, **extra_env)
    return subprocess.run(ARGS + list(extra_args), cwd=ROOT, env=env, capture_output=True,
                          text=True, timeout=300)


def test_reference_line_contract():
    r = _run({"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"}, ["--gpus", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["metric"] == "fused GRPO loss fwd+bwd tokens/s" and d["unit"] == "tokens/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == "tiny"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert cb["one_thread"]["cores"] == 1 and 0 < cb["one_thread"]["value"]
    assert d["ms_per_step_extrapolated"] is True and d["sample_wall_s_per_step"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_other_ranks_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, ["--gpus", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]
