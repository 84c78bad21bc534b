"""The N>1 bench flow (torchrun launch, LPT group sharding, per-rank steps with the sharded
collectives, barrier + max-over-ranks device timing, e2e, rank 0 printing one JSON line) on
one GPU: two ranks share cuda:0 through gloo and the library's callback communicator
(AGENTRL_BENCH_SHARED_GPU=1), since NCCL cannot place two ranks on one device."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_shared_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "qwen7b", "--steps", "2",
           "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, env={**os.environ, "AGENTRL_BENCH_SHARED_GPU": "1"},
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["status"] == 0 and j["value"] > 0
    assert j["config"]["parallelism"] == "dp2"
    assert j["config"]["grad_W_collective"].startswith("reduce-scatter fused")  # P2P windows
    assert j["e2e"]["value"] > 0 and j["gpu_launches"] > 0
    assert "cpu_baseline" not in j
