"""The A/B variants of the CUDA path stay parity-green (each in its own process: the library
reads the AGENTRL_* switches once):
  AGENTRL_GEMM_PAIR=0       1-CTA cta_group::1 GEMMs (128 x 256 tiles)
  AGENTRL_GEMM_SCHED=static static persistent tile striding
  AGENTRL_GEMM_NSPLIT=1     256-column backward tiles
  AGENTRL_GEMM_FULLGRID=1   one CTA (pair) per tile
  AGENTRL_ADV_COOP=0        3-kernel adv-norm path
  AGENTRL_GROUP_M / _BWD    raster group sizes
  AGENTRL_FWD_KSUB=1        one 64-wide K atom per forward stage
  AGENTRL_FWD_CHUNKS=n      forward row chunks (merge overlap; default 1)
  AGENTRL_MERGE_BPS=n       merge blocks per SM (default: the occupancy limit, one wave)
  AGENTRL_THROTTLE_LEAD=n   backward progress throttle (0 = off; 1 with EVERY=1: lockstep)
Schedule-only switches must not change a bit of the result (test_schedule_variants_bitwise).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = [
    {"AGENTRL_GEMM_PAIR": "0"},
    {"AGENTRL_GEMM_SCHED": "static"},
    {"AGENTRL_GEMM_NSPLIT": "1"},
    {"AGENTRL_GEMM_FULLGRID": "1"},
    {"AGENTRL_ADV_COOP": "0"},
    {"AGENTRL_GROUP_M": "1", "AGENTRL_GROUP_M_BWD": "3"},
    {"AGENTRL_L2POL": "222222"},
    {"AGENTRL_FWD_KSUB": "1", "AGENTRL_FWD_CHUNKS": "1", "AGENTRL_THROTTLE_LEAD": "0"},
    {"AGENTRL_GEMM_PAIR": "0", "AGENTRL_THROTTLE_LEAD": "2", "AGENTRL_THROTTLE_EVERY": "1"},
]

# switches that only change the schedule / staging / stream placement, never the arithmetic
SCHEDULE_ONLY = [
    {"AGENTRL_THROTTLE_LEAD": "0"},
    {"AGENTRL_THROTTLE_LEAD": "1", "AGENTRL_THROTTLE_EVERY": "1"},
    {"AGENTRL_FWD_CHUNKS": "4"},
    {"AGENTRL_FWD_CHUNKS": "8"},
    {"AGENTRL_BWD_OVERLAP": "1"},
    {"AGENTRL_MERGE_BPS": "1"},
    {"AGENTRL_MERGE_BPS": "8"},
    {"AGENTRL_FWD_KSUB": "1"},
    {"AGENTRL_GEMM_SCHED": "static"},
    {"AGENTRL_GEMM_FULLGRID": "1"},
    {"AGENTRL_GROUP_M": "1", "AGENTRL_GROUP_M_BWD": "3"},
    {"AGENTRL_L2POL": "222222"},
    {"AGENTRL_GEMM_NSPLIT": "1"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k[8:]}={v}" for k, v in e.items()))
def test_variant_parity(env):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


def _dump(env, path):
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_dump.py"), str(path)],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    import numpy as np
    return dict(np.load(path))


@pytest.fixture(scope="module")
def default_dump(tmp_path_factory):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _dump({}, tmp_path_factory.mktemp("dflt") / "d.npz")


@pytest.mark.parametrize("env", SCHEDULE_ONLY,
                         ids=lambda e: ",".join(f"{k[8:]}={v}" for k, v in e.items()))
def test_schedule_variants_bitwise(env, default_dump, tmp_path):
    """Tile order, progress throttle, row chunks, K atoms per stage, L2 policies and grid
    shape change no arithmetic: loss, adv, grad_hidden and grad_W are bit-identical."""
    import numpy as np
    got = _dump(env, tmp_path / "v.npz")
    for k, v in default_dump.items():
        assert np.array_equal(got[k], v), k
