"""The A/B variants of the CUDA path stay parity-green (each in its own process: the library
reads the AGENTRL_* switches once):
  AGENTRL_GEMM_PAIR=0       1-CTA cta_group::1 GEMMs (128 x 256 tiles)
  AGENTRL_GEMM_SCHED=static static persistent tile striding
  AGENTRL_GEMM_NSPLIT=1     256-column backward tiles
  AGENTRL_GEMM_FULLGRID=1   one CTA (pair) per tile
  AGENTRL_ADV_COOP=0        3-kernel adv-norm path
  AGENTRL_GROUP_M / _BWD    raster group sizes
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
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k[8:]}={v}" for k, v in e.items()))
def test_variant_parity(env):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
