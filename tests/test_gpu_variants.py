"""The A/B build variants of the CUDA path stay parity-green.  Schedule and staging switches are
compile-time constants (paper_2510_04206_b200/build.py VARIANTS); each variant is the same
sources built with -D overrides and loaded in its own process (AGENTRL_LIB):
  pair0        1-CTA cta_group::1 GEMMs (128 x 256 tiles)
  static       static persistent tile striding
  narrow       256-column backward tiles
  fullgrid     one CTA (pair) per tile
  raster       raster group sizes 1 / 3 and evict_last on every operand
  ksub1        one 64-wide K atom per forward stage
  lead0        backward progress throttle off
  lockstep     throttle lead 1 checked every k-block (every pair waits for the slowest)
  pair0_lead2  1-CTA GEMMs with a lead-2 throttle
  coop0        3-kernel adv-norm path
Schedule-only switches must not change a bit of the result (test_schedule_variants_bitwise),
and the lockstep build must actually wait (the throttle's wait counter)."""
import os
import subprocess
import sys

import pytest

from variants import variant_env

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

VARIANTS = ["pair0", "static", "narrow", "fullgrid", "raster", "ksub1", "lead0", "pair0_lead2",
            "coop0", "ksplit3"]
# switches that only change the schedule / staging / stream placement, never the arithmetic
SCHEDULE_ONLY = ["lead0", "lockstep", "ksub1", "static", "fullgrid", "raster", "narrow", "pf8"]


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", VARIANTS)
def test_variant_parity(name):
    _cuda()
    env = variant_env(name)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


def _dump(env, path):
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_dump.py"), str(path)],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    import numpy as np
    return dict(np.load(path))


@pytest.fixture(scope="module")
def default_dump(tmp_path_factory):
    _cuda()
    return _dump({}, tmp_path_factory.mktemp("dflt") / "d.npz")


@pytest.mark.parametrize("name", SCHEDULE_ONLY)
def test_schedule_variants_bitwise(name, default_dump, tmp_path):
    """Tile order, progress throttle, K atoms per stage, L2 policies, tile width and grid shape
    change no arithmetic: loss, adv, grad_hidden and grad_W are bit-identical (ragged, parity7b
    and the long-K config longk)."""
    import numpy as np
    got = _dump(variant_env(name), tmp_path / "v.npz")
    for k, v in default_dump.items():
        if k == "throttle_waits":
            continue
        assert np.array_equal(got[k], v), k
    if name == "lockstep":  # lead 1: the throttle must have held pairs back
        assert got["throttle_waits"][1] > 0 and got["throttle_waits"][2] > 0, got["throttle_waits"]
