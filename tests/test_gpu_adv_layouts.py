"""Part 1 on adversarial layouts (tests/_adv_layout_check.py) under each adv-norm driver:
the small cooperative driver (default for <= 2048 trajectories), the large cooperative driver
(AGENTRL_ADV_SMALL=0) and the 3-kernel path (AGENTRL_ADV_COOP=0).  One process per driver:
the library reads the switches once."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{}, {"AGENTRL_ADV_SMALL": "0"}, {"AGENTRL_ADV_COOP": "0"}],
                         ids=["small", "large", "three_kernel"])
def test_adv_layouts(env):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_adv_layout_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
