"""Part 1 on adversarial layouts (tests/_adv_layout_check.py) under each adv-norm driver:
the small cooperative driver (default for <= 2048 trajectories), the large cooperative driver
(build variant advlarge), the 3-kernel path (coop0) and the small driver staging 64-chunk
windows so that trajectories cross window boundaries inside a block (kc64).  One process per
library (AGENTRL_LIB)."""
import os
import subprocess
import sys

import pytest

from variants import variant_env

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("name", [None, "advlarge", "coop0", "kc64"],
                         ids=["small", "large", "three_kernel", "small_kc64"])
def test_adv_layouts(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = variant_env(name) if name else {}
    r = subprocess.run([sys.executable, os.path.join(HERE, "_adv_layout_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
