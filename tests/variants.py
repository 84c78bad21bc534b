"""Variant libraries for the A/B parity tests: the same sources built with -D overrides of the
compile-time schedule switches (paper_2510_04206_b200/build.py VARIANTS), loaded in a subprocess
through AGENTRL_LIB.  (Build plumbing only.)"""
import importlib.util
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _builder():
    spec = importlib.util.spec_from_file_location(
        "_agentrl_build", os.path.join(ROOT, "paper_2510_04206_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def variant_env(name: str) -> dict:
    """{"AGENTRL_LIB": path} of the named variant, building it if missing or out of date
    (skips when nvcc is unavailable and no prebuilt library exists)."""
    import pytest
    b = _builder()
    path = b.variant_path(name)
    if not os.path.exists(b.NVCC) and not shutil.which("nvcc"):
        if not os.path.exists(path):
            pytest.skip("no nvcc and no prebuilt variant " + name)
        return {"AGENTRL_LIB": path}
    return {"AGENTRL_LIB": b.build_variant(name)}


def variant_flags(name: str) -> list:
    return list(_builder().VARIANTS[name])
