"""Host-side checks (no GPU): the C-ABI library loads and exports every symbol that
include/agentrl.h declares; the oracle and the CUDA path share no code; workspace
planning is sane; the binding refuses to run without the library (no fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "agentrl.h")
PKG = os.path.join(ROOT, "paper_2510_04206_b200")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(agentrl_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    import __graft_entry__
    return __graft_entry__._load_builder().build()


def test_build_works_without_prebuilt_library(tmp_path):
    """A fresh checkout has no .so: the builder (loaded by path, never through the package,
    whose __init__ refuses to load without the library) must produce one from scratch."""
    import __graft_entry__
    b = __graft_entry__._load_builder()
    b.LIB = str(tmp_path / "libagentrl.so")
    b.BUILD = str(tmp_path / "obj")
    out = b.build(force=True)
    lib = ctypes.CDLL(out)
    assert hasattr(lib, "agentrl_grpo_step")


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    import paper_2510_04206_b200 as ag
    assert set(ag.EXPORTED) == set(names)


def test_sm100a_code_in_library(libpath):
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "arch = sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in out, mnem  # tcgen05.mma, TMA loads, tcgen05.ld


def test_host_calls_without_gpu(libpath):
    import paper_2510_04206_b200 as ag
    assert ag.lib().agentrl_version() == 100
    assert ag.status_string(ag.ERR_WORKSPACE).startswith("workspace")
    assert ag.status_string(ag.ST_NO_TOKENS).startswith("no loss-masked")
    ws = ag.agentrl_grpo_step_workspace_size(131072, 640, 80, 5, 4096, 151552)
    # the bf16 P~ buffer dominates: rows_cap * V * 2 bytes, rows_cap = T without a bound
    assert ws >= 131072 * 151552 * 2
    assert ws < 131072 * 151552 * 2 * 1.1
    # sized by the caller's bound on the masked rows instead (glm9b: T_eff = 53,039 -> 16.1 GB)
    ws_b = ag.agentrl_grpo_step_workspace_size(131072, 640, 80, 5, 4096, 151552, max_rows=53039)
    rows_cap = (53039 + 127) // 128 * 128
    assert rows_cap * 151552 * 2 <= ws_b < rows_cap * 151552 * 2 * 1.1
    assert ag.agentrl_policy_loss_workspace_size(131072, 4096, 151552, max_rows=53039) < ws_b
    assert ag.agentrl_task_adv_norm_workspace_size(0, 0, 0, 1) > 0


def test_oracle_and_product_share_no_code():
    prod = []
    for dp, _, fs in os.walk(PKG):
        prod += [os.path.join(dp, f) for f in fs if f.endswith((".py", ".cu", ".cuh", ".h"))]
    for p in prod:
        s = open(p).read()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", s, re.M), p
        assert "agentrl_oracle" not in s, p
    for dp, _, fs in os.walk(os.path.join(ROOT, "oracle")):
        for f in fs:
            if f.endswith((".py", ".c", ".h")):
                s = open(os.path.join(dp, f)).read()
                code_lines = [ln for ln in s.splitlines()
                              if re.match(r"\s*(#\s*include|import|from)\b", ln)]
                for ln in code_lines:
                    assert "paper_2510_04206_b200" not in ln and "agentrl.h" not in ln, (f, ln)
                    assert "csrc" not in ln and "synth" not in ln, (f, ln)
    s = open(os.path.join(ROOT, "synth", "__init__.py")).read()
    assert "import oracle" not in s and "paper_2510_04206_b200" not in s


def test_missing_library_fails_loudly(tmp_path):
    code = ("import sys, os, shutil; sys.path.insert(0, %r);"
            "import importlib.util as u;"
            "spec = u.spec_from_file_location('x', %r);"
            "m = u.module_from_spec(spec);"
            "m.__file__ = os.path.join(%r, '__init__.py');"
            "spec.loader.exec_module(m)") % (ROOT, os.path.join(PKG, "__init__.py"), str(tmp_path))
    # exec the binding with its __file__ pointing at an empty dir -> must raise ImportError
    src = open(os.path.join(PKG, "__init__.py")).read()
    fake = tmp_path / "__init__.py"
    fake.write_text(src)
    r = subprocess.run(["python", "-c", f"import runpy; runpy.run_path({str(fake)!r})"],
                       capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr
    del code


def test_reduce_scatter_mode_contract(libpath):
    """grad_W_mode 2 (reduce-scatter row shards) needs V % world == 0: SHAPE before any device
    work.  Host-side checks only (fake, aligned, never-dereferenced
    pointers; the call returns before touching the device).  Mode 4 does not exist."""
    import paper_2510_04206_b200 as m
    comm = m.CallbackComm(3, 0, lambda *a: None)
    fake = 1 << 20
    args = m.LossArgs(T=16, d=64, V=2000, hidden=fake, W_head=fake, target=fake, adv_tok=fake,
                      old_logp=fake, loss_mask=fake, clip_eps_low=0.2, clip_eps_high=0.2,
                      logit_scale=1.0, n_mask_global=fake, grad_W_mode=2)
    out = m.LossOut(loss=fake, grad_hidden=fake, grad_W=fake)
    call = lambda: m._lib.agentrl_policy_loss_fwd_bwd(ctypes.byref(args), ctypes.byref(out), fake,
                                                      1 << 30, comm.handle, fake, None)
    assert call() == m.ERR_SHAPE          # 2000 % 3 != 0
    args.V = 2016                          # divisible: passes this check, fails later (no GPU)
    assert call() not in (m.ERR_SHAPE, m.ERR_INVALID_ARG, 0)
    args.grad_W_mode = 4
    assert call() == m.ERR_INVALID_ARG
    # the peer window needs a communicator (and, past the host checks, a device); size 0
    # disables it (nothing to free here: a no-op)
    assert m._lib.agentrl_comm_enable_peer_window(comm.handle, 0) == m.OK
    assert m._lib.agentrl_comm_enable_peer_window(None, 1 << 20) == m.ERR_INVALID_ARG
    # mode 3 (vocabulary-parallel head) needs a communicator and is not a fused-step mode
    args.grad_W_mode = 3
    assert m._lib.agentrl_policy_loss_fwd_bwd(ctypes.byref(args), ctypes.byref(out), fake,
                                              1 << 30, None, fake, None) == m.ERR_INVALID_ARG
    assert call() not in (m.ERR_SHAPE, m.ERR_INVALID_ARG, 0)  # passes the host checks
    assert (m.agentrl_policy_loss_workspace_size_vp(1024, 64, 512, 4)
            >= m.agentrl_policy_loss_workspace_size(1024, 64, 512) + 8 * 4 * 1024 + 4 * 1024 * 64)
    comm.destroy()


def test_product_library_reads_one_runtime_switch():
    """Schedule and staging choices are compile-time constants (build.py VARIANTS); the only
    environment switch the library reads is the documented AGENTRL_C3_P2P."""
    hits = []
    for f in sorted(x for x in os.listdir(os.path.join(PKG, "csrc")) if x.endswith((".cu", ".cuh", ".h"))):
        src = open(os.path.join(PKG, "csrc", f)).read()
        hits += re.findall(r'getenv\("([A-Z_0-9]+)"\)', src)
    assert hits == ["AGENTRL_C3_P2P"], hits
