"""The C-ABI library loads without a GPU and exports every symbol that
include/hear_b200.h declares; task-table layouts agree with the C structs."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hear_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:hb|hear)_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2104_09164_b200 import _native as nat
    L = ctypes.CDLL(nat.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_layouts_and_version():
    from paper_2104_09164_b200 import _native as nat
    L = nat.lib()            # checks every task-table layout against C sizeof
    assert L.hb_version() == 1


def test_oracle_builds_and_loads():
    from oracle.cpu_engine import lib
    assert lib().or_num_threads() >= 1


def test_no_cpu_fallback():
    """The product path fails loudly: a missing kernel library raises on load,
    and the engine refuses to build a ring without a CUDA device."""
    import subprocess
    import sys
    code = ("import os, sys\n"
            "sys.path.insert(0, %r)\n"
            "from paper_2104_09164_b200 import _native as nat\n"
            "try:\n"
            "    nat.lib()\n"
            "except nat.NativeError as e:\n"
            "    assert 'no CPU fallback' in str(e), e\n"
            "    print('missing-lib raised')\n") % ROOT
    env = dict(os.environ, HEAR_B200_LIB="/nonexistent/libhear_b200.so")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert out.returncode == 0 and "missing-lib raised" in out.stdout, out.stderr

    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present: the no-device branch is not reachable")
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    with pytest.raises(nat.NativeError, match="CUDA device"):
        CkksBackend(gen_params("toy-fast"), seed=1)


def test_every_hear_symbol_is_called():
    """Guard: the integration stub (run as written by test_gpu_boundary.py) binds
    every hear_* entry point the header declares."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hdr = re.sub(r"/\*.*?\*/", "", open(os.path.join(root, "include", "hear_b200.h")).read(),
                 flags=re.S)
    declared = set(re.findall(r"\b(hear_[a-z0-9_]+)\s*\(", hdr))
    stub = open(os.path.join(root, "integration", "hear_ring_b200.py")).read()
    called = set(re.findall(r"_L\.(hear_[a-z0-9_]+)\b", stub))
    assert declared == called, declared ^ called
