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
