"""CPU-only checks of the C-ABI library: it loads, exports every symbol the headers declare, and its
host logic (schedule, argument validation) behaves as documented. No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import cacheblend_oracle as O
from paper_2405_16444_b200 import _lib
from paper_2405_16444_b200.build import build
from tests.conftest import ROOT


@pytest.fixture(scope="module")
def L():
    build()
    return _lib.lib()


def _declared():
    names = []
    for h in ("cacheblend.h", "cacheblend_ops.h"):
        with open(os.path.join(ROOT, "include", h)) as f:
            names += re.findall(r"^CB_API [^(]*?\b(cb_\w+)\(", f.read(), flags=re.M)
    return names


def test_exports_every_declared_symbol(L):
    decl = _declared()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_lib.EXPORTED)


def test_schedule_matches_oracle(L):
    for r in (0.0, 0.05, 0.1, 0.15, 0.18, 0.3, 0.5, 0.77, 1.0):
        for n in (0, 1, 7, 96, 3072, 8192, 10240):
            for layers in (1, 2, 3, 32, 60, 80):
                out = (ctypes.c_int32 * layers)()
                assert L.cb_schedule(r, n, layers, out) == 0
                assert list(out) == O.schedule(r, n, layers), (r, n, layers)


def test_schedule_rejects_bad_ratio(L):
    out = (ctypes.c_int32 * 4)()
    assert L.cb_schedule(1.5, 10, 4, out) == -1
    assert b"ratio" in L.cb_last_error()
    assert L.cb_schedule(-0.1, 10, 4, out) == -1


def test_model_validation(L):
    m = _lib.CbModel(2, 64, 4, 4, 16, 256, 512, 10000.0, 1e-5, 1, 256)
    nb = ctypes.c_size_t()
    assert L.cb_workspace_size(ctypes.byref(m), 96, ctypes.byref(nb)) == 0 and nb.value > 0
    bad = _lib.CbModel(2, 64, 4, 4, 15, 256, 512, 10000.0, 1e-5, 1, 256)   # odd head_dim
    assert L.cb_workspace_size(ctypes.byref(bad), 96, ctypes.byref(nb)) == -1
    assert b"even" in L.cb_last_error()
    bad = _lib.CbModel(2, 64, 4, 3, 16, 256, 512, 10000.0, 1e-5, 1, 256)    # n_q % n_kv
    assert L.cb_workspace_size(ctypes.byref(bad), 96, ctypes.byref(nb)) == -1
    bad = _lib.CbModel(2, 64, 4, 4, 16, 256, 512, 10000.0, 1e-5, 7, 256)    # dtype
    assert L.cb_workspace_size(ctypes.byref(bad), 96, ctypes.byref(nb)) == -1


def test_null_context_rejected(L):
    assert L.cb_rope_realign(None, None, None, None, None, 1, 1, 1, None) == -1
    assert L.cb_blend_layer(None, 0, None, None, None, 0, 0, 0, None, None, None, 1, None, None, None, None) == -1


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2405_16444_b200", "libcacheblend.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out
