"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/mmas.h declares, and rejects invalid arguments before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2003_11902_b200 import build as mbuild
from paper_2003_11902_b200 import mmas

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    mbuild.build()
    return mmas.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "mmas.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mmas_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert sorted(mmas.EXPORTED) == names


def test_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mbuild.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("kw,frag", [
    (dict(n=2), "3 <= n"),
    (dict(rho=1.0), "rho"),
    (dict(alpha=1.5), "alpha"),
    (dict(cand_len=10), "cand_len"),
    (dict(n_ants=0), "n_ants"),
    (dict(beta=-1.0), "beta"),
    (dict(local_search=2), "local_search"),
    (dict(tabu=2), "tabu"),
    (dict(tabu=1), "cand_len == 0"),          # compact tabu needs the full-row path (R27)
    (dict(selection=2), "selection"),
    (dict(selection=1, fallback=1), "roulette"),
    (dict(world=2, rank=2), "rank"),
])
def test_invalid_arguments_rejected_without_gpu(L, kw, frag):
    c = np.arange(20, dtype=np.float64)
    cfg = mmas.Config()
    L.mmas_config_init(ctypes.byref(cfg))
    cfg.coords = c.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    cfg.n, cfg.n_ants, cfg.cand_len = 10, 5, 3
    for k, v in kw.items():
        setattr(cfg, k, v)
    h = ctypes.c_void_p()
    st = L.mmas_create_ex(ctypes.byref(cfg), ctypes.byref(h))
    assert st == mmas.MMAS_EINVAL and not h.value
    assert frag in L.mmas_last_error().decode()


def test_null_context_is_an_error(L):
    assert L.mmas_iterate(None, 1) == mmas.MMAS_EINVAL
    L.mmas_destroy(None)   # no-op
    assert L.mmas_create(None, 10, 1.0, 2.0, 0.5, 5, 3, 1) is None
