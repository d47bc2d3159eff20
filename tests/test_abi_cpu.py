"""CPU-only checks of the C-ABI boundary: the library builds for sm_100a,
loads, exports every symbol include/sparse_conv.h declares, and its pure-host
functions (shape rules, status strings, argument errors) behave.  No compute
calls are made here (there is no GPU in the dev container)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sparse_conv.h")


@pytest.fixture(scope="module")
def sc():
    from paper_1704_07724_b200 import build
    build.build()
    from paper_1704_07724_b200 import sparseconv
    return sparseconv


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(?:sc_status|const char \*|size_t|int32_t)\s*(\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("sparse_conv_create", "sparse_conv_forward", "dense_conv_forward", "sparse_conv_destroy"):
        assert f in fns


def test_library_exports_every_declared_symbol(sc):
    lib = ctypes.CDLL(sc.LIB_PATH)
    for f in declared_functions():
        assert hasattr(lib, f), f
    assert sorted(sc.EXPORTS) == declared_functions()


def test_library_is_sm100a(sc):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_output_shape_rules(sc):
    assert sc.output_shape(64, 20, 12, 12, 50, 5, 5) == (64, 50, 8, 8)
    assert sc.output_shape(1, 20, 11, 11, 64, 5, 5, 2, 1) == (1, 64, 5, 5)   # P:137, floor form (R1)
    assert sc.output_shape(128, 96, 27, 27, 256, 5, 5, 1, 2, 2) == (128, 256, 27, 27)
    with pytest.raises(sc.SparseConvError) as e:
        sc.output_shape(1, 3, 4, 4, 2, 1, 1, 1, 0, 2)
    assert e.value.status == 2
    with pytest.raises(sc.SparseConvError):
        sc.output_shape(1, 1, 2, 2, 1, 5, 5, 1, 0)
    with pytest.raises(sc.SparseConvError):
        sc.output_shape(1, 1, 2, 2, 1, 1, 1, 1, -1)
    with pytest.raises(sc.SparseConvError):
        sc.output_shape(0, 1, 2, 2, 1, 1, 1, 1, 0)


def test_output_shape_matches_oracle_rule(sc):
    import oracle
    rng = np.random.default_rng(0)
    for _ in range(200):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        p, t = int(rng.integers(0, 4)), int(rng.integers(1, 4))
        r, s = int(rng.integers(1, h + 2 * p + 1)), int(rng.integers(1, w + 2 * p + 1))
        assert sc.output_shape(2, 3, h, w, 4, r, s, t, p) == oracle.output_shape(2, 3, h, w, 4, r, s, t, p)


def test_status_strings(sc):
    L = sc.lib()
    for code in range(6):
        assert L.sc_status_string(code)
    assert L.sc_status_string(99) == b"unknown status"


def test_create_without_gpu_fails_cleanly(sc):
    L = sc.lib()
    p = sc.ConvParams(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 0)
    plan = ctypes.c_void_p(1234)
    st = L.sparse_conv_create(ctypes.byref(p), None, None, 0, ctypes.byref(plan))
    assert st != 0 and plan.value is None
    assert L.sparse_conv_destroy(None) == 0
    bad = sc.ConvParams(1, 3, 3, 3, 2, 3, 3, 1, 1, 2, 0)
    assert L.sparse_conv_create(ctypes.byref(bad), None, None, 0, ctypes.byref(plan)) == 2
    assert L.sparse_conv_forward(None, 1, None, None, None) == 1
    assert b"plan is NULL" in L.sc_last_error()
