"""The run-time variant generator (csrc/jit.cu, a C++ port of
tools/gen_gather.py:gen_variant) emits exactly the code of the Python generator
that produced the shipped, GPU-validated variants.  Host-only: runs without a
GPU (the library loads; no device call is made)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import gen_gather  # noqa: E402

# (R, S, P, T, W, TY, KL, NW, MINB, CH, STAGES): shipped variants of every kind -- k-quads
# (V21), k-triples with a single f32 slot (V10), x-pairs (V29), stride 2 (V40), 1x1 (V43), 5x5 k-pairs
CASES = [
    (3, 3, 1, 1, 13, 2, 4, 11, 1, 16, 2),
    (3, 3, 1, 1, 13, 3, 3, 11, 1, 8, 4),
    (5, 5, 2, 1, 28, 4, 1, 11, 1, 16, 2),
    (5, 5, 1, 2, 11, 5, 2, 11, 1, 8, 2),
    (1, 1, 0, 1, 14, 2, 4, 11, 1, 32, 2),
    (5, 5, 2, 1, 7, 5, 2, 11, 1, 8, 2),
    (7, 3, 0, 1, 20, 1, 1, 11, 1, 16, 2),
]


@pytest.fixture(scope="module")
def sc():
    from paper_1704_07724_b200 import sparseconv
    try:
        sparseconv.lib()
    except RuntimeError as e:
        pytest.skip(str(e))
    return sparseconv


@pytest.mark.parametrize("case", CASES)
def test_cpp_generator_matches_python(sc, case):
    R, S, P, T, W, TY, KL, NW, MINB, CH, STAGES = case
    py = gen_gather.gen_variant(1000, "jit", R, S, P, W, TY, KL, NW, MINB, CH, STAGES, T=T)
    cpp = sc.jit_variant_source(R, S, P, T, W, TY, KL, NW, MINB, CH, STAGES, 3, 254, 1000)
    assert cpp.rstrip("\n") == py.rstrip("\n")
