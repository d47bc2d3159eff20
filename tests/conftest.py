import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden_kv(name):
    """key value... lines of a tests/golden fixture (comments start with #)."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            out[key] = vals
    return out


def read_table2():
    rows = []
    with open(os.path.join(GOLDEN, "table2_layers.csv")) as f:
        lines = [l.strip() for l in f if l.strip() and not l.startswith("#")]
    header = lines[0].split(",")
    for l in lines[1:]:
        vals = l.split(",")
        d = dict(zip(header, vals))
        rows.append(dict(name=d["name"], C=int(d["C"]), H=int(d["H"]), W=int(d["W"]), K=int(d["K"]),
                         R=int(d["R"]), S=int(d["S"]), P=int(d["P"]), T=int(d["T"]),
                         sparsity=float(d["sparsity"])))
    return rows


@pytest.fixture(scope="session")
def golden_kv():
    return read_golden_kv


@pytest.fixture(scope="session")
def table2():
    return read_table2()
