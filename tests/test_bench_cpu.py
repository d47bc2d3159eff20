"""CPU checks of bench.py's host logic: the MAC counts behind the roofline
numerator against the oracle, and the multi-rank orchestration
(`--gpus N` starts N ranks itself; sharding, barriers, max over ranks, one
line from rank 0) with a stubbed step under gloo."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import bench
import oracle
from conftest import ROOT
from paper_1704_07724_b200 import datagen

CASES = ([(datagen.CONFIGS[c].with_batch(2), datagen.CONFIG_SPARSITY[c][0]) for c in datagen.CONFIGS] +
         [(shp.with_batch(2), 0.95) for shp in datagen.C5_LAYERS] + datagen.table2_shapes(n=2))


@pytest.mark.parametrize("shp,s", CASES, ids=[c[0].name for c in CASES])
def test_bench_mac_counts_equal_oracle(shp, s):
    x = datagen.activations(shp, s, seed=4)
    x[0, 0, 0, 0] = -0.0                      # R7: -0.0 is a zero
    dense, exact, nnz = bench.mac_counts(x, shp)
    assert dense == oracle.dense_macs(shp.n, shp.c, shp.h, shp.w, shp.k, shp.r, shp.s, shp.stride, shp.pad,
                                      shp.groups)
    assert exact == oracle.exact_nonzero_macs(x, shp.k, shp.r, shp.s, shp.stride, shp.pad, shp.groups)
    assert nnz == round((1 - oracle.sparsity(x)) * x.size)


def _run_bench(args, env_extra=None):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return r, lines


@pytest.mark.parametrize("config,scaling,batch", [("C5", "strong", 1024), ("C2", "weak", 256)])
def test_gpus2_launches_two_ranks_and_prints_one_line(config, scaling, batch):
    r, lines = _run_bench(["--gpus", "2", "--config", config, "--cpu-stub", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["config"]["global_batch"] == batch and line["config"]["parallelism"] == "dp2"
    assert line["config"]["images_per_step"] == batch       # every image of the job on exactly one rank
    assert line["steps"] == 2 and line["warmup"] == 3


def test_world_size_must_match_gpus():
    r, lines = _run_bench(["--gpus", "1", "--cpu-stub", "--steps", "1"], {"WORLD_SIZE": "2"})
    assert r.returncode == 2 and not lines
