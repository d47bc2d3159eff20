"""bench.py keeps the driver's contract: one JSON line with the required keys, device-timed value,
roofline and end-to-end objects, clocks, and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run_bench("--steps", "3", "--warmup", "3", "--no-sweep", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["value"] > 0
    assert d["scaling"] == "weak" and d["higher_is_better"] is True
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] < 1 and r["achieved"] > 0 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3 * 2
    assert d["clocks"]["sm_mhz"] > 0


def test_bench_reference_arm():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_pair_config_two_streams():
    """C4 = C4a + C4b forked onto two streams: one line, both layers' work."""
    d = run_bench("--config", "C4", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["scaling"] == "weak"
    assert set(d["layers_alone_us"]) == {"C4a", "C4b"}
    assert d["roofline_step"]["dense_macs"] > 0 and d["dense_tc"]["us_sequential"] > 0


def test_bench_chain_config_strong_scaling_line():
    """C5 (the scaling config): the 1024-image chain on the ranks present (here one)."""
    d = run_bench("--config", "C5", "--gpus", "1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline")
    assert d["n_gpus"] == 1 and d["scaling"] == "strong" and d["config"]["global_batch"] == 1024
    assert len(d["layers_unfused_us"]) == 3 and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.parametrize("config,batch", [("C2", 256), ("C5", 1024)])
def test_two_ranks_on_one_gpu_functional(config, batch):
    """The multi-rank path on hardware with fewer GPUs than ranks (this pool: one): `--gpus 2`
    re-launches under torchrun, the ranks share the GPU and synchronise over gloo
    (SC_DIST_BACKEND=gloo; their kernels never wait on one another), shard the batch
    (C2: weak, each rank its own 128 images; C5: the 1024 images split), time between
    barriers and take the max over ranks.  The line says it is not a scaling number."""
    env = dict(os.environ, SC_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-sweep"],
                       capture_output=True, text=True, cwd=ROOT, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["global_batch"] == batch
    assert "functional_only" in d["config"]

