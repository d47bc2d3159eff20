#!/usr/bin/env python3
"""bench.py -- headline benchmark of the ReLU-sparse convolution (arXiv 1704.07724).

Metric (BASELINE.json): sparse conv dense-equivalent GFLOP/s (and nonzero-MAC/s,
% roofline) at s = 0.9 / 0.95 / 0.99.  Workload (BASELINE.json configs[1], the
config the metric is quoted on): AlexNet conv3, N=128 images per GPU,
256x13x13 -> 384 filters 3x3, pad 1, stride 1, fp32, i.i.d. Bernoulli(1-s) *
|N(0,1)| activations; the headline line is s = 0.95.

A "step" = one sparse_conv_forward (stage 1 compaction + stage 2 gather conv)
over the 128-image batch, inputs resident in HBM.  Steps rotate over several
input/output sets whose total (>= 220 MB) exceeds the 126 MB L2.  Each step is
one CUDA-graph replay (graph captured around the C-ABI call) so host launch
latency does not leak into the device time.

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--sparsity S] [--config C2]
  python bench.py --impl reference ...   (the CPU oracle as the reference arm)
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (weak scaling: each
rank processes its own 128 images, batch-sharded by global image index; no
collective on the data path, P:71 -- images are independent).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1704_07724_b200 import datagen  # noqa: E402

METRIC = "sparse conv dense-equiv GFLOP/s & nonzero-MAC/s at s=0.9/0.95/0.99; % roofline"
SM_COUNT = 148
FMA_PER_CLK_PER_SM = 128          # FP32 lanes per SM (B200), DESIGN.md "Roofline"
F_MAX_GHZ = 1.965                 # clocks.max.sm


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ counting
def coverage(extent_in, k, stride, pad, extent_out):
    """#taps mapping input coordinate i to a valid output (inverse map, R6)."""
    cov = np.zeros(extent_in, dtype=np.int64)
    for i in range(extent_in):
        for r in range(k):
            num = i + pad - r
            if num >= 0 and num % stride == 0 and num // stride < extent_out:
                cov[i] += 1
    return cov


def mac_counts(x, shp):
    """dense MACs and exact nonzero MACs of one batch."""
    dense = x.shape[0] * shp.ho * shp.wo * shp.r * shp.s * shp.k * (shp.c // shp.groups)
    ch = coverage(shp.h, shp.r, shp.stride, shp.pad, shp.ho)
    cw = coverage(shp.w, shp.s, shp.stride, shp.pad, shp.wo)
    per_pos = (x != 0).sum(axis=(0, 1)).astype(np.int64)
    exact = int((shp.k // shp.groups) * (ch[:, None] * cw[None, :] * per_pos).sum())
    return dense, exact, int(np.count_nonzero(x))


def algorithmic_bytes(shp, n, nnz, idx_bytes, num_lists):
    """Two-stage minimum traffic: dense in + dense out + weights + bias
    + compacted lists written once and read once."""
    dense_in = 4 * n * shp.c * shp.h * shp.w
    dense_out = 4 * n * shp.k * shp.ho * shp.wo
    wts = 4 * shp.k * (shp.c // shp.groups) * shp.r * shp.s + 4 * shp.k
    lists = nnz * (4 + idx_bytes) + 4 * num_lists
    return dense_in + dense_out + wts + 2 * lists, dense_in, lists


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons in a background thread."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append(mhz)
                for bit, name in self.REASONS.items():
                    if rs & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": len(self.samples)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_name(shp, s):
    return (f"{shp.name}: N={shp.n}/GPU, {shp.c}x{shp.h}x{shp.w} -> {shp.k} {shp.r}x{shp.s} "
            f"stride {shp.stride} pad {shp.pad} groups {shp.groups}, s={s}")


def cpu_oracle_rate(shp, x_imgs, w, b, min_s=10.0, max_s=30.0):
    """Time the fp64 oracle (as it stands) on host cores; repeat passes over the
    given images until >= min_s.  Returns (dense-equiv GFLOP/s, images, seconds)."""
    import oracle  # the one product-side place the oracle may run (cpu_baseline leg)
    oracle.build()
    per_img_flops = 2 * shp.ho * shp.wo * shp.r * shp.s * shp.k * (shp.c // shp.groups)
    t0 = time.perf_counter()
    done = 0
    i = 0
    while True:
        xi = x_imgs[i % x_imgs.shape[0]: i % x_imgs.shape[0] + 1]
        oracle.conv_fp64(xi, w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
        done += 1
        i += 1
        el = time.perf_counter() - t0
        if el >= min_s or (el >= max_s * 0.5 and done >= 1):
            break
    el = time.perf_counter() - t0
    return per_img_flops * done / el / 1e9, done, el


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    shp = datagen.CONFIGS[args.config]
    s = args.sparsity
    w, b = datagen.weights(shp)
    import oracle
    oracle.build()
    per_img_flops = 2 * shp.ho * shp.wo * shp.r * shp.s * shp.k * (shp.c // shp.groups)
    # bounded sample per step: images chosen so one step takes ~1-3 s of CPU work
    x = datagen.activations(shp, s, start=0, count=8)
    t0 = time.perf_counter()
    oracle.conv_fp64(x[:1], w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
    t1 = time.perf_counter() - t0
    m = int(max(1, min(8, 2.0 // max(t1, 1e-3))))
    xs = x[:m]
    for _ in range(args.warmup):
        oracle.conv_fp64(xs, w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.conv_fp64(xs, w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_img_flops * m * len(times) / tot / 1e9
    sample = f"{m} of the {shp.n} images of the workload per step (fp64 oracle, OpenMP), {args.steps} steps"
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(shp, s)},
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": host_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    from paper_1704_07724_b200 import sparseconv as sc

    shp = datagen.CONFIGS[args.config]
    s_head = args.sparsity
    n = shp.n
    w, b = datagen.weights(shp)                     # same seed on every rank: replicated weights
    conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups)
    launches_per_step = conv.launch_counts[0]
    peaks, peak_kind = measured_peaks()
    hbm_gbs = float(peaks.get("hbm_gbs", 6650.0))
    fp32_peak_tflops = SM_COUNT * FMA_PER_CLK_PER_SM * 2 * F_MAX_GHZ / 1e3   # 74.4
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size

    def measure(s, steps, warmup, sets_min_bytes=2 * 126 * 2 ** 20, main=False):
        per_set = 4 * n * (shp.c * shp.h * shp.w + shp.k * shp.ho * shp.wo)
        nsets = max(2, -(-max(sets_min_bytes, 2 * l2_bytes) // per_set))
        xs, outs, counts = [], [], []
        for si in range(nsets):
            start = (si * ws + rank) * n                     # global image index (shard-independent data)
            xh = datagen.activations(shp, s, start=start, count=n)
            counts.append(mac_counts(xh, shp))
            xs.append(torch.from_numpy(xh).to(dev))
            outs.append(torch.empty((n, shp.k, shp.ho, shp.wo), device=dev))
        stream = torch.cuda.Stream(dev)
        graphs, graphs_gather, graphs_compact = [], [], []
        with torch.cuda.stream(stream):
            for si in range(nsets):            # eager warm-up once per set (also sets kernel attributes)
                conv.forward(xs[si], outs[si], stream=stream)
            stream.synchronize()
            for si in range(nsets):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                    conv.forward(xs[si], outs[si], stream=stream)
                graphs.append(g)
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1, stream=stream, capture_error_mode="relaxed"):
                conv.compact(xs[0], stream=stream)
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=stream, capture_error_mode="relaxed"):
                conv.gather(n, outs[0], stream=stream)
        res = {}
        with torch.cuda.stream(stream):
            for i in range(warmup):
                graphs[i % nsets].replay()
            stream.synchronize()
            if ws > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(steps):
                graphs[i % nsets].replay()
            e1.record(stream)
            e1.synchronize()
            torch.cuda.synchronize(dev)
            elapsed_ms = e0.elapsed_time(e1)
            if ws > 1:
                t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                elapsed_ms = float(t.item())
                torch.distributed.barrier()
            res["ms_per_step"] = elapsed_ms / steps
            # per-stage durations on the launching stream (gather = the dominant kernel):
            # set 0's lists are rebuilt by the compaction graph before the gather graph runs
            reps = max(steps, 50)
            g1.replay()
            stream.synchronize()
            for name, g in (("gather", g2), ("compact", g1)):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for _ in range(reps):
                    g.replay()
                a1.record(stream)
                a1.synchronize()
                res[f"{name}_us"] = a0.elapsed_time(a1) * 1e3 / reps
        dense = sum(c[0] for c in counts) / nsets
        exact = sum(c[1] for c in counts) / nsets
        nnz = sum(c[2] for c in counts) / nsets
        res.update(dense=dense, exact=exact, nnz=nnz, exact_set0=counts[0][1], nsets=nsets,
                   realized_s=1 - nnz / (n * shp.c * shp.h * shp.w))
        del graphs, graphs_gather, graphs_compact, g1, g2
        return res

    clocks = ClockSampler(dev.index)
    with clocks:
        head = measure(s_head, args.steps, args.warmup, main=True)
        sweep = {}
        if not args.no_sweep:
            for s in (0.9, 0.95, 0.99):
                if abs(s - s_head) < 1e-9:
                    continue
                sweep[s] = measure(s, max(args.steps, 20), max(args.warmup, 3))
        # clocks need a long enough loaded window: keep replaying the headline workload ~0.5 s
        if head["ms_per_step"] * args.steps < 300.0:
            measure(s_head, int(400.0 / max(head["ms_per_step"], 1e-3)) + 1, 3)

    # --- end to end through the public API with host buffers (pinned) -------------
    xh = datagen.activations(shp, s_head, start=rank * n, count=n)
    h_in = torch.from_numpy(xh).pin_memory()
    h_out = torch.empty((n, shp.k, shp.ho, shp.wo)).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        conv.forward_host(h_in, h_out)
    if ws > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        conv.forward_host(h_in, h_out)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if ws > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    def gflops(dense, ms):
        return 2 * dense * ws / (ms * 1e-3) / 1e9

    v = head
    value = gflops(v["dense"], v["ms_per_step"])
    nz_rate = v["exact"] * ws / (v["ms_per_step"] * 1e-3)
    idx_bytes = 1
    lists = n * shp.c * 1
    tot_bytes, _, _ = algorithmic_bytes(shp, n, v["nnz"], idx_bytes, lists)
    t_fp32 = v["exact"] / (fp32_peak_tflops / 2 * 1e12)
    t_hbm = tot_bytes / (hbm_gbs * 1e9)
    t_roof = max(t_fp32, t_hbm)
    # dominant kernel roofline: stage-2 gather, FP32 FMA (ALU) bound
    g_flops = 2 * v["exact_set0"]
    achieved = g_flops / (v["gather_us"] * 1e-6) / 1e12
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(v["ms_per_step"], 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(shp, s_head), "global_batch": n * ws, "parallelism": f"dp{ws}",
                   "l2": f"{v['nsets']} rotating input/output sets ({v['nsets'] * 4 * n * (shp.c * shp.h * shp.w + shp.k * shp.ho * shp.wo) / 2 ** 20:.0f} MiB > L2)",
                   "timing": "CUDA events around K CUDA-graph replays (one sparse_conv_forward each)",
                   "realized_sparsity": round(v["realized_s"], 5), "variant": conv.variant[1]},
        "nonzero_mac_per_s": round(nz_rate, 1),
        "pct_roofline": round(100 * t_roof / (v["ms_per_step"] * 1e-3), 2),
        "roofline_step": {"t_roof_us": round(t_roof * 1e6, 3), "t_fp32_us": round(t_fp32 * 1e6, 3),
                          "t_hbm_us": round(t_hbm * 1e6, 3), "bytes": int(tot_bytes),
                          "exact_nonzero_macs": int(v["exact"]), "dense_macs": int(v["dense"])},
        "roofline": {"kernel": "gather (stage 2)", "bound": "alu", "achieved": round(achieved, 3),
                     "peak": round(fp32_peak_tflops, 2), "unit": "TFLOP/s", "frac": round(achieved / fp32_peak_tflops, 4),
                     "traffic": None,
                     "peak_note": "FP32 FMA: 148 SMs x 128 lanes x 2 flop x 1.965 GHz (unit counts x max clock)"},
        "stages_us": {"compact": round(v["compact_us"], 3), "gather": round(v["gather_us"], 3)},
        "compact_hbm": {"achieved_gbs": round(4 * n * shp.c * shp.h * shp.w / (v["compact_us"] * 1e-6) / 1e9, 1),
                        "peak_gbs": hbm_gbs, "peak_kind": peak_kind},
        "sweep": {str(s): {"value": round(gflops(r["dense"], r["ms_per_step"]), 2),
                           "nonzero_mac_per_s": round(r["exact"] * ws / (r["ms_per_step"] * 1e-3), 1),
                           "ms_per_step": round(r["ms_per_step"], 5),
                           "pct_roofline": round(100 * max(r["exact"] / (fp32_peak_tflops / 2 * 1e12),
                                                           algorithmic_bytes(shp, n, r["nnz"], 1, lists)[0] /
                                                           (hbm_gbs * 1e9)) / (r["ms_per_step"] * 1e-3), 2),
                           "gather_us": round(r["gather_us"], 3), "compact_us": round(r["compact_us"], 3)}
                  for s, r in sweep.items()},
        "e2e": {"value": round(gflops(v["dense"], e2e_s * 1e3), 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(h_in.numel() * 4), "d2h_bytes_per_step": int(h_out.numel() * 4),
                "ms_per_step": round(e2e_s * 1e3, 4), "api": "sparse_conv_forward_host (pinned host buffers)"},
        "gpu_launches": int(args.steps * launches_per_step),
        "clocks": clocks.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, imgs, secs = cpu_oracle_rate(shp, datagen.activations(shp, s_head, start=0, count=min(n, 16)), w, b)
        line["cpu_baseline"] = {"value": round(rate, 3), "unit": "GFLOP/s", "cores": host_cores(), "kind": "oracle",
                                "sample": f"{imgs} single-image oracle calls over images 0..15 of the workload "
                                          f"({secs:.1f} s, fp64 7-loop, OpenMP)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--sparsity", type=float, default=0.95)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
