#!/usr/bin/env python3
"""bench.py -- headline benchmark of the ReLU-sparse convolution (arXiv 1704.07724).

Metric (BASELINE.json): sparse conv dense-equivalent GFLOP/s (and nonzero-MAC/s,
% roofline) at s = 0.9 / 0.95 / 0.99.  Default workload (BASELINE.json
configs[1], the config the metric is quoted on): AlexNet conv3, N=128 images per
GPU, 256x13x13 -> 384 filters 3x3, pad 1, stride 1, fp32, i.i.d.
Bernoulli(1-s) * |N(0,1)| activations; the headline line is s = 0.95 and the
other two sparsities are reported under "sweep".

A "step" = one sparse_conv_forward (stage 1 compaction + stage 2 gather conv)
over the batch, inputs resident in HBM.  Steps rotate over several input/output
sets whose total exceeds 2x the 126 MB L2.  Each step is one CUDA-graph replay
(captured around the C-ABI call).  Per-stage device times come from graphs
holding REPS back-to-back launches (host launch cost excluded).

--config C5: the AlexNet conv3->conv4->conv5 chain (BASELINE.json configs[4]),
N=1024 images split over the ranks (strong scaling), ReLU fused into the
epilogues of conv3/conv4; a step = the three layers.

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--sparsity S] [--config C2]
  python bench.py --impl reference ...   (the CPU oracle as the reference arm)
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N.  C2 etc.: weak
scaling, each rank its own 128 images (global image index, shard-independent
data); C5: the 1024-image batch is sharded.  No collective on the data path
(images are independent); NCCL only for barriers and max-over-ranks time.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1704_07724_b200 import datagen, shard  # noqa: E402

METRIC = "sparse conv dense-equiv GFLOP/s & nonzero-MAC/s at s=0.9/0.95/0.99; % roofline"
SM_COUNT = 148
FMA_PER_CLK_PER_SM = 128          # FP32 lanes per SM (B200), DESIGN.md "Kernels and their rooflines"
F_MAX_GHZ = 1.965                 # clocks.max.sm
FP32_PEAK_TFLOPS = SM_COUNT * FMA_PER_CLK_PER_SM * 2 * F_MAX_GHZ / 1e3   # 74.4
REPS = 20                         # launches per stage-timing graph


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def measured_traffic(variant_name):
    """Traffic figures of one gather launch from the committed ncu capture
    (profiles/gather_traffic.json): dict(traffic_bytes, dram_bytes, l2_write_bytes,
    l2_to_sm_bytes) or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "gather_traffic.json")) as f:
            t = json.load(f).get(variant_name)
    except OSError:
        return None
    return t if isinstance(t, dict) else None


def measured_fma_census(workload):
    """Hardware FFMA/FFMA2 census of the gather for `workload` ("C2 s=0.95") from the
    committed ncu run (profiles/r2_fma_census.json, tools/fma_census.py) or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_fma_census.json")) as f:
            rows = json.load(f)["workloads"]
    except (OSError, KeyError, ValueError):
        return None
    for r in rows:
        if r["workload"] == workload:
            return {k: r[k] for k in ("executed_lane_fmas", "exact_nonzero_macs", "dense_macs", "wasted_fma_factor",
                                      "skipped_vs_dense_exact", "skipped_vs_dense_executed")}
    return None


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
    """dense MACs, exact nonzero MACs and nnz of one batch
    (x: numpy or torch tensor; counted on its device)."""
    n = x.shape[0]
    dense = n * shp.ho * shp.wo * shp.r * shp.s * shp.k * (shp.c // shp.groups)
    ch = coverage(shp.h, shp.r, shp.stride, shp.pad, shp.ho)
    cw = coverage(shp.w, shp.s, shp.stride, shp.pad, shp.wo)
    if isinstance(x, np.ndarray):
        per_pos = (x != 0).sum(axis=(0, 1)).astype(np.int64)
        nnz = int(np.count_nonzero(x))
    else:
        per_pos = (x != 0).sum(dim=(0, 1)).cpu().numpy().astype(np.int64)
        nnz = int((x != 0).sum().item())
    exact = int((shp.k // shp.groups) * (ch[:, None] * cw[None, :] * per_pos).sum())
    return dense, exact, nnz


def algorithmic_bytes(shp, n, nnz, num_lists):
    """Two-stage minimum traffic: dense in + dense out + weights + bias
    + compacted lists written once and read once (8 B per entry: value + position,
    one marker per list, reading R9)."""
    dense_in = 4 * n * shp.c * shp.h * shp.w
    dense_out = 4 * n * shp.k * shp.ho * shp.wo
    wts = 4 * shp.k * (shp.c // shp.groups) * shp.r * shp.s + 4 * shp.k
    lists = 8 * (nnz + num_lists)
    return dense_in + dense_out + wts + 2 * lists


def roofline_times(exact, nbytes, hbm_gbs):
    t_fp32 = exact / (FP32_PEAK_TFLOPS / 2 * 1e12)
    t_hbm = nbytes / (hbm_gbs * 1e9)
    return t_fp32, t_hbm, max(t_fp32, t_hbm)


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
def workload_name(shp, s, n):
    return (f"{shp.name}: N={n}/GPU, {shp.c}x{shp.h}x{shp.w} -> {shp.k} {shp.r}x{shp.s} "
            f"stride {shp.stride} pad {shp.pad} groups {shp.groups}, s={s}")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def per_image_flops(shp):
    return 2 * shp.ho * shp.wo * shp.r * shp.s * shp.k * (shp.c // shp.groups)


def cpu_oracle_rate(layers, x_imgs, weights, min_s=10.0, max_s=30.0):
    """Time the fp64 oracle (as it stands) on host cores, one image at a time
    through every layer, until >= min_s.  Returns (dense-equiv GFLOP/s, images, s)."""
    import oracle  # the one product-side place the oracle may run (cpu_baseline leg)
    oracle.build()
    flops = sum(per_image_flops(shp) for shp in layers)
    t0 = time.perf_counter()
    done = 0
    while True:
        xi = x_imgs[done % x_imgs.shape[0]: done % x_imgs.shape[0] + 1]
        for li, shp in enumerate(layers):
            w, b = weights[li]
            y, _ = oracle.conv_fp64(xi, w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
            xi = np.maximum(y, 0.0).astype(np.float32) if li + 1 < len(layers) else None
        done += 1
        el = time.perf_counter() - t0
        if el >= min_s or el >= max_s:
            break
    el = time.perf_counter() - t0
    return flops * done / el / 1e9, done, el


C4_PAIR = (datagen.C4A, datagen.C4B)   # "C4": inception-3a 3x3 and 5x5 branches together


def default_sparsity(config):
    """Headline sparsity of a config (BASELINE.json): C1 s=0.9; C3 the per-channel
    recipe (R12); C2/C4a/C4b/C4 s=0.95 (the north star's s >= 0.95 bar)."""
    return {"C1": 0.9, "C3": "channel"}.get(config, 0.95)


def layers_for(config):
    if config == "C5":
        return list(datagen.C5_LAYERS), datagen.c5_weights(), datagen.C5_FIRST_SPARSITY
    shp = datagen.CONFIGS[config]
    return [shp], [datagen.weights(shp)], None


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, _ = shard.dist_env()
    if rank != 0:
        return 0
    layers, weights, s_first = layers_for(args.config)
    s = s_first if s_first is not None else args.sparsity
    if args.config == "C4":
        layers, weights = list(C4_PAIR), [datagen.weights(shp) for shp in C4_PAIR]
    import oracle
    oracle.build()
    flops_img = sum(per_image_flops(shp) for shp in layers)
    x = datagen.activations(layers[0], s, start=0, count=8)

    def one(xs):
        for li, shp in enumerate(layers):
            w, b = weights[li]
            y, _ = oracle.conv_fp64(xs, w, b, shp.stride, shp.pad, shp.groups, want_mass=False)
            xs = np.maximum(y, 0.0).astype(np.float32) if li + 1 < len(layers) else None

    t0 = time.perf_counter()
    one(x[:1])
    t1 = time.perf_counter() - t0
    m = int(max(1, min(8, 2.0 // max(t1, 1e-3))))   # ~1-2 s of CPU work per step
    xs = x[:m]
    for _ in range(args.warmup):
        one(xs)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one(xs)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = flops_img * m * len(times) / tot / 1e9
    n_img = layers[0].n
    sample = (f"{m} of the {n_img} images of the workload per step through "
              f"{'the 3-layer chain' if len(layers) > 1 else 'the layer'} (fp64 oracle, OpenMP), {args.steps} steps")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
            "higher_is_better": True, "scaling": "strong" if args.config == "C5" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(layers[0], s, n_img)},
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": host_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def graph_time_us(torch, stream, fn, reps=REPS):
    """Device time of fn from a CUDA graph of `reps` back-to-back calls."""
    with torch.cuda.stream(stream):
        fn()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
            for _ in range(reps):
                fn()
        g.replay()
        stream.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        b.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def rotating_time_us(torch, stream, fns, reps, prologue=False):
    """Average device time of one call when calls rotate over the input/output
    sets (fns[i] works on set i; the sets together exceed 2x L2, so every call
    starts L2-cold, as the timed step does).  One CUDA graph per set.  With
    prologue=True, fns[i]() runs a setup eagerly (e.g. stage 1 of set i before a
    stage-2 timing, as in the step) and returns the callable to time; the setup
    is re-run before every timed call, outside the events."""
    graphs = []
    with torch.cuda.stream(stream):
        for f in fns:
            timed = f() if prologue else f
            if not prologue:
                f()
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                timed()
            graphs.append(g)
        for g in graphs:                       # warm-up replays
            g.replay()
        stream.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if prologue:
            tot = 0.0
            for i in range(reps):
                fns[i % len(fns)]()
                a.record(stream)
                graphs[i % len(graphs)].replay()
                b.record(stream)
                b.synchronize()
                tot += a.elapsed_time(b)
            return tot * 1e3 / reps
        a.record(stream)
        for i in range(reps):
            graphs[i % len(graphs)].replay()
        b.record(stream)
        b.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def timed_steps(torch, stream, graphs, steps, warmup, ws, dev):
    """W untimed + K timed replays (rotating over graphs), barrier + sync on both
    sides, CUDA events on the launching stream, max over ranks."""
    with torch.cuda.stream(stream):
        for i in range(warmup):
            graphs[i % len(graphs)].replay()
        stream.synchronize()
        shard.barrier(ws)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            graphs[i % len(graphs)].replay()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize(dev)
    return shard.max_over_ranks(e0.elapsed_time(e1), ws, dev) / steps


PIPE_ROUND = 12  # batches per sparse_conv_forward_batches graph (at least; whole rounds of the sets)


def batch_graphs(torch, stream, conv, xs, outs, counts):
    """CUDA graphs of sparse_conv_forward_batches over c batches cycling through the sets,
    one per c in counts."""
    conv.reserve_batches()
    gs = {}
    with torch.cuda.stream(stream):
        for c in sorted(set(counts)):
            bx = [xs[i % len(xs)] for i in range(c)]
            bo = [outs[i % len(outs)] for i in range(c)]
            conv.forward_batches(bx, bo, stream=stream)
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                conv.forward_batches(bx, bo, stream=stream)
            gs[c] = g
    return gs


def pipe_round(nsets):
    return nsets * -(-PIPE_ROUND // nsets)


def timed_batches(torch, stream, gs, nsets, steps, warmup, ws, dev):
    """Like timed_steps, for pipelined steps: W untimed + K timed batches as replays of
    sparse_conv_forward_batches graphs of pipe_round(nsets) batches (a last shorter one for
    the remainder); each replay drains the pipeline at its end."""
    rnd = pipe_round(nsets)

    def seq(k):
        return [gs[rnd]] * (k // rnd) + ([gs[k % rnd]] if k % rnd else [])

    with torch.cuda.stream(stream):
        for g in seq(warmup):
            g.replay()
        stream.synchronize()
        shard.barrier(ws)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for g in seq(steps):
            g.replay()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize(dev)
    return shard.max_over_ranks(e0.elapsed_time(e1), ws, dev) / steps


def dense_two_stream_us(torch, stream, convs, xs, outs):
    """Dense path per batch with the same cross-batch overlap the sparse steps get: two plans
    (each its own channels-last workspace), batches alternating between two streams, one
    CUDA graph over pipe_round(len(xs)) batches cycling the rotating sets."""
    side = [torch.cuda.Stream(stream.device), torch.cuda.Stream(stream.device)]
    nb = pipe_round(len(xs))

    def run():
        for sd in side:
            sd.wait_stream(stream)
        for i in range(nb):
            convs[i % 2].dense_forward(xs[i % len(xs)], outs[i % len(outs)], stream=side[i % 2])
        for sd in side:
            stream.wait_stream(sd)

    return graph_time_us(torch, stream, run, reps=2) / nb


def run_single(args, torch, dev, ws, rank, sc):
    shp = datagen.CONFIGS[args.config]
    n = shp.n
    w, b = datagen.weights(shp)                     # same seed on every rank: replicated weights
    conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), n, shp.c, shp.h, shp.w,
                         shp.stride, shp.pad, shp.groups)
    lists_per_batch = n * conv.lists(1)["tiles"] * shp.c
    conv_d2 = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), n, shp.c, shp.h, shp.w,
                            shp.stride, shp.pad, shp.groups)  # second dense workspace (dense_two_stream_us)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    stream = torch.cuda.Stream(dev)
    # f3: measured crossover sparsity for this batch (before any capture)
    conv.s_star_calibrated = conv.calibrate_crossover(n, stream)

    def measure(s, steps, warmup):
        per_set = 4 * n * (shp.c * shp.h * shp.w + shp.k * shp.ho * shp.wo)
        nsets = max(2, -(-2 * max(l2_bytes, 126 * 2 ** 20) // per_set))
        xs, outs, counts = [], [], []
        for si in range(nsets):
            start = shard.image_start(si, rank, ws, n)   # global image index: shard-independent data
            xd = torch.from_numpy(datagen.activations(shp, s, start=start, count=n)).to(dev)
            counts.append(mac_counts(xd, shp))
            xs.append(xd)
            outs.append(torch.empty((n, shp.k, shp.ho, shp.wo), device=dev))
        graphs = []
        with torch.cuda.stream(stream):
            for si in range(nsets):
                conv.forward(xs[si], outs[si], stream=stream)
            stream.synchronize()
            for si in range(nsets):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
                    conv.forward(xs[si], outs[si], stream=stream)
                graphs.append(g)
        res = {"unpipelined_ms_per_step": timed_steps(torch, stream, graphs, steps, warmup, ws, dev)}
        del graphs
        if args.no_pipeline:
            res["ms_per_step"] = res["unpipelined_ms_per_step"]
        else:
            # the step as a user with a stream of batches runs it: sparse_conv_forward_batches
            # overlaps batch b+1's stage 1 (and first stage-2 wave) with batch b's last stage-2 wave
            rnd = pipe_round(nsets)
            gs = batch_graphs(torch, stream, conv, xs, outs, [rnd, steps % rnd or rnd, warmup % rnd or rnd])
            res["ms_per_step"] = timed_batches(torch, stream, gs, nsets, steps, warmup, ws, dev)
            del gs
        # per-stage and dense-path times on the same rotating sets as the step (cold L2, like the
        # step itself); the set-0 graph replays (L2-warm) are reported beside them, labelled
        rot = max(steps, 2 * nsets)
        res["compact_us"] = rotating_time_us(torch, stream, [lambda i=i: conv.compact(xs[i], stream=stream)
                                                             for i in range(nsets)], rot)
        def stage1_then_gather(i):
            conv.compact(xs[i], stream=stream)
            return lambda: conv.gather(n, outs[i], stream=stream)

        res["gather_us"] = rotating_time_us(torch, stream, [lambda i=i: stage1_then_gather(i) for i in range(nsets)],
                                            rot, prologue=True)
        res["dense_tc_us"] = rotating_time_us(torch, stream, [lambda i=i: conv.dense_forward(xs[i], outs[i],
                                                                                             stream=stream)
                                                              for i in range(nsets)], rot)
        res["dense_tc_2stream_us"] = dense_two_stream_us(torch, stream, [conv, conv_d2], xs, outs)
        res["compact_warm_us"] = graph_time_us(torch, stream, lambda: conv.compact(xs[0], stream=stream))
        res["gather_warm_us"] = graph_time_us(torch, stream, lambda: conv.gather(n, outs[0], stream=stream))
        res["dense_tc_warm_us"] = graph_time_us(torch, stream,
                                                lambda: conv.dense_forward(xs[0], outs[0], stream=stream), reps=5)
        # context only: the library convolution of torch (cuDNN), exact FP32 and TF32
        wd = torch.from_numpy(w).to(dev)
        bd = torch.from_numpy(b).to(dev)

        def cudnn(i, tf32):
            torch.backends.cudnn.allow_tf32 = tf32
            torch.nn.functional.conv2d(xs[i], wd, bd, stride=shp.stride, padding=shp.pad, groups=shp.groups)

        for tf32 in (False, True):
            torch.backends.cudnn.allow_tf32 = tf32
            res[f"cudnn_{'tf32' if tf32 else 'fp32'}_us"] = rotating_time_us(
                torch, stream, [lambda i=i, t=tf32: cudnn(i, t) for i in range(nsets)], rot)
        torch.backends.cudnn.allow_tf32 = True
        res["auto_us"] = rotating_time_us(torch, stream, [lambda i=i: conv.forward_auto(xs[i], outs[i],
                                                                                        stream=stream)
                                                          for i in range(nsets)], rot)
        res["auto_path"] = "sparse" if conv.last_path()[0] == sc.SC_PATH_SPARSE else "dense"
        dense = sum(c[0] for c in counts) / nsets
        exact = sum(c[1] for c in counts) / nsets
        nnz = sum(c[2] for c in counts) / nsets
        res.update(dense=dense, exact=exact, nnz=nnz, exact_set0=counts[0][1], nnz_set0=counts[0][2], nsets=nsets,
                   set_mib=nsets * per_set / 2 ** 20, realized_s=1 - nnz / (n * shp.c * shp.h * shp.w))
        return res

    return shp, n, conv, lists_per_batch, measure


def run_ours(args):
    import torch
    ws, rank, local = shard.dist_env()
    dev = shard.init(ws, local)
    from paper_1704_07724_b200 import sparseconv as sc

    peaks, peak_kind = measured_peaks()
    hbm_gbs = float(peaks.get("hbm_gbs", 6650.0))
    print(f"bench: rank {rank}/{ws} on {dev} ({torch.cuda.get_device_name(dev)})", file=sys.stderr, flush=True)
    if args.config == "C5":
        return run_chain(args, torch, dev, ws, rank, sc, hbm_gbs, peak_kind)
    if args.config == "C4":
        return run_pair(args, torch, dev, ws, rank, sc, hbm_gbs, peak_kind)
    shp, n, conv, lists_per_batch, measure = run_single(args, torch, dev, ws, rank, sc)
    s_head = args.sparsity
    clocks = ClockSampler(dev.index)
    with clocks:
        head = measure(s_head, args.steps, args.warmup)
        sweep = {}
        if not args.no_sweep:
            for s in datagen.CONFIG_SPARSITY[args.config]:
                if s != s_head:
                    sweep[s] = measure(s, max(args.steps, 20), max(args.warmup, 3))

    # --- end to end through the public API with host buffers (pinned) -------------
    xh = datagen.activations(shp, s_head, start=shard.image_start(0, rank, ws, n), count=n)
    h_in = torch.from_numpy(xh).pin_memory()
    h_out = torch.empty((n, shp.k, shp.ho, shp.wo)).pin_memory()
    # each call is synchronous (host buffers in, host buffers out): timed one by one on the host
    # clock, the median call is the figure (a mean over a few calls is at the mercy of host jitter)
    e2e_steps = max(5, min(args.steps, 30))
    for _ in range(3):
        conv.forward_host(h_in, h_out)
    shard.barrier(ws)
    e2e_calls = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        conv.forward_host(h_in, h_out)
        e2e_calls.append(time.perf_counter() - t0)
    e2e_mean = sum(e2e_calls) / len(e2e_calls)
    e2e_single = shard.max_over_ranks(sorted(e2e_calls)[len(e2e_calls) // 2], ws, dev)
    # a stream of batches end to end: sparse_conv_forward_host_batches over K batches per call
    # (three rotating pinned input / output sets; every batch's copies inside the call), host
    # clock around each synchronous call, median of 3 calls, per batch
    e2e_k = max(6, min(args.steps, 24))
    hb_in = [h_in] + [torch.from_numpy(datagen.activations(shp, s_head, start=shard.image_start(j, rank, ws, n),
                                                             count=n)).pin_memory() for j in (1, 2)]
    hb_out = [h_out] + [torch.empty((n, shp.k, shp.ho, shp.wo)).pin_memory() for _ in (1, 2)]
    seq_in = [hb_in[i % 3] for i in range(e2e_k)]
    seq_out = [hb_out[i % 3] for i in range(e2e_k)]
    conv.forward_host_batches(seq_in, seq_out)
    shard.barrier(ws)
    piped = []
    for _ in range(3):
        t0 = time.perf_counter()
        conv.forward_host_batches(seq_in, seq_out)
        piped.append((time.perf_counter() - t0) / e2e_k)
    e2e_s = shard.max_over_ranks(sorted(piped)[1], ws, dev)

    def gflops(dense, ms):
        return 2 * dense * ws / (ms * 1e-3) / 1e9

    def summary(r):
        nbytes = algorithmic_bytes(shp, n, r["nnz"], lists_per_batch)
        t_fp32, t_hbm, t_roof = roofline_times(r["exact"], nbytes, hbm_gbs)
        return nbytes, t_fp32, t_hbm, t_roof

    v = head
    value = gflops(v["dense"], v["ms_per_step"])
    nbytes, t_fp32, t_hbm, t_roof = summary(v)
    # exact MACs averaged over the rotating sets, like the kernel time
    achieved = 2 * v["exact"] / (v["gather_us"] * 1e-6) / 1e12
    vname = conv.variant[1]
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(v["ms_per_step"], 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(shp, s_head, n), "global_batch": n * ws, "parallelism": f"dp{ws}",
                   **shared_gpu_note(ws),
                   "l2": f"{v['nsets']} rotating input/output sets ({v['set_mib']:.0f} MiB > 2x L2)",
                   "timing": ("CUDA events around K CUDA-graph replays (one sparse_conv_forward each), max over ranks"
                              if args.no_pipeline else
                              "CUDA events around K batches run as CUDA-graph replays of sparse_conv_forward_batches "
                              f"of {pipe_round(v['nsets'])} batches cycling the {v['nsets']} rotating sets "
                              "(batch b+1's stage 1 overlaps batch b's "
                              "stage 2; every batch's output identical to sparse_conv_forward), max over ranks"),
                   "realized_sparsity": round(v["realized_s"], 5), "variant": vname},
        "pipelined": not args.no_pipeline,
        "unpipelined_ms_per_step": round(v["unpipelined_ms_per_step"], 5),
        "unpipelined_value": round(gflops(v["dense"], v["unpipelined_ms_per_step"]), 2),
        "nonzero_mac_per_s": round(v["exact"] * ws / (v["ms_per_step"] * 1e-3), 1),
        "pct_roofline": round(100 * t_roof / (v["ms_per_step"] * 1e-3), 2),
        "roofline_step": {"t_roof_us": round(t_roof * 1e6, 3), "t_fp32_us": round(t_fp32 * 1e6, 3),
                          "t_hbm_us": round(t_hbm * 1e6, 3), "bytes": int(nbytes),
                          "exact_nonzero_macs": int(v["exact"]), "dense_macs": int(v["dense"])},
        "roofline": {"kernel": f"gather (stage 2, {vname})", "bound": "alu", "achieved": round(achieved, 3),
                     "peak": round(FP32_PEAK_TFLOPS, 2), "unit": "TFLOP/s",
                     "frac": round(achieved / FP32_PEAK_TFLOPS, 4),
                     "traffic": (measured_traffic(vname) or {}).get("traffic_bytes"),
                     "traffic_detail": measured_traffic(vname),
                     "per_launch": "2 x exact nonzero MACs of one 128-image batch (mean over the rotating sets)",
                     "peak_note": "FP32 FMA: 148 SMs x 128 lanes x 2 flop x 1.965 GHz (unit counts x max clock)"},
        "fma_census": measured_fma_census(f"{args.config} s={s_head}"),
        "wasted_fma_factor": (measured_fma_census(f"{args.config} s={s_head}") or {}).get("wasted_fma_factor"),
        "stages_us": {"compact": round(v["compact_us"], 3), "gather": round(v["gather_us"], 3),
                      "compact_l2_warm": round(v["compact_warm_us"], 3), "gather_l2_warm": round(v["gather_warm_us"], 3),
                      "note": "compact/gather: rotating sets (L2-cold, as the step); *_l2_warm: set-0 graph replays"},
        "compact_hbm": {"achieved_gbs": round(4 * n * shp.c * shp.h * shp.w / (v["compact_us"] * 1e-6) / 1e9, 1),
                        "peak_gbs": hbm_gbs, "peak_kind": peak_kind},
        "dense_tc": {"us": round(v["dense_tc_us"], 3), "l2_warm_us": round(v["dense_tc_warm_us"], 3),
                     "gflops": round(gflops(v["dense"], v["dense_tc_us"] / 1e3), 2),
                     "sparse_speedup": round(v["dense_tc_us"] / (v["ms_per_step"] * 1e3), 3),
                     "two_stream_us": round(v["dense_tc_2stream_us"], 3),
                     "sparse_speedup_vs_two_stream": round(v["dense_tc_2stream_us"] / (v["ms_per_step"] * 1e3), 3),
                     "note": "in-library tcgen05 TF32 implicit-GEMM conv (dense_conv_forward) on the same batch, "
                             "same rotating sets (L2-cold) as the sparse step; us: back to back on one stream; "
                             "two_stream_us: per batch with batches alternating between two streams and two plans "
                             "(the cross-batch overlap the pipelined sparse steps get)"},
        "cudnn_context": {"fp32_us": round(v["cudnn_fp32_us"], 3), "tf32_us": round(v["cudnn_tf32_us"], 3),
                          "note": "torch.nn.functional.conv2d (cuDNN) on the same rotating sets; context only, not "
                                  "part of the library"},
        "sweep": {str(s): {"value": round(gflops(r["dense"], r["ms_per_step"]), 2),
                           "nonzero_mac_per_s": round(r["exact"] * ws / (r["ms_per_step"] * 1e-3), 1),
                           "ms_per_step": round(r["ms_per_step"], 5),
                           "unpipelined_ms_per_step": round(r["unpipelined_ms_per_step"], 5),
                           "pct_roofline": round(100 * summary(r)[3] / (r["ms_per_step"] * 1e-3), 2),
                           "gather_frac_fp32": round(2 * r["exact"] / (r["gather_us"] * 1e-6) / 1e12
                                                     / FP32_PEAK_TFLOPS, 4),
                           "gather_us": round(r["gather_us"], 3), "compact_us": round(r["compact_us"], 3),
                           "dense_tc_speedup": round(r["dense_tc_us"] / (r["ms_per_step"] * 1e3), 3),
                           "dense_tc_two_stream_speedup": round(r["dense_tc_2stream_us"] / (r["ms_per_step"] * 1e3), 3),
                           "auto_us": round(r["auto_us"], 3), "auto_path": r["auto_path"]}
                  for s, r in sweep.items()},
        "crossover": {"s_star": round(conv.s_star_calibrated, 4), "auto_us": round(v["auto_us"], 3),
                      "auto_path": v["auto_path"],
                      "note": "sparse_conv_forward_auto: device-side nnz count picks sparse iff s >= s*; s* "
                              "calibrated by sparse_conv_calibrate_crossover for this batch (SURVEY 8f row f3)"},
        "e2e": {"value": round(gflops(v["dense"], e2e_s * 1e3), 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(h_in.numel() * 4), "d2h_bytes_per_step": int(h_out.numel() * 4),
                "ms_per_step": round(e2e_s * 1e3, 4), "batches_per_call": e2e_k,
                "statistic": "per batch: host clock around a synchronous call of K batches, median of 3 calls, max over "
                             "ranks",
                "api": "sparse_conv_forward_host_batches (pinned host buffers; each batch copied in and its result "
                       "copied out inside the call)",
                "single_call": {"value": round(gflops(v["dense"], e2e_single * 1e3), 2),
                                "ms_per_step": round(e2e_single * 1e3, 4), "ms_mean": round(e2e_mean * 1e3, 4),
                                "calls": e2e_steps, "statistic": "median call, host clock, max over ranks",
                                "api": "sparse_conv_forward_host"}},
        "gpu_launches": int(args.steps * conv.launch_counts[0]),
        "clocks": clocks.summary(),
    }
    # the gather also against the in-run FP32 pipe probe and the observed clock
    try:
        probe = {"ffma_lane_fma_per_clk_sm": round(sc.probe_fma(0), 2),
                 "ffma2_lane_fma_per_clk_sm": round(sc.probe_fma(1), 2)}
        mhz = line["clocks"].get("sm_mhz") or F_MAX_GHZ * 1e3
        best = max(probe.values())
        peak_probe = SM_COUNT * best * 2 * mhz * 1e6 / 1e12
        probe.update(clock_mhz=mhz, peak_tflops=round(peak_probe, 2), frac=round(achieved / peak_probe, 4),
                     note="peak = 148 SMs x the best probed lane-FMA/clk x 2 flop x the median SM clock seen")
        line["roofline"]["vs_probe"] = probe
    except Exception as exc:  # the probe is context only
        line["roofline"]["vs_probe"] = {"error": str(exc)[:120]}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, imgs, secs = cpu_oracle_rate([shp], datagen.activations(shp, s_head, start=0, count=min(n, 16)),
                                           [datagen.weights(shp)])
        line["cpu_baseline"] = {"value": round(rate, 3), "unit": "GFLOP/s", "cores": host_cores(), "kind": "oracle",
                                "sample": f"{imgs} single-image oracle calls over images 0..15 of the workload "
                                          f"({secs:.1f} s, fp64 7-loop, OpenMP)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    shard.finalize(ws)
    return 0


def run_chain(args, torch, dev, ws, rank, sc, hbm_gbs, peak_kind):
    """C5: conv3 -> ReLU -> conv4 -> ReLU -> conv5 on this rank's share of 1024 images."""
    layers, weights, s_first = layers_for("C5")
    n_total = layers[0].n
    lo, hi = shard.shard_range(n_total, rank, ws)
    n = hi - lo
    convs = []
    for li, shp in enumerate(layers):
        w, b = weights[li]
        convs.append(sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), n, shp.c, shp.h,
                                   shp.w, shp.stride, shp.pad, shp.groups, fuse_relu=li + 1 < len(layers)))
    x0 = torch.from_numpy(datagen.activations(layers[0], s_first, start=lo, count=n)).to(dev)
    bufs = [x0] + [torch.empty((n, shp.k, shp.ho, shp.wo), device=dev) for shp in layers]
    stream = torch.cuda.Stream(dev)

    outs_fused = [None] * (len(convs) - 1) + [bufs[-1]]

    def step():  # one sparse_conv_forward_chain: intermediate layers emit the next stage-1 lists (f1)
        sc.chain_forward(convs, bufs[0], outs_fused, stream=stream)

    with torch.cuda.stream(stream):  # materialise the intermediate activations once (sparsity report)
        for li, conv in enumerate(convs):
            conv.forward(bufs[li], bufs[li + 1], stream=stream)
        stream.synchronize()

    with torch.cuda.stream(stream):
        step()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
            step()
    counts = [mac_counts(bufs[li], shp) for li, shp in enumerate(layers)]   # realized per-layer inputs
    clocks = ClockSampler(dev.index)
    with clocks:
        ms = timed_steps(torch, stream, [g], args.steps, args.warmup, ws, dev)
        layer_us = [graph_time_us(torch, stream, (lambda c=conv, a=bufs[li], o=bufs[li + 1]:
                                                  c.forward(a, o, stream=stream)), reps=5)
                    for li, conv in enumerate(convs)]
    dense = sum(c[0] for c in counts)
    exact = sum(c[1] for c in counts)
    nbytes = sum(algorithmic_bytes(shp, n, counts[li][2], n * convs[li].lists(1)["tiles"] * shp.c)
                 for li, shp in enumerate(layers))
    t_fp32, t_hbm, t_roof = roofline_times(exact, nbytes, hbm_gbs)
    total_dense = shard.sum_over_ranks(dense, ws, dev)
    total_exact = shard.sum_over_ranks(exact, ws, dev)
    value = 2 * total_dense / (ms * 1e-3) / 1e9
    # e2e through the public API with host buffers: layer by layer, activations stay on the device
    h_in = torch.from_numpy(x0.cpu().numpy()).pin_memory()
    h_out = torch.empty(tuple(bufs[-1].shape)).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))

    def e2e_step():
        bufs[0].copy_(h_in, non_blocking=True)
        step()
        h_out.copy_(bufs[-1], non_blocking=True)
        torch.cuda.synchronize(dev)

    with torch.cuda.stream(stream):
        e2e_step()
        shard.barrier(ws)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = shard.max_over_ranks((time.perf_counter() - t0) / e2e_steps, ws, dev)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"c5 chain conv3->conv4->conv5, N={n_total} total ({n}/GPU), first input s={s_first}",
                   "global_batch": n_total, "parallelism": f"dp{ws}", **shared_gpu_note(ws),
                   "l2": "inputs larger than L2 (177 MB/GPU at N=1)",
                   "timing": "CUDA events around K graph replays of sparse_conv_forward_chain (intermediate layers "
                             "emit the next layer's stage-1 lists, no dense intermediates), max over ranks",
                   "layer_input_sparsity": [round(1 - c[2] / (n * shp.c * shp.h * shp.w), 4)
                                            for c, shp in zip(counts, layers)],
                   "variants": [c.variant[1] for c in convs]},
        "nonzero_mac_per_s": round(total_exact / (ms * 1e-3), 1),
        "pct_roofline": round(100 * t_roof / (ms * 1e-3), 2),
        "layers_unfused_us": [round(t, 2) for t in layer_us],
        "e2e": {"value": round(2 * total_dense / e2e_s / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(h_in.numel() * 4), "d2h_bytes_per_step": int(h_out.numel() * 4),
                "ms_per_step": round(e2e_s * 1e3, 4)},
        "gpu_launches": int(args.steps * sum(c.launch_counts[0] for c in convs)),  # 3 per layer either way
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    shard.finalize(ws)
    return 0


def run_pair(args, torch, dev, ws, rank, sc, hbm_gbs, peak_kind):
    """C4 = C4a + C4b (inception-3a 3x3 and 5x5 branches, BASELINE.json configs[3]) run
    together on two streams, as SURVEY 8d asks: a step = both sparse forwards on this
    rank's 128 images, forked from and joined into one stream, one CUDA graph per
    rotating input set (weak scaling over ranks)."""
    s = args.sparsity
    shps = C4_PAIR
    n = shps[0].n
    convs = []
    for shp in shps:
        w, b = datagen.weights(shp)
        convs.append(sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), n, shp.c, shp.h, shp.w,
                                   shp.stride, shp.pad, shp.groups))
    main = torch.cuda.Stream(dev)
    side = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    per_set = sum(4 * n * (shp.c * shp.h * shp.w + shp.k * shp.ho * shp.wo) for shp in shps)
    nsets = max(2, -(-2 * max(l2_bytes, 126 * 2 ** 20) // per_set))
    xs, outs, counts = [], [], []
    for si in range(nsets):
        start = shard.image_start(si, rank, ws, n)
        xs.append([torch.from_numpy(datagen.activations(shp, s, start=start, count=n)).to(dev) for shp in shps])
        outs.append([torch.empty((n, shp.k, shp.ho, shp.wo), device=dev) for shp in shps])
        counts.append([mac_counts(x, shp) for x, shp in zip(xs[-1], shps)])

    def step(si):  # fork both layers off `main`, join back
        ev = torch.cuda.Event()
        ev.record(main)
        for j in range(2):
            side[j].wait_event(ev)
            convs[j].forward(xs[si][j], outs[si][j], stream=side[j])
            done = torch.cuda.Event()
            done.record(side[j])
            main.wait_event(done)

    graphs = []
    with torch.cuda.stream(main):
        for si in range(nsets):
            step(si)
        main.synchronize()
        for si in range(nsets):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=main, capture_error_mode="relaxed"):
                step(si)
            graphs.append(g)
    gs = {}
    if not args.no_pipeline:
        # pipelined steps: each layer's batches through sparse_conv_forward_batches on its stream
        def rounds(c):
            ev = torch.cuda.Event()
            ev.record(main)
            for j in range(2):
                side[j].wait_event(ev)
                convs[j].forward_batches([xs[i % nsets][j] for i in range(c)], [outs[i % nsets][j] for i in range(c)],
                                         stream=side[j])
                done = torch.cuda.Event()
                done.record(side[j])
                main.wait_event(done)

        for c in convs:
            c.reserve_batches()
        rnd = pipe_round(nsets)
        with torch.cuda.stream(main):
            for c in sorted({rnd, args.steps % rnd or rnd, args.warmup % rnd or rnd}):
                rounds(c)
                main.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=main, capture_error_mode="relaxed"):
                    rounds(c)
                gs[c] = g
    clocks = ClockSampler(dev.index)
    with clocks:
        ms_unpiped = timed_steps(torch, main, graphs, args.steps, args.warmup, ws, dev)
        ms = ms_unpiped if args.no_pipeline else timed_batches(torch, main, gs, nsets, args.steps, args.warmup, ws, dev)
        alone = [rotating_time_us(torch, main, [lambda i=i, j=j: convs[j].forward(xs[i][j], outs[i][j], stream=main)
                                               for i in range(nsets)], max(args.steps, 2 * nsets))
                 for j in range(2)]
        dense_alone = [rotating_time_us(torch, main, [lambda i=i, j=j: convs[j].dense_forward(xs[i][j], outs[i][j],
                                                                                             stream=main)
                                                     for i in range(nsets)], max(args.steps, 2 * nsets))
                       for j in range(2)]
    del graphs, gs
    dense = sum(c[0] for cs in counts for c in cs) / nsets
    exact = sum(c[1] for cs in counts for c in cs) / nsets
    nbytes = sum(algorithmic_bytes(shp, n, sum(cs[j][2] for cs in counts) / nsets,
                                   n * convs[j].lists(1)["tiles"] * shp.c) for j, shp in enumerate(shps))
    t_fp32, t_hbm, t_roof = roofline_times(exact, nbytes, hbm_gbs)
    value = 2 * dense * ws / (ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"C4 = C4a + C4b on two streams: {workload_name(shps[0], s, n)}; "
                               f"{workload_name(shps[1], s, n)}",
                   "global_batch": n * ws, "parallelism": f"dp{ws}", **shared_gpu_note(ws),
                   "l2": f"{nsets} rotating input/output sets ({nsets * per_set / 2 ** 20:.0f} MiB > 2x L2)",
                   "timing": ("CUDA events around K graph replays (both layers forked onto two streams), max over ranks"
                              if args.no_pipeline else
                              f"CUDA events around K batches as CUDA-graph replays of {pipe_round(nsets)} batches: both "
                              "layers forked onto two streams, each through sparse_conv_forward_batches (batch b+1's "
                              "stage 1 overlaps batch b's stage 2), max over ranks"),
                   "variants": [c.variant[1] for c in convs]},
        "pipelined": not args.no_pipeline,
        "unpipelined_ms_per_step": round(ms_unpiped, 5),
        "nonzero_mac_per_s": round(exact * ws / (ms * 1e-3), 1),
        "pct_roofline": round(100 * t_roof / (ms * 1e-3), 2),
        "roofline_step": {"t_roof_us": round(t_roof * 1e6, 3), "t_fp32_us": round(t_fp32 * 1e6, 3),
                          "t_hbm_us": round(t_hbm * 1e6, 3), "bytes": int(nbytes), "bound": "hbm" if t_hbm > t_fp32
                          else "alu", "exact_nonzero_macs": int(exact), "dense_macs": int(dense)},
        "layers_alone_us": {"C4a": round(alone[0], 2), "C4b": round(alone[1], 2)},
        "dense_tc": {"us_sequential": round(sum(dense_alone), 3), "C4a_us": round(dense_alone[0], 2),
                     "C4b_us": round(dense_alone[1], 2),
                     "sparse_speedup": round(sum(dense_alone) / (ms * 1e3), 3),
                     "note": "in-library tcgen05 TF32 dense conv of both layers back to back, same rotating sets"},
        "gpu_launches": int(args.steps * sum(c.launch_counts[0] for c in convs)),
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    shard.finalize(ws)
    return 0


# Paper Table 3: Xeon E5-2630v4 CPU, Caffe+MKL GEMM vs ISC, ms and printed speedup.
# Context only (another machine, batch size unstated).
PAPER_TABLE3 = {"LeNet-Conv2": (0.854, 0.123, 6.96), "AlexNetC-Conv3": (0.329, 0.122, 2.69),
                "AlexNetI-Conv4": (4.874, 1.660, 2.94), "GoogLeNet-Inception4a.1": (1.795, 1.292, 1.39),
                "GoogLeNet-Inception4a.2": (0.943, 0.558, 1.69), "GoogLeNet-Inception4e.3": (7.602, 4.782, 1.59),
                "GoogLeNet-Inception5a.1": (1.912, 0.645, 2.97), "GoogLeNet-Inception5a.2": (0.742, 0.258, 2.87),
                "GoogLeNet-Inception5b.3": (4.410, 0.931, 4.74), "GoogLeNet-Inception5b.5": (1.560, 0.220, 7.11)}


def run_table2(args):
    """B200 analogue of the paper's Table 3: every Table 2 layer
     at its printed sparsity, N=128 synthetic images: the sparse
    forward (both stages) vs the in-library tcgen05 dense convolution, device
    times from CUDA graphs of back-to-back launches."""
    import torch
    from paper_1704_07724_b200 import sparseconv as sc
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    rows = []
    for shp, s in datagen.table2_shapes(n=args.table2_batch):
        x = torch.from_numpy(datagen.activations(shp, s)).to(dev)
        w, b = datagen.weights(shp)
        conv = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h, shp.w,
                             shp.stride, shp.pad, shp.groups)
        out = torch.empty((shp.n,) + conv.out_shape, device=dev)
        t_s = graph_time_us(torch, stream, lambda: conv.forward(x, out, stream=stream))
        # a stream of batches through sparse_conv_forward_batches (12 per call; batches b and b+2
        # share a stage-2 stream, so two output buffers)
        out2 = torch.empty_like(out)
        conv.reserve_batches()
        t_p = graph_time_us(torch, stream, lambda: conv.forward_batches([x] * 12, [out, out2] * 6, stream=stream),
                            reps=3) / 12
        try:
            t_d = graph_time_us(torch, stream, lambda: conv.dense_forward(x, out, stream=stream), reps=5)
            # the dense path given the same cross-batch overlap: a second plan (its own channels-last
            # workspace), batches alternating between two streams
            conv2 = sc.SparseConv(torch.from_numpy(w).to(dev), torch.from_numpy(b).to(dev), shp.n, shp.c, shp.h,
                                  shp.w, shp.stride, shp.pad, shp.groups)
            side = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

            def dense_2s():
                for sd in side:
                    sd.wait_stream(stream)
                for i in range(12):
                    (conv, conv2)[i % 2].dense_forward(x, (out, out2)[i % 2], stream=side[i % 2])
                for sd in side:
                    stream.wait_stream(sd)

            t_d2 = graph_time_us(torch, stream, dense_2s, reps=3) / 12
            del conv2
        except sc.SparseConvError:
            t_d = t_d2 = None
        s_star = conv.calibrate_crossover(shp.n, stream)
        t_a = graph_time_us(torch, stream, lambda: conv.forward_auto(x, out, stream=stream), reps=5)
        path = "sparse" if conv.last_path()[0] == sc.SC_PATH_SPARSE else "dense"
        dense, exact, nnz = mac_counts(x, shp)
        cpu = PAPER_TABLE3.get(shp.name)
        rows.append({"layer": shp.name, "shape": f"{shp.c}x{shp.h}x{shp.w}->{shp.k} {shp.r}x{shp.s} p{shp.pad} "
                                                 f"t{shp.stride}", "s": s, "variant": conv.variant[1],
                     "sparse_us": round(t_s, 2), "sparse_pipelined_us": round(t_p, 2),
                     "dense_tc_us": None if t_d is None else round(t_d, 2),
                     "b200_speedup_sparse_over_dense": None if t_d is None else round(t_d / t_s, 3),
                     "dense_tc_2stream_us": None if t_d2 is None else round(t_d2, 2),
                     "b200_speedup_pipelined": None if t_d2 is None else round(min(t_d, t_d2) / t_p, 3),
                     "s_star": round(s_star, 4), "auto_us": round(t_a, 2), "auto_path": path,
                     "sparse_frac_fp32": round(2 * exact / (t_s * 1e-6) / 1e12 / FP32_PEAK_TFLOPS, 4),
                     "paper_cpu_gemm_ms": cpu[0] if cpu else None, "paper_cpu_isc_ms": cpu[1] if cpu else None,
                     "paper_cpu_speedup": cpu[2] if cpu else None})
    print(json.dumps({"table2": rows, "batch": args.table2_batch, "data": "synthetic",
                      "note": "paper_cpu_* from PAPER.md Table 3 (Xeon E5-2630v4), context only"}), flush=True)
    return 0


def run_backward(args):
    """sparse_conv_backward (plane lists + wgrad + split reduce + dbias +
    ReLU-masked dgrad) on the workload's batch at several sparsities, graph-timed, with
    the library dense backward (cuDNN via torch autograd, TF32 allowed and not) as context."""
    import torch
    from paper_1704_07724_b200 import sparseconv as sc
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    shp = datagen.CONFIGS[args.config]
    n = shp.n
    w, b = datagen.weights(shp)
    wd = torch.from_numpy(w).to(dev)
    conv = sc.SparseConv(wd, torch.from_numpy(b).to(dev), n, shp.c, shp.h, shp.w, shp.stride, shp.pad, shp.groups)
    d = torch.from_numpy(np.random.default_rng(31).standard_normal((n, shp.k, shp.ho, shp.wo)).astype(np.float32))
    d = d.to(dev)
    out_dw = torch.empty_like(wd)
    out_db = torch.empty(shp.k, device=dev)
    out_dz = torch.empty((n, shp.c, shp.h, shp.w), device=dev)
    L = sc.lib()
    def ptr(t):
        return None if t is None else ctypes.c_void_p(t.data_ptr())

    def bwd(x, dw=out_dw, db=out_db, dz=out_dz):
        sc._check(L.sparse_conv_backward(conv._plan, n, ptr(x), ptr(d), ptr(dw), ptr(db), ptr(dz),
                                         sc._stream_handle(stream)))

    def cudnn(x, tf32):
        torch.backends.cudnn.allow_tf32 = tf32
        xr = x.clone().requires_grad_(True)
        wr = wd.clone().requires_grad_(True)
        br = torch.zeros(shp.k, device=dev, requires_grad=True)
        with torch.cuda.stream(stream):
            for _ in range(3):
                o = torch.nn.functional.conv2d(xr, wr, br, stride=shp.stride, padding=shp.pad, groups=shp.groups)
                o.backward(d)
            stream.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                o = torch.nn.functional.conv2d(xr, wr, br, stride=shp.stride, padding=shp.pad, groups=shp.groups)
                o.backward(d)
            e.record(stream)
            e.synchronize()
        return a.elapsed_time(e) * 1e3 / 10  # includes the forward: an upper bound on the backward alone

    rows = {}
    for s in (0.9, 0.95, 0.99):
        x = torch.from_numpy(datagen.activations(shp, s)).to(dev)
        dense, exact, nnz = mac_counts(x, shp)
        t_all = graph_time_us(torch, stream, lambda: bwd(x), reps=10)
        t_w = graph_time_us(torch, stream, lambda: bwd(x, db=None, dz=None), reps=10)
        t_z = graph_time_us(torch, stream, lambda: bwd(x, dw=None, db=None), reps=10)
        flops = 2 * 2 * exact  # wgrad and dgrad each run the exact nonzero MACs
        rows[str(s)] = {"us": round(t_all, 2), "wgrad_us": round(t_w, 2), "dgrad_us": round(t_z, 2),
                        "nonzero_tflops": round(flops / (t_all * 1e-6) / 1e12, 3),
                        "frac_fp32": round(flops / (t_all * 1e-6) / 1e12 / FP32_PEAK_TFLOPS, 4),
                        "cudnn_fwd_bwd_tf32_us": round(cudnn(x, True), 2),
                        "cudnn_fwd_bwd_fp32_us": round(cudnn(x, False), 2)}
    torch.backends.cudnn.allow_tf32 = True
    print(json.dumps({"backward": rows, "workload": workload_name(shp, args.sparsity, n), "data": "synthetic",
                      "note": "sparse_conv_backward (dw, dbias, ReLU-masked dz) graph-timed, L2-warm; cudnn_* = "
                              "torch conv2d forward+backward (dw, db, dx) per step, context only"}), flush=True)
    return 0


def shared_gpu_note(ws):
    """config entries of a run whose ranks share GPUs (SC_DIST_BACKEND=gloo, shard.shares_gpus)."""
    import torch
    if ws > 1 and shard.shares_gpus():
        return {"functional_only": f"{ws} ranks on {torch.cuda.device_count()} GPU(s) over gloo: a check of the "
                                   "multi-rank path (launch, process group, shard, barriers, max over ranks), "
                                   "not a scaling measurement"}
    return {}


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` with N > 1 outside torchrun: start N ranks on this node
    (one process per GPU, NCCL over 127.0.0.1) with the same arguments; rank 0
    prints the line.  Returns the launcher's exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench: launching {args.gpus} ranks: {' '.join(cmd[1:])}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def run_stub(args):
    """CPU stand-in for the GPU arm (tests only: `--cpu-stub`, gloo): the same rank
    orchestration -- shard by image (C5: the 1024-image batch split over ranks;
    others: each rank its own batch), W untimed + K timed steps between barriers,
    max over ranks of the elapsed time, one JSON line from rank 0 -- around a stub
    step (a nonzero count of the rank's images: no arithmetic of the method)."""
    import torch.distributed as dist
    ws, rank, _ = shard.dist_env()
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("gloo")
    layers, _, s_first = layers_for(args.config if args.config != "C4" else "C4a")
    s = s_first if s_first is not None else args.sparsity
    shp = layers[0]
    if args.config == "C5":
        lo, hi = shard.shard_range(shp.n, rank, ws)
        scaling, global_batch = "strong", shp.n
    else:
        lo = shard.image_start(0, rank, ws, shp.n)
        hi = lo + shp.n
        scaling, global_batch = "weak", shp.n * ws
    x = datagen.activations(shp, s, start=lo, count=min(hi - lo, 8))   # a bounded slice: orchestration only

    def step():
        return int(np.count_nonzero(x))

    for _ in range(args.warmup):
        step()
    shard.barrier(ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = shard.max_over_ranks(time.perf_counter() - t0, ws)
    images = shard.sum_over_ranks(hi - lo, ws)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": round(images * args.steps / el, 3), "unit": "stub images/s",
                          "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(1e3 * el / args.steps, 5), "higher_is_better": True,
                          "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                          "stub": "cpu orchestration test (no GPU work; not a benchmark number)",
                          "config": {"workload": args.config, "global_batch": global_batch,
                                     "images_per_step": int(images), "parallelism": f"dp{ws}"}}), flush=True)
    shard.finalize(ws)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(datagen.CONFIGS) + ["C4", "C5"])
    ap.add_argument("--sparsity", default=None,
                    help="input sparsity (default per config: C1 0.9, C3 'channel', else 0.95)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="time each step as one sparse_conv_forward (no overlap across batches)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--table2", action="store_true", help="paper Table 2 layers: sparse vs dense on B200")
    ap.add_argument("--table2-batch", type=int, default=128)
    ap.add_argument("--backward", action="store_true", help="f4: sparse backward vs library dense backward")
    ap.add_argument("--cpu-stub", action="store_true", help=argparse.SUPPRESS)   # tests: orchestration on CPU
    args = ap.parse_args()
    if args.sparsity is None:
        args.sparsity = default_sparsity(args.config)
    elif args.sparsity != "channel":
        args.sparsity = float(args.sparsity)
    ws_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and ws_env is None:
        return relaunch_under_torchrun(args)
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench: WORLD_SIZE={ws_env} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.backward:
        return run_backward(args)
    if args.table2:
        return run_table2(args)
    if args.warmup < 3:
        args.warmup = 3
    if args.cpu_stub:
        return run_stub(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
