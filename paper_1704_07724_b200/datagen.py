"""Seeded synthetic inputs for the five BASELINE.json configs and the paper's
Table 2 shapes.

This module holds NO arithmetic of the method: it only draws random numbers.
It is the one module both the oracle side (tests) and the product side
(bench, tests) use.  Recipe (reading R16):

* Counter-based streams: every tensor slice is drawn from
  ``np.random.SeedSequence([seed, config_id, tensor_id, index])`` so an image's
  data does not depend on which rank generates it or on the batch split.
* Activations (stand-in for ReLU outputs): i.i.d. mask
  ``u >= s`` (Bernoulli(1-s) nonzero) times ``|N(0,1)|`` values.
* Weights and bias: ``N(0, 0.01^2)``.
* C3: per-channel sparsity ``s_c ~ U(0.85, 0.99)`` shared by all images, and
  ``round(0.05*C)`` fully-zero ("dead") channels picked by a seeded permutation
  (R12).
* C5 chain: the first input at s=0.95; later inputs are ReLU of the previous
  layer's output (computed by whoever runs the chain, not here); biases of
  conv3/conv4 are shifted by the constants in ``c5_bias_shift.json`` written by
  ``tools/calibrate_c5.py`` (R13).

Since MNIST/CIFAR/ImageNet activations and trained weights are not available,
these synthetic tensors stand in for the paper's workloads.
"""
from __future__ import annotations

import dataclasses
import hashlib
import json
import os

import numpy as np

# tensor ids inside a config's seed space
T_INPUT, T_WEIGHT, T_BIAS, T_CHANNEL = 0, 1, 2, 3


@dataclasses.dataclass(frozen=True)
class ConvShape:
    name: str
    config_id: int
    n: int
    c: int
    h: int
    w: int
    k: int
    r: int
    s: int
    stride: int = 1
    pad: int = 0
    groups: int = 1

    @property
    def ho(self):
        return (self.h + 2 * self.pad - self.r) // self.stride + 1

    @property
    def wo(self):
        return (self.w + 2 * self.pad - self.s) // self.stride + 1

    def with_batch(self, n):
        return dataclasses.replace(self, n=n)


# BASELINE.json configs[0..4]
C1 = ConvShape("lenet_conv2", 1, 64, 20, 12, 12, 50, 5, 5, 1, 0, 1)
C2 = ConvShape("alexnet_conv3", 2, 128, 256, 13, 13, 384, 3, 3, 1, 1, 1)
C3 = ConvShape("alexnet_conv2_g2", 3, 128, 96, 27, 27, 256, 5, 5, 1, 2, 2)
C4A = ConvShape("inception3a_3x3", 4, 128, 96, 28, 28, 128, 3, 3, 1, 1, 1)
C4B = ConvShape("inception3a_5x5", 5, 128, 16, 28, 28, 32, 5, 5, 1, 2, 1)
C5_LAYERS = (
    ConvShape("c5_conv3", 6, 1024, 256, 13, 13, 384, 3, 3, 1, 1, 1),
    ConvShape("c5_conv4", 7, 1024, 384, 13, 13, 384, 3, 3, 1, 1, 1),
    ConvShape("c5_conv5", 8, 1024, 384, 13, 13, 256, 3, 3, 1, 1, 1),
)
CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4a": C4A, "C4b": C4B}
CONFIG_SPARSITY = {"C1": (0.9,), "C2": (0.9, 0.95, 0.99), "C3": ("channel",),
                   "C4a": (0.9, 0.95, 0.99), "C4b": (0.9, 0.95, 0.99)}
C5_FIRST_SPARSITY = 0.95


def table2_shapes(n=1):
    """PAPER.md:128-149 (Table 2): C, HxW, K, RxS, P, T, sparsity per layer.
    Parsed from tests/golden/table2_layers.csv is the pinned copy; this is the
    generator-side copy used only to draw inputs of these shapes."""
    rows = [
        ("LeNet-Conv2", 20, 11, 64, 5, 1, 2, 0.95),
        ("AlexNetC-Conv3", 32, 6, 64, 5, 2, 1, 0.9),
        ("AlexNetI-Conv4", 384, 5, 384, 3, 1, 1, 0.9),
        ("GoogLeNet-Inception4a.1", 480, 14, 192, 1, 0, 1, 0.9),
        ("GoogLeNet-Inception4a.2", 192, 14, 96, 1, 0, 1, 0.9),
        ("GoogLeNet-Inception4e.3", 160, 14, 320, 3, 1, 1, 0.9),
        ("GoogLeNet-Inception5a.1", 832, 7, 256, 1, 0, 1, 0.95),
        ("GoogLeNet-Inception5a.2", 256, 7, 160, 1, 0, 1, 0.9),
        ("GoogLeNet-Inception5b.3", 192, 7, 384, 3, 1, 1, 0.95),
        ("GoogLeNet-Inception5b.5", 48, 7, 128, 5, 2, 1, 0.95),
    ]
    return [(ConvShape(nm, 101 + i, n, c, hw, hw, k, rs, rs, t, p, 1), sp)
            for i, (nm, c, hw, k, rs, p, t, sp) in enumerate(rows)]


def _rng(seed, config_id, tensor_id, index):
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence([int(seed), int(config_id), int(tensor_id), int(index)])))


def channel_sparsity(shape: ConvShape, seed=0):
    """C3 (R12): per-channel s_c ~ U(0.85, 0.99); round(0.05*C) dead channels
    (s_c = 1) chosen by a seeded permutation.  Shared by every image."""
    rng = _rng(seed, shape.config_id, T_CHANNEL, 0)
    s_c = rng.uniform(0.85, 0.99, size=shape.c)
    dead = rng.permutation(shape.c)[: int(round(0.05 * shape.c))]
    s_c[dead] = 1.0
    return s_c


def activations(shape: ConvShape, sparsity, seed=0, start=0, count=None):
    """Images [start, start+count) of a config: Bernoulli(1-s) mask * |N(0,1)|.
    ``sparsity`` is a float, a per-channel array, or "channel" (C3 recipe)."""
    count = shape.n - start if count is None else count
    per_img = (shape.c, shape.h, shape.w)
    if isinstance(sparsity, str):
        if sparsity != "channel":
            raise ValueError(sparsity)
        sparsity = channel_sparsity(shape, seed)
    s_arr = np.asarray(sparsity, dtype=np.float64)
    thr = s_arr.reshape(-1, 1, 1) if s_arr.ndim == 1 else s_arr
    out = np.empty((count,) + per_img, dtype=np.float32)
    for i in range(count):
        rng = _rng(seed, shape.config_id, T_INPUT, start + i)
        u = rng.random(per_img)
        v = np.abs(rng.standard_normal(per_img, dtype=np.float32))
        out[i] = np.where(u >= thr, v, np.float32(0.0))
    return out


def weights(shape: ConvShape, seed=0, std=0.01, layer_tag=0):
    """W [K][C/G][R][S] and bias [K], both N(0, std^2)."""
    wshape = (shape.k, shape.c // shape.groups, shape.r, shape.s)
    rw = _rng(seed, shape.config_id, T_WEIGHT + 10 * layer_tag, 0)
    rb = _rng(seed, shape.config_id, T_BIAS + 10 * layer_tag, 0)
    w = (rw.standard_normal(wshape) * std).astype(np.float32)
    b = (rb.standard_normal(shape.k) * std).astype(np.float32)
    return w, b


def integer_case(shape: ConvShape, sparsity=0.5, seed=0):
    """Exact-integer data (SURVEY 8c pins): in in {1..7} on a Bernoulli(1-s)
    mask, W in {-8..8}, bias in {-16..16}.  Every product and partial sum is an
    integer below 2^24 in magnitude for the configs used, so fp32 and TF32
    arithmetic are exact and any order of summation gives identical bits."""
    rng = _rng(seed, shape.config_id, 99, 0)
    per = (shape.n, shape.c, shape.h, shape.w)
    mask = rng.random(per) >= sparsity
    x = np.where(mask, rng.integers(1, 8, size=per), 0).astype(np.float32)
    w = rng.integers(-8, 9, size=(shape.k, shape.c // shape.groups, shape.r, shape.s)).astype(np.float32)
    b = rng.integers(-16, 17, size=shape.k).astype(np.float32)
    return x, w, b


def c5_bias_shift():
    """Per-layer bias shifts q_l (R13) written by tools/calibrate_c5.py."""
    path = os.path.join(os.path.dirname(__file__), "c5_bias_shift.json")
    with open(path) as f:
        return json.load(f)


def c5_weights(seed=0):
    """Weights and shifted biases of the conv3->conv4->conv5 chain (R13)."""
    shifts = c5_bias_shift()
    out = []
    for li, shp in enumerate(C5_LAYERS):
        w, b = weights(shp, seed)
        q = shifts.get(shp.name, 0.0)
        out.append((w, (b - np.float32(q)).astype(np.float32)))
    return out


def sha256(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
