"""Convolutional networks on the pipeline session (VGG-style stages, BASELINE
configs[3]).

The reference trains MLPs only (`proj/include/pipesim/trainer.hpp:50-64`;
convolutional architectures are a non-goal, `SPEC.md:379`).  This module
extends its network description with 3x3 / pad-1 convolutions and 2x2 max
pooling (`pb_layer_spec`, include/pipesim_b200.h) so the same session —
nF1B / 1F1B / sequential replay, version pool, device version tags, CUDA
graph — trains a VGG-16 pipeline.  Everything after construction is the
ordinary `pipesim.Session` API.

Conventions (csrc/session.hpp LayerSpec): NHWC activations flattened per
sample; conv weights [out][9*in] with k = (3r + s) * in + c, then b[out];
the first linear layer reads the last conv output flattened in NHWC order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from ._session_abi import pb_layer_net, pb_layer_spec

ACTIVATIONS = ("linear", "relu", "tanh", "sigmoid")
LOSSES = ("mse", "softmax_cross_entropy")


@dataclass
class ConvLayer:
    kind: str  # "conv" | "linear"
    in_: int
    out: int
    h: int = 0
    w: int = 0
    pool: bool = False
    act: str = "relu"

    def fan_in(self) -> int:
        return 9 * self.in_ if self.kind == "conv" else self.in_

    def param_count(self) -> int:
        return self.out * self.fan_in() + self.out

    def in_elems(self) -> int:
        return self.h * self.w * self.in_ if self.kind == "conv" else self.in_

    def out_elems(self) -> int:
        if self.kind == "linear":
            return self.out
        hw = (self.h // 2) * (self.w // 2) if self.pool else self.h * self.w
        return hw * self.out

    def flops(self) -> float:
        """Forward flops per sample (2 per multiply-add)."""
        return 2.0 * self.out * self.fan_in() * (self.h * self.w if self.kind == "conv" else 1)


@dataclass
class ConvNetSpec:
    layers: List[ConvLayer]
    loss: str = "softmax_cross_entropy"
    stage_layers: Optional[Sequence[int]] = None  # None: flop-balanced partition

    layer_net = True  # pipesim.Session dispatches on this

    def layer_count(self) -> int:
        return len(self.layers)

    def layer(self, i) -> ConvLayer:
        return self.layers[i]

    def param_count(self) -> int:
        return sum(l.param_count() for l in self.layers)

    @property
    def widths(self) -> List[int]:
        """Per-sample input elements of every layer, then the classes."""
        return [l.in_elems() for l in self.layers] + [self.layers[-1].out_elems()]

    def flops_per_sample(self) -> float:
        """Forward + backward flops of one training sample: forward, the
        weight gradient and the input gradient of every layer but the first."""
        f = [l.flops() for l in self.layers]
        return 2.0 * sum(f) + sum(f[1:])

    def _c(self, workers: Optional[int] = None):
        arr = (pb_layer_spec * len(self.layers))()
        for i, l in enumerate(self.layers):
            arr[i] = pb_layer_spec(1 if l.kind == "conv" else 0, l.in_, l.out, l.h, l.w,
                                   int(l.pool), ACTIVATIONS.index(l.act))
        st = None
        if self.stage_layers is not None:
            st = np.ascontiguousarray(self.stage_layers, np.int32)
        spec = pb_layer_net(len(self.layers), arr, LOSSES.index(self.loss),
                            st.ctypes.data_as(C.POINTER(C.c_int)) if st is not None else None)
        spec._keep = (arr, st)
        return spec

    def partition(self, workers: int) -> List[int]:
        """Layers per stage (pb_partition_layers: largest stage's forward
        flops minimised), or the explicit stage_layers."""
        if self.stage_layers is not None:
            return list(self.stage_layers)
        fl = np.zeros(workers, np.int32)
        nl = np.zeros(workers, np.int32)
        spec = self._c()
        N.check(N.lib().pb_partition_layers(C.byref(spec), workers,
                                            fl.ctypes.data_as(C.POINTER(C.c_int)),
                                            nl.ctypes.data_as(C.POINTER(C.c_int))))
        return [int(v) for v in nl]


def vgg(cfg: Sequence, image: int = 224, in_ch: int = 3, classes: int = 1000,
        hidden: int = 4096, fc_layers: int = 3) -> ConvNetSpec:
    """A VGG network: `cfg` lists conv output channels and "M" for a 2x2
    max pool (which the preceding conv layer does), then fc_layers linear
    layers (hidden, ..., classes)."""
    layers: List[ConvLayer] = []
    h = w = image
    c = in_ch
    for v in cfg:
        if v == "M":
            if not layers or layers[-1].pool:
                raise ValueError("a pool must follow a conv layer")
            layers[-1].pool = True
            h //= 2
            w //= 2
            continue
        layers.append(ConvLayer("conv", c, int(v), h, w, False, "relu"))
        c = int(v)
    feat = h * w * c
    for i in range(fc_layers):
        last = i == fc_layers - 1
        out = classes if last else hidden
        layers.append(ConvLayer("linear", feat, out, act="linear" if last else "relu"))
        feat = out
    return ConvNetSpec(layers)


VGG16 = (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
         512, 512, 512, "M")


def vgg16(image: int = 224, classes: int = 1000) -> ConvNetSpec:
    """VGG-16 (13 conv + 3 FC) on image x image x 3 inputs."""
    return vgg(VGG16, image=image, classes=classes)


def init_params(spec: ConvNetSpec, seed: int) -> np.ndarray:
    """He-uniform weights U(+-sqrt(6 / fan_in)) and zero biases per layer,
    in the flat layout (per layer W [out][fan_in], then b).  The reference's
    U(+-1/sqrt(fan_in)) (trainer.cpp:557-569) shrinks ReLU activations by
    ~2.4x per layer, which a 16-layer conv net cannot train through."""
    rng = np.random.default_rng(seed)
    parts = []
    for l in spec.layers:
        a = np.sqrt(6.0 / l.fan_in())
        parts.append(rng.uniform(-a, a, l.out * l.fan_in()))
        parts.append(np.zeros(l.out))
    return np.concatenate(parts)


def synthetic_images(rows: int, spec: ConvNetSpec, seed: int = 7):
    """ImageNet-shaped synthetic data: NHWC images U[0, 1) as float32 rows
    and int32 class labels."""
    rng = np.random.default_rng(seed)
    x = rng.random((rows, spec.layers[0].in_elems()), dtype=np.float32)
    classes = spec.layers[-1].out_elems()
    y = rng.integers(0, classes, rows).astype(np.int32)
    return x, y
