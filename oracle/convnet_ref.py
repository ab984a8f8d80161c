"""TEST INFRASTRUCTURE ONLY — fp64 CPU restatement of the conv-stage math.

The reference's networks are MLPs (`proj/src/trainer.cpp:179-267`); VGG-style
conv stages (BASELINE configs[3]) have no reference counterpart
(`/root/reference/SPEC.md:379` lists convolutional architectures as a
non-goal), so their parity is UNPINNED against the reference and anchored
here instead: the reference's own replay (`pipesim_np.train_epoch`, pinned to
the compiled reference) with its Linear stage math replaced by the same
contracts for 3x3 / pad-1 convolutions and 2x2 max pooling, computed by
torch in float64 on the CPU.  The replay — pins, latest-weights backward,
version retention, loss per micro-batch — is the reference's, unchanged.

Conventions shared with the product (`csrc/session.hpp` LayerSpec):
  * activations are NHWC, flattened per sample (rows of h*w*c values);
  * conv weights are [out][9*in] with k = (3r + s) * in + c, then b[out];
  * a pooled conv layer's output is max_pool2d(act(conv(x) + b), 2);
  * the first linear layer reads the last conv output flattened in NHWC.
Never imported by the product package.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np
import torch
import torch.nn.functional as F

from . import pipesim_np as O


@dataclass
class Layer:
    kind: str  # "conv" | "linear"
    in_: int
    out: int
    h: int = 0
    w: int = 0
    pool: bool = False
    act: str = "relu"

    def fan_in(self):
        return 9 * self.in_ if self.kind == "conv" else self.in_

    def param_count(self):
        return self.out * self.fan_in() + self.out

    def out_elems(self):
        if self.kind == "linear":
            return self.out
        hw = (self.h // 2) * (self.w // 2) if self.pool else self.h * self.w
        return hw * self.out


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64))


def _act(z, a):
    if a == "relu":
        return torch.where(z > 0, z, torch.zeros_like(z))
    if a == "linear":
        return z
    raise ValueError(a)


def _dact(z, a):
    """trainer.cpp:155-169 (derivative from the pre-activation)."""
    if a == "relu":
        return (z > 0).to(z.dtype)
    return torch.ones_like(z)


def _split(p, layer):
    n = layer.out * layer.fan_in()
    return p[:n].reshape(layer.out, layer.fan_in()), p[n:n + layer.out]


def _wt(Wm, layer):  # [out][9*in] tap-major -> torch [out][in][3][3]
    return Wm.reshape(layer.out, 3, 3, layer.in_).permute(0, 3, 1, 2)


def stage_forward(layers: List[Layer], params, x):
    """stage_forward (trainer.cpp:179-206) for conv / linear layers.  The
    cache holds per layer the pre-activation z (conv: NCHW before pooling)
    and the layer output a (pooled, flattened NHWC rows)."""
    p = _t(params)
    cur = _t(x)
    n = cur.shape[0]
    cache = {"input": np.asarray(x), "z": [], "a": []}
    off = 0
    for L in layers:
        Wm, b = _split(p[off:], L)
        off += L.param_count()
        if L.kind == "conv":
            X = cur.reshape(n, L.h, L.w, L.in_).permute(0, 3, 1, 2)
            z = F.conv2d(X, _wt(Wm, L), b, padding=1)
            a = _act(z, L.act)
            if L.pool:
                a = F.max_pool2d(a, 2)
            cur = a.permute(0, 2, 3, 1).reshape(n, -1)
        else:
            z = cur @ Wm.T + b
            cur = _act(z, L.act)
        cache["z"].append(z.numpy())
        cache["a"].append(cur.numpy())
    return cache


def stage_backward(layers: List[Layer], prop, cache, delta):
    """stage_backward (trainer.cpp:216-267): dZ from act' of the cached
    pre-activation (routed through the pooling window's maximum first), the
    weight gradient against the cached input, the delta through the
    propagation weights `prop`."""
    p = _t(prop)
    offs, off = [], 0
    for L in layers:
        offs.append(off)
        off += L.param_count()
    grad = torch.zeros(off, dtype=torch.float64)
    d = _t(delta)
    n = d.shape[0]
    for l in range(len(layers) - 1, -1, -1):
        L = layers[l]
        xin = _t(cache["input"] if l == 0 else cache["a"][l - 1])
        z = _t(cache["z"][l])
        Wm, _ = _split(p[offs[l]:], L)
        if L.kind == "conv":
            ho, wo = (L.h // 2, L.w // 2) if L.pool else (L.h, L.w)
            dout = d.reshape(n, ho, wo, L.out).permute(0, 3, 1, 2)
            if L.pool:
                a = _act(z, L.act)
                _, idx = F.max_pool2d(a, 2, return_indices=True)
                dout = F.max_unpool2d(dout, idx, 2, output_size=a.shape[-2:])
            dz = dout * _dact(z, L.act)
            X = xin.reshape(n, L.h, L.w, L.in_).permute(0, 3, 1, 2)
            gw = torch.nn.grad.conv2d_weight(X, (L.out, L.in_, 3, 3), dz, padding=1)
            nw = L.out * L.fan_in()
            grad[offs[l]:offs[l] + nw] = gw.permute(0, 2, 3, 1).reshape(-1)
            grad[offs[l] + nw:offs[l] + nw + L.out] = dz.sum((0, 2, 3))
            dx = torch.nn.grad.conv2d_input((n, L.in_, L.h, L.w), _wt(Wm, L), dz, padding=1)
            d = dx.permute(0, 2, 3, 1).reshape(n, -1)
        else:
            dz = d * _dact(z, L.act)
            nw = L.out * L.in_
            grad[offs[l]:offs[l] + nw] = (dz.T @ xin).reshape(-1)
            grad[offs[l] + nw:offs[l] + nw + L.out] = dz.sum(0)
            d = dz @ Wm
    return grad.numpy(), d.numpy()


# ----------------------------------------------------- bf16-storage variant
# The same contracts with the B200 path's storage rounding applied: bf16
# weight copies and bf16 activations / deltas between kernels (fp32 masters
# and accumulation are kept in fp64 here).  It separates the bf16 path's
# representation error from everything else: max pooling then routes the
# gradient to the first maximum of the *rounded* window exactly as the
# device does (ties within bf16's 2^-8 spacing are common and move the
# gradient to another pixel), so what remains is accumulation order.
def _r16(t):
    return t.to(torch.bfloat16).to(torch.float64)


def _pool_first_max(a):
    """2x2 max pooling of NCHW `a`; returns (pooled, one-hot mask of the first
    maximum of each window in (0,0) (0,1) (1,0) (1,1) order)."""
    n, c, h, w = a.shape
    win = a.reshape(n, c, h // 2, 2, w // 2, 2).permute(0, 1, 2, 4, 3, 5).reshape(
        n, c, h // 2, w // 2, 4)
    m, idx = win.max(-1)  # torch returns the first index of the maximum
    first = torch.zeros_like(win).scatter_(-1, idx.unsqueeze(-1), 1.0)
    # double-check the first-occurrence rule on ties
    eq = (win == m.unsqueeze(-1)).to(torch.int64)
    want = (eq.cumsum(-1) == 1) & (eq == 1)
    assert torch.equal(first.bool(), want)
    mask = first.reshape(n, c, h // 2, w // 2, 2, 2).permute(0, 1, 2, 4, 3, 5).reshape(n, c, h, w)
    return m, mask


def stage_forward16(layers: List[Layer], params, x):
    p = _t(params)
    cur = _r16(_t(x))
    n = cur.shape[0]
    cache = {"input": cur.numpy(), "z": [], "a": []}
    off = 0
    for i, L in enumerate(layers):
        Wm, b = _split(p[off:], L)
        Wm = _r16(Wm)
        off += L.param_count()
        # the network's logits (a linear-activation Linear layer) stay fp32
        last = L.kind == "linear" and L.act == "linear"
        if L.kind == "conv":
            X = cur.reshape(n, L.h, L.w, L.in_).permute(0, 3, 1, 2)
            a = _r16(_act(F.conv2d(X, _wt(Wm, L), b, padding=1), L.act))
            pre = a.permute(0, 2, 3, 1).reshape(n, -1)
            if L.pool:
                a, _ = _pool_first_max(a)
            cur = a.permute(0, 2, 3, 1).reshape(n, -1)
            cache["z"].append(pre.numpy())
        else:
            z = cur @ Wm.T + b
            cur = _act(z, L.act)
            if not last:  # the logits stay fp32 (loss kernel input)
                cur = _r16(cur)
            cache["z"].append(cur.numpy())
        cache["a"].append(cur.numpy())
    return cache


def stage_backward16(layers: List[Layer], prop, cache, delta):
    """The device's order: the delta arrives gated; a pooled conv routes it
    to the first maximum of the rounded window; the weight gradient reads the
    bf16 input; the dgrad multiplies by act' of the stored (bf16) input and
    rounds the result to bf16."""
    p = _t(prop)
    offs, off = [], 0
    for L in layers:
        offs.append(off)
        off += L.param_count()
    grad = torch.zeros(off, dtype=torch.float64)
    d = _r16(_t(delta))
    n = d.shape[0]
    for l in range(len(layers) - 1, -1, -1):
        L = layers[l]
        xin = _t(cache["input"] if l == 0 else cache["a"][l - 1])
        Wm, _ = _split(p[offs[l]:], L)
        Wm = _r16(Wm)
        gate_act = "relu" if l == 0 else layers[l - 1].act
        if L.kind == "conv":
            ho, wo = (L.h // 2, L.w // 2) if L.pool else (L.h, L.w)
            dz = d.reshape(n, ho, wo, L.out).permute(0, 3, 1, 2)
            if L.pool:
                pre = _t(cache["z"][l]).reshape(n, L.h, L.w, L.out).permute(0, 3, 1, 2)
                _, mask = _pool_first_max(pre)
                dz = F.interpolate(dz, scale_factor=2, mode="nearest") * mask
            X = xin.reshape(n, L.h, L.w, L.in_).permute(0, 3, 1, 2)
            gw = torch.nn.grad.conv2d_weight(X, (L.out, L.in_, 3, 3), dz, padding=1)
            nw = L.out * L.fan_in()
            grad[offs[l]:offs[l] + nw] = gw.permute(0, 2, 3, 1).reshape(-1)
            grad[offs[l] + nw:offs[l] + nw + L.out] = dz.sum((0, 2, 3))
            dx = torch.nn.grad.conv2d_input((n, L.in_, L.h, L.w), _wt(Wm, L), dz, padding=1)
            d = dx.permute(0, 2, 3, 1).reshape(n, -1)
        else:
            dz = d
            nw = L.out * L.in_
            grad[offs[l]:offs[l] + nw] = (dz.T @ xin).reshape(-1)
            grad[offs[l] + nw:offs[l] + nw + L.out] = dz.sum(0)
            d = dz @ Wm
        # act' of the layer below from its stored output (= this input)
        d = _r16(d * _dact(xin, gate_act))
    return grad.numpy(), d.numpy()


class ConvMath:
    """layer_math for pipesim_np.train_epoch: per-stage layer lists."""

    def __init__(self, layers: List[Layer], stage_layers: List[int], storage="fp64"):
        self.layers, f = [], 0
        for c in stage_layers:
            self.layers.append(layers[f:f + c])
            f += c
        self.sizes = [sum(L.param_count() for L in st) for st in self.layers]
        if storage == "bf16":
            self.forward, self.backward = stage_forward16, stage_backward16
        else:
            self.forward, self.backward = stage_forward, stage_backward


def train_epoch(layers: List[Layer], stage_layers, N, B, M, lr, x, y, params,
                mode="timeprest", storage="fp64"):
    """train_epoch (trainer.cpp:642-660) over a conv network: the reference's
    replay with conv stage math; softmax cross-entropy on dense targets.
    storage="bf16" applies the B200 path's bf16 storage rounding."""
    net = O.Net([1, 1], ["linear"], "softmax_cross_entropy")
    return O.train_epoch(net, len(stage_layers), N, B, M, lr, np.asarray(x, np.float64),
                         np.asarray(y, np.float64), np.asarray(params, np.float64), mode=mode,
                         layer_math=ConvMath(layers, stage_layers, storage))
