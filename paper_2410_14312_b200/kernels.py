"""Per-op access to the sm_100a layer kernels on torch CUDA tensors.

Torch is only the device-memory / stream plumbing here: every op is a call
through the C ABI (``pb_linear_fwd`` ...), which launches the hand-written
kernels.  Used by the kernel parity tests and by diagnostics.
"""
from __future__ import annotations

import torch

from . import _native

ACT = {"linear": 0, "relu": 1, "tanh": 2, "sigmoid": 3}
LOSS = {"mse": 0, "softmax_cross_entropy": 1}


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _ld(t):
    assert t.dim() == 2 and t.stride(1) == 1
    return t.stride(0)


def padded_bf16(rows: int, cols: int, device="cuda") -> torch.Tensor:
    """bf16 [rows, cols] view over a buffer whose row stride is a multiple of 8."""
    ld = (cols + 7) // 8 * 8
    return torch.zeros(rows, ld, dtype=torch.bfloat16, device=device)[:, :cols]


def linear_fwd(x, w, bias, act="linear", y16=None, y32=None):
    rows, inn = x.shape
    out = w.shape[0]
    _native.check(_native.lib().pb_linear_fwd(
        _stream(), _ptr(x), rows, inn, _ld(x), _ptr(w), out, _ld(w), _ptr(bias),
        ACT[act], _ptr(y16), _ld(y16) if y16 is not None else 0,
        _ptr(y32), _ld(y32) if y32 is not None else 0))


def linear_bwd_dx(dz, w, xin, act_prev, d):
    rows, out = dz.shape
    inn = w.shape[1]
    _native.check(_native.lib().pb_linear_bwd_dx(
        _stream(), _ptr(dz), rows, out, _ld(dz), _ptr(w), inn, _ld(w), _ptr(xin),
        _ld(xin) if xin is not None else 0, ACT[act_prev], _ptr(d), _ld(d)))


def linear_bwd_dw_sgd(dz, x, w_cur, w_new, w16, lr):
    rows, out = dz.shape
    inn = x.shape[1]
    _native.check(_native.lib().pb_linear_bwd_dw_sgd(
        _stream(), _ptr(dz), rows, out, _ld(dz), _ptr(x), inn, _ld(x), _ptr(w_cur),
        _ptr(w_new), _ld(w_cur), _ptr(w16), _ld(w16) if w16 is not None else 0,
        float(lr)))


def linear_bwd_dw_sgd_split(dz, x, hi_cur, lo_cur, hi_new, lo_new, lr):
    """Split-master wgrad+SGD: hi_* bf16 [out, ld], lo_* int16 [out, ld]."""
    rows, out = dz.shape
    inn = x.shape[1]
    _native.check(_native.lib().pb_linear_bwd_dw_sgd_split(
        _stream(), _ptr(dz), rows, out, _ld(dz), _ptr(x), inn, _ld(x), _ptr(hi_cur),
        _ptr(lo_cur), _ptr(hi_new), _ptr(lo_new), _ld(hi_cur), float(lr)))


def split_master(w, hi, lo):
    out, inn = w.shape
    _native.check(_native.lib().pb_split_master(_stream(), _ptr(w), out, inn, _ld(w), _ptr(hi),
                                                _ptr(lo), _ld(hi)))


def join_master(hi, lo, w):
    out, inn = w.shape
    _native.check(_native.lib().pb_join_master(_stream(), _ptr(hi), _ptr(lo), out, inn, _ld(hi),
                                               _ptr(w), _ld(w)))


def bias_sgd(dz, b_cur, b_new, b_copy, lr):
    rows, out = dz.shape
    _native.check(_native.lib().pb_bias_sgd(
        _stream(), _ptr(dz), rows, out, _ld(dz), _ptr(b_cur), _ptr(b_new),
        _ptr(b_copy), float(lr)))


def loss_fwd_bwd(y, t, loss, act_last, denom, dz, row_loss):
    rows, cols = y.shape
    _native.check(_native.lib().pb_loss_fwd_bwd(
        _stream(), _ptr(y), rows, cols, _ld(y), _ptr(t), _ld(t), LOSS[loss],
        ACT[act_last], float(denom), _ptr(dz), _ld(dz), _ptr(row_loss)))


def graph_time_us(fns, reps: int = 60) -> float:
    """Device time per call of a kernel launch, cycling through `fns` (e.g.
    closures over several operand copies, so that operands larger than L2 are
    re-read from HBM as inside the pipeline).  The calls are captured in one
    CUDA graph, so the per-call host cost of the C ABI path is excluded, then
    replayed after a warm-up and timed with CUDA events on the stream."""
    if callable(fns):
        fns = [fns]
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):  # warm-up on the capture stream (per-stream workspaces)
        for f in fns:
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            fns[i % len(fns)]()
    g.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()  # replay (and the events) run here
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    g.replay()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / reps


# ---------------------------------------------------------------- conv stages
# NHWC bf16 activations as torch [n, h, w, c] contiguous tensors; conv weights
# [cout, 9 * cin] (tap-major K, k = (3r + s) * cin + c).

def conv_fwd(x, w, bias, act, y):
    n, h, ww, cin = x.shape
    cout = w.shape[0]
    _native.check(_native.lib().pb_conv_fwd(
        _stream(), _ptr(x), n, h, ww, cin, _ptr(w), cout, _ld(w), _ptr(bias), ACT[act], _ptr(y)))


def conv_bwd_dx(dz, w, xin, act_prev, d):
    n, h, ww, cout = dz.shape
    cin = d.shape[-1]
    _native.check(_native.lib().pb_conv_bwd_dx(
        _stream(), _ptr(dz), n, h, ww, cout, _ptr(w), cin, _ld(w), _ptr(xin), ACT[act_prev],
        _ptr(d)))


def conv_bwd_dw_sgd(dz, x, w_cur, w_new, w16, lr):
    n, h, ww, cout = dz.shape
    cin = x.shape[-1]
    _native.check(_native.lib().pb_conv_bwd_dw_sgd(
        _stream(), _ptr(dz), n, h, ww, cout, _ptr(x), cin, _ptr(w_cur), _ptr(w_new),
        _ld(w_cur), _ptr(w16), _ld(w16) if w16 is not None else 0, float(lr)))


def maxpool2_fwd(x, y):
    n, h, ww, c = x.shape
    _native.check(_native.lib().pb_maxpool2_fwd(_stream(), _ptr(x), n, h, ww, c, _ptr(y)))


def maxpool2_bwd(d_out, x, y, d_in):
    n, h, ww, c = x.shape
    _native.check(_native.lib().pb_maxpool2_bwd(_stream(), _ptr(d_out), _ptr(x), _ptr(y), n, h,
                                                ww, c, _ptr(d_in)))


def im2col_first(x, out):
    n, h, ww, c = x.shape
    _native.check(_native.lib().pb_im2col_first(_stream(), _ptr(x), h * ww * c, n, h, ww, c,
                                                _ptr(out), _ld(out)))
