"""TEST INFRASTRUCTURE ONLY — ctypes access to the compiled reference.

oracle/_ref/libpipesim_ref.so is the UNMODIFIED reference library
(/root/reference/proj/src, built by oracle/Makefile) plus oracle/ref_shim.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may use it, as the checker or the timed baseline —
never as the product path.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libpipesim_ref.so"
_lib = None


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise FileNotFoundError(f"{LIB} not built (make -C oracle)")
        _lib = C.CDLL(str(LIB))
    return _lib


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(code):
    if code != 0:
        buf = C.create_string_buffer(4096)
        lib().ref_last_error(buf, 4096)
        raise RefError(code, buf.value.decode())


def schedule(w, n, m, mode=0):
    """Grid as int array [W][H][3] = (kind, mini, micro); kind 0/1/2."""
    h = C.c_int()
    code = lib().ref_schedule(w, n, m, mode, C.byref(h), None, 0)
    if code not in (0, 7):
        _check(code)
    cells = np.zeros((w, h.value, 3), dtype=np.int32)
    _check(lib().ref_schedule(w, n, m, mode, C.byref(h), _ip(cells), h.value))
    return cells


def validate(w, n, m, mode, cells):
    """validate_schedule on a [W][H][3] grid -> [(kind, message)]."""
    cells = np.ascontiguousarray(cells, np.int32)
    nv = C.c_int()
    kinds = np.zeros(4096, np.int32)
    msg = C.create_string_buffer(1 << 20)
    _check(lib().ref_validate(w, n, m, mode, _ip(cells), cells.shape[1], C.byref(nv),
                              _ip(kinds), 4096, msg, 1 << 20))
    lines = msg.value.decode().split("\n")
    return [(int(kinds[i]), lines[i]) for i in range(nv.value)]


def render_ascii(w, n, m, mode=0):
    buf = C.create_string_buffer(1 << 20)
    _check(lib().ref_render_ascii(w, n, m, mode, buf, 1 << 20))
    return buf.value.decode()


def schedule_document(w, n, m, mode=0):
    """The reference's schedule document JSON (export.cpp:78-139)."""
    buf = C.create_string_buffer(1 << 24)
    _check(lib().ref_schedule_document(w, n, m, mode, buf, 1 << 24))
    return buf.value.decode()


def ledger(w, n, m, mode=0):
    units = n if mode == 0 else 1
    commits = np.zeros((m * w, 4), np.int32)
    pins = np.zeros((m * units, 4), np.int32)
    cons = np.zeros((m * w, 4), np.int32)
    us = np.zeros(m, np.int32)
    fcs = np.zeros(m + 1, np.int32)
    _check(lib().ref_ledger(w, n, m, mode, _ip(commits), _ip(pins), _ip(cons), _ip(us),
                            _ip(fcs)))
    return dict(commits=commits, pins=pins, consumptions=cons, update_source=us,
                full_commit_slot=fcs)


def retention(w, n, m, mode=0):
    iv = np.zeros((w, m + 1, 3), np.int32)
    peak = np.zeros(w, np.int32)
    _check(lib().ref_retention(w, n, m, mode, _ip(iv), _ip(peak)))
    return iv, peak


def measure_v(w, n, m, mode=0, strict=True):
    v = C.c_int()
    _check(lib().ref_measure_v(w, n, m, mode, int(strict), C.byref(v)))
    return v.value


def closed_form_v(w, n):
    v = C.c_int()
    _check(lib().ref_closed_form_v(w, n, C.byref(v)))
    return v.value


def _net(widths, acts):
    wa = np.ascontiguousarray(widths, np.int32)
    aa = np.ascontiguousarray(acts, np.int32)
    return wa, aa


def param_count(widths):
    return int(sum(widths[i] * widths[i + 1] + widths[i + 1] for i in range(len(widths) - 1)))


def init_params(widths, acts, loss, seed):
    wa, aa = _net(widths, acts)
    out = np.zeros(param_count(widths))
    _check(lib().ref_init_params(len(widths) - 1, _ip(wa), _ip(aa), loss,
                                 C.c_uint64(seed), _dp(out)))
    return out


def partition(widths, acts, loss, w):
    wa, aa = _net(widths, acts)
    fl = np.zeros(w, np.int32)
    nl = np.zeros(w, np.int32)
    _check(lib().ref_partition(len(widths) - 1, _ip(wa), _ip(aa), loss, w, _ip(fl), _ip(nl)))
    return fl, nl


def synthetic(samples, seed):
    x = np.zeros((samples, 2))
    y = np.zeros((samples, 2))
    _check(lib().ref_synthetic(samples, C.c_uint64(seed), _dp(x), _dp(y)))
    return x, y


MODES = {"timeprest": 0, "pipedream": 1, "sequential": 2}


def train(widths, acts, loss, w, n, b, m, lr, seed, mode, x, y, params, epochs=1,
          observe=False):
    """Run `epochs` reference epochs. Returns dict(params, losses, pinned,
    consumed, log, held, seconds)."""
    mode_id = MODES[mode] if isinstance(mode, str) else mode
    wa, aa = _net(widths, acts)
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    p_in = np.ascontiguousarray(params, np.float64)
    p_out = np.zeros_like(p_in)
    units = n if mode_id == 0 else 1
    losses = np.zeros((epochs, m))
    pinned = np.zeros((epochs, m, units), np.int32)
    consumed = np.zeros((epochs, m), np.int32)
    cap = 1 << 22
    text = C.create_string_buffer(cap)
    held = None
    held_ptr, held_cap = None, 0
    if observe:
        h = schedule(w, n, m, 0 if mode_id != 1 else 1).shape[1]
        held = np.zeros((h, w, m + 1), np.int32)
        held_ptr, held_cap = _ip(held), h
    secs = C.c_double()
    _check(lib().ref_train(len(widths) - 1, _ip(wa), _ip(aa), loss, w, n, b, m,
                           C.c_double(lr), C.c_uint64(seed), mode_id, epochs, _dp(x),
                           _dp(y), _dp(p_in), _dp(p_out), _dp(losses), _ip(pinned),
                           _ip(consumed), text, cap, held_ptr, held_cap, C.byref(secs)))
    return dict(params=p_out, losses=losses, pinned=pinned, consumed=consumed,
                log=text.value.decode(), held=held, seconds=secs.value)


def network_loss(widths, acts, loss, params, x, y):
    wa, aa = _net(widths, acts)
    out = C.c_double()
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    _check(lib().ref_network_loss(len(widths) - 1, _ip(wa), _ip(aa), loss,
                                  _dp(np.ascontiguousarray(params, np.float64)),
                                  x.shape[0], _dp(x), _dp(y), C.byref(out)))
    return out.value


def network_gradient(widths, acts, loss, params, x, y):
    wa, aa = _net(widths, acts)
    out = np.zeros(param_count(widths))
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    _check(lib().ref_network_gradient(len(widths) - 1, _ip(wa), _ip(aa), loss,
                                      _dp(np.ascontiguousarray(params, np.float64)),
                                      x.shape[0], _dp(x), _dp(y), _dp(out)))
    return out


def checkpoint_stage(stage_id, first_layer, layers, version, params, loss, epoch, path):
    """Reference checkpoint_stage; layers = [(in, out, act_id), ...]."""
    lay = np.ascontiguousarray(layers, np.int32)
    p = np.ascontiguousarray(params, np.float64)
    _check(lib().ref_checkpoint_stage(stage_id, first_layer, len(lay), _ip(lay), version,
                                      _dp(p), len(p), loss, epoch, str(path).encode()))


def restore_stage(path, expected_stage=0, expected_epoch=0, cap=1 << 24):
    """Reference restore_stage -> (params, version, epoch)."""
    out = np.zeros(cap)
    n, v, e = C.c_int(), C.c_int(), C.c_int()
    _check(lib().ref_restore_stage(str(path).encode(), expected_stage, expected_epoch, _dp(out),
                                   cap, C.byref(n), C.byref(v), C.byref(e)))
    return out[:n.value].copy(), v.value, e.value


def digest_seconds(values):
    """(seconds, digest) of the reference's params_digest over `values`."""
    v = np.ascontiguousarray(values, np.float64)
    secs = C.c_double()
    out = C.create_string_buffer(17)
    _check(lib().ref_digest_seconds(_dp(v), C.c_int64(len(v)), C.byref(secs), out))
    return secs.value, out.value.decode()
