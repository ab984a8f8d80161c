"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot path.

A numpy / pure-Python restatement of pipesim's pipeline step, used as the
parity checker for the B200 build (tests/, __graft_entry__.smoke(),
bench.py's cpu_baseline leg).  It is never imported by the product package.

It is pinned against the compiled reference itself (oracle/_ref, see
tests/test_oracle.py) and against the reference's golden files, which are
regenerated into tests/golden/ by tests/golden/make_golden.py.

Every function cites the reference file:line it restates
(paths relative to /root/reference/proj).
"""
from __future__ import annotations

import math
from collections import deque

import numpy as np

# --------------------------------------------------------------- randomness

_NN, _MM = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)


class MT19937_64:
    """std::mt19937_64, vectorised twist (bit-identical to libstdc++).

    Used through next_uniform (trainer.cpp:141-143) and raw draws."""

    def __init__(self, seed: int):
        mt = np.zeros(_NN, dtype=np.uint64)
        mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        f = 6364136223846793005
        prev = int(mt[0])
        for i in range(1, _NN):
            prev = (f * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            mt[i] = prev
        self.mt = mt
        self.idx = _NN

    @staticmethod
    def _mix(upper, lower, far):
        y = (upper & _UM) | (lower & _LM)
        mag = np.where((y & np.uint64(1)) != 0, _MATRIX_A, np.uint64(0))
        return far ^ (y >> np.uint64(1)) ^ mag

    def _twist(self):
        mt = self.mt
        mt[0:_NN - _MM] = self._mix(mt[0:_NN - _MM], mt[1:_NN - _MM + 1], mt[_MM:_NN])
        # i in [NN-MM, NN-1): far = mt[i + MM - NN], already updated above
        for lo in range(_NN - _MM, _NN - 1, _MM):
            hi = min(lo + _MM, _NN - 1)
            mt[lo:hi] = self._mix(mt[lo:hi], mt[lo + 1:hi + 1],
                                  mt[lo + _MM - _NN:hi + _MM - _NN])
        mt[_NN - 1] = self._mix(mt[_NN - 1:_NN], mt[0:1], mt[_MM - 1:_MM])[0]
        self.idx = 0

    @staticmethod
    def _temper(x):
        x = x ^ ((x >> np.uint64(29)) & np.uint64(0x5555555555555555))
        x = x ^ ((x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
        x = x ^ ((x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
        return x ^ (x >> np.uint64(43))

    def draw(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        pos = 0
        while pos < count:
            if self.idx >= _NN:
                self._twist()
            take = min(count - pos, _NN - self.idx)
            out[pos:pos + take] = self._temper(self.mt[self.idx:self.idx + take])
            self.idx += take
            pos += take
        return out

    def __call__(self) -> int:
        return int(self.draw(1)[0])

    def uniform(self, count: int) -> np.ndarray:
        """next_uniform (trainer.cpp:141-143): (rng() >> 11) * 2^-53."""
        return (self.draw(count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


# --------------------------------------------------------------- model setup
ACTS = ("linear", "relu", "tanh", "sigmoid")
LOSSES = ("mse", "softmax_cross_entropy")


def param_count(widths):
    return sum(widths[i] * widths[i + 1] + widths[i + 1] for i in range(len(widths) - 1))


def init_network_params(widths, seed):
    """trainer.cpp:557-569: U(-1/sqrt(in), 1/sqrt(in)) layer by layer, W then b."""
    g = MT19937_64(seed)
    parts = []
    for l in range(len(widths) - 1):
        n = widths[l] * widths[l + 1] + widths[l + 1]
        parts.append((2.0 * g.uniform(n) - 1.0) * (1.0 / math.sqrt(widths[l])))
    return np.concatenate(parts) if parts else np.zeros(0)


def partition_model(widths, workers):
    """trainer.cpp:104-135.  Returns [(first_layer, n_layers)] per stage."""
    L = len(widths) - 1
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if L < workers:
        raise ValueError("cannot split layers across stages")
    counts = [widths[l] * widths[l + 1] + widths[l + 1] for l in range(L)]
    target = sum(counts) / workers
    out, nxt = [], 0
    for s in range(1, workers + 1):
        first = nxt
        remaining = workers - s
        taken = 0.0
        while nxt < L - remaining:
            if s < workers and taken >= target:
                break
            taken += counts[nxt]
            nxt += 1
            if s < workers and taken >= target:
                break
        out.append((first, nxt - first))
    return out


def make_synthetic_task(samples, seed):
    """trainer.cpp:609-626 (rejection sampling, margin 0.1)."""
    g = MT19937_64(seed)
    x = np.zeros((samples, 2))
    y = np.zeros((samples, 2))
    for i in range(samples):
        while True:
            a = 2.0 * g.uniform(1)[0] - 1.0
            b = 2.0 * g.uniform(1)[0] - 1.0
            m = 0.8 * a - 0.6 * b
            if abs(m) >= 0.1:
                break
        x[i] = (a, b)
        y[i, 0 if m > 0.0 else 1] = 1.0
    return x, y


def make_classification_task(rows, features, classes, seed=7):
    """SURVEY §8(d) synthetic inputs: x ~ U[0,1) from mt19937_64(seed) row-major,
    then labels rng() % C, one-hot.  (Restates pb_make_classification_task.)"""
    g = MT19937_64(seed)
    x = g.uniform(rows * features).reshape(rows, features)
    labels = (g.draw(rows) % np.uint64(classes)).astype(np.int64)
    y = np.zeros((rows, classes))
    y[np.arange(rows), labels] = 1.0
    return x, y


# --------------------------------------------------------------- text / digest
def format_double(v: float) -> str:
    """std::to_chars(double) shortest round trip (text.cpp:24-28): the
    shorter of fixed and scientific notation, fixed on ties."""
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    r = repr(float(v))
    neg = r.startswith("-")
    if neg:
        r = r[1:]
    if "e" in r:
        mant, exp = r.split("e")
        exp = int(exp)
    else:
        mant, exp = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    point = len(ip) + exp  # decimal point position relative to digits of ip+fp
    lead = len(ip + fp) - len((ip + fp).lstrip("0"))
    point -= lead
    digits = digits.rstrip("0") or "0"
    # value = 0.digits * 10^point
    nd = len(digits)
    # scientific: d[.ddd]e±XX
    sexp = point - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + \
        ("-" if sexp < 0 else "+") + f"{abs(sexp):02d}"
    if point <= 0:
        fix = "0." + "0" * (-point) + digits
    elif point >= nd:
        fix = digits + "0" * (point - nd)
    else:
        fix = digits[:point] + "." + digits[point:]
    best = fix if len(fix) <= len(sci) else sci
    return ("-" if neg else "") + best


def fnv1a64_hex(data: bytes) -> str:
    """text.cpp:39-51.  The reference's offset basis is 1469598103934665603
    (not the textbook 14695981039346656037)."""
    h = 1469598103934665603
    for c in data:
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def params_digest(flat) -> str:
    """trainer.cpp:599-607."""
    return fnv1a64_hex("".join(format_double(float(v)) + "\n" for v in flat).encode())


# --------------------------------------------------------------- schedule
IDLE, FWD, BWD = 0, 1, 2


def build_schedule(W, N, M, mode="timeprest"):
    """schedule.cpp:95-196.  Returns int array [W][H][3] (kind, mini, micro)."""
    if W < 2:
        raise ValueError("workers")
    if N < 2:
        raise ValueError("micro_batches")
    if M < 1:
        raise ValueError("mini_batches")
    nf1b = mode == "timeprest"
    units = N if nf1b else 1
    cap = 0 if nf1b else W
    pending = deque((k, j if nf1b else 0) for k in range(1, M + 1) for j in range(1, units + 1))
    queues = [deque() for _ in range(W + 2)]
    reserved = {}
    exited = {}
    started = completed = 0
    cells = {}
    left = M * units * W + M * W
    t = 0
    while left > 0:
        t += 1
        for s in range(1, W + 1):
            if (s, t) in reserved:
                cells[(s, t)] = (BWD, reserved[(s, t)], 0)
                if s == 1:
                    completed += 1
                left -= 1
                continue
            unit = None
            if s == 1:
                if pending:
                    ok = True
                    if cap > 0 and pending[0][1] <= 1:
                        ok = started - completed < cap
                    if ok:
                        unit = pending.popleft()
            elif queues[s] and queues[s][0][1] < t:
                unit = queues[s].popleft()[0]
            if unit is None:
                continue
            k, j = unit
            cells[(s, t)] = (FWD, k, j)
            left -= 1
            if s == 1 and j <= 1:
                started += 1
            if s < W:
                queues[s + 1].append((unit, t))
            else:
                exited[k] = exited.get(k, 0) + 1
                if exited[k] == units:
                    for st in range(W, 0, -1):
                        reserved[(st, t + 1 + (W - st))] = k
    H = max(tt for (_, tt) in cells) if cells else 0
    grid = np.zeros((W, H, 3), np.int32)
    for (s, tt), c in cells.items():
        grid[s - 1, tt - 1] = c
    return grid


def _slot_maps(grid):
    fwd, bwd = {}, {}
    W, H, _ = grid.shape
    for s in range(W):
        for t in range(H):
            kind, k, j = (int(v) for v in grid[s, t])
            if kind == FWD:
                fwd.setdefault((k, j, s + 1), t + 1)
            elif kind == BWD:
                bwd.setdefault((k, s + 1), t + 1)
    return fwd, bwd


def assign_versions(grid, W, N, M, mode="timeprest"):
    """ledger.cpp:54-119 (without the structural validation pass)."""
    nf1b = mode == "timeprest"
    units = N if nf1b else 1
    fwd, bwd = _slot_maps(grid)
    fcs = [0] + [bwd[(k, 1)] for k in range(1, M + 1)]

    def latest_before(slot):
        v = 0
        for k in range(1, M + 1):
            if fcs[k] < slot:
                v = k
        return v

    commits = sorted(((k, k, s, bwd[(k, s)]) for k in range(1, M + 1)
                      for s in range(W, 0, -1)), key=lambda c: c[3])
    pins = []
    for k in range(1, M + 1):
        for j in range(1, units + 1):
            micro = j if nf1b else 0
            inj = fwd[(k, micro, 1)]
            pins.append((k, micro, inj, latest_before(inj)))
    pin_of = {(p[0], p[1]): p[3] for p in pins}
    us, cons = [], []
    for k in range(1, M + 1):
        if nf1b:
            us.append(latest_before(bwd[(k, W)]))
            for s in range(W, 0, -1):
                arr = bwd[(k, s)]
                used = 0
                for v in range(1, k):
                    if bwd[(v, s)] < arr:
                        used = v
                cons.append((k, s, arr, used))
        else:
            st = pin_of[(k, 0)]
            us.append(st)
            for s in range(W, 0, -1):
                cons.append((k, s, bwd[(k, s)], st))
    return dict(commits=np.array(commits, np.int32), pins=np.array(pins, np.int32),
                consumptions=np.array(cons, np.int32),
                update_source=np.array(us, np.int32), full_commit_slot=np.array(fcs, np.int32))


def measure_version_difference(update_source, W, N, M, strict=True):
    """ledger.cpp:121-142."""
    if strict and M < 2 * (W + N):
        raise ValueError("insufficient horizon")
    if M < 2:
        raise ValueError("insufficient horizon")
    v = 0
    for k in range(M // 2 + 1, M + 1):
        gap = k - int(update_source[k - 1])
        if v == 0:
            v = gap
        if gap != v:
            raise ValueError("version difference not steady")
    return v


def closed_form_v(W, N):
    """ledger.cpp:144-147."""
    if W < 2 or N < 2:
        raise ValueError("domain")
    return (W + N - 2) // N


def retention_timeline(grid, ledger, W, M, mode="timeprest"):
    """ledger.cpp:224-264.  Returns (intervals [W][M+1][3], peak[W])."""
    nf1b = mode == "timeprest"
    fwd, bwd = _slot_maps(grid)
    H = grid.shape[1]
    riders = {}
    for k, j, _, v in ledger["pins"]:
        riders.setdefault(int(v), []).append((int(k), int(j)))
    iv = np.zeros((W, M + 1, 3), np.int32)
    peak = np.zeros(W, np.int32)
    for s in range(1, W + 1):
        def commit(v):
            return 0 if v == 0 else bwd[(v, s)]
        for v in range(M + 1):
            until = commit(v + 1) if v < M else H
            for k, j in riders.get(v, []):
                until = max(until, fwd[(k, j, s)])
                if not nf1b:
                    until = max(until, bwd[(k, s)])
            iv[s - 1, v] = (v, commit(v), until + 1)
        best = 0
        for t in range(1, H + 1):
            best = max(best, int(((iv[s - 1, :, 1] <= t) & (t < iv[s - 1, :, 2])).sum()))
        peak[s - 1] = best
    return iv, peak


def render_ascii(grid):
    """render.cpp:40-65 (the timeline golden format)."""
    W, H, _ = grid.shape

    def label(c):
        kind, k, j = (int(v) for v in c)
        if kind == IDLE:
            return ""
        if kind == BWD:
            return f"B{k}"
        return f"{k}" + (chr(ord("A") + (j - 1) % 26) if j > 0 else "")

    width = max([2] + [len(label(grid[s, t])) for s in range(W) for t in range(H)])
    lines = []
    for s in range(W):
        line = " ".join(label(grid[s, t]).ljust(width) for t in range(H)).rstrip()
        lines.append(line + "\n")
    return "".join(lines)


# --------------------------------------------------------------- layer math
def _act(z, a):
    if a == "relu":
        return np.where(z > 0.0, z, 0.0)
    if a == "tanh":
        return np.tanh(z)
    if a == "sigmoid":
        return 1.0 / (1.0 + np.exp(-z))
    return z


def _dact(z, a):
    """trainer.cpp:155-169 (derivative from the pre-activation)."""
    if a == "relu":
        return (z > 0.0).astype(np.float64)
    if a == "tanh":
        t = np.tanh(z)
        return 1.0 - t * t
    if a == "sigmoid":
        s = 1.0 / (1.0 + np.exp(-z))
        return s * (1.0 - s)
    return np.ones_like(z)


def _layers(widths, acts, first, count):
    return [(widths[l], widths[l + 1], acts[l]) for l in range(first, first + count)]


def stage_forward(layers, params, x):
    """trainer.cpp:179-206.  Returns cache dict(input, z[], a[])."""
    cache = {"input": x, "z": [], "a": []}
    off = 0
    cur = x
    for (i, o, a) in layers:
        W = params[off:off + o * i].reshape(o, i)
        b = params[off + o * i:off + o * i + o]
        z = cur @ W.T + b
        cur = _act(z, a)
        cache["z"].append(z)
        cache["a"].append(cur)
        off += o * i + o
    return cache


def stage_backward(layers, prop, cache, delta):
    """trainer.cpp:216-267.  Returns (grad, input_delta)."""
    grad = np.zeros_like(prop)
    offs = []
    off = 0
    for (i, o, a) in layers:
        offs.append(off)
        off += o * i + o
    for l in range(len(layers) - 1, -1, -1):
        i, o, a = layers[l]
        x = cache["input"] if l == 0 else cache["a"][l - 1]
        W = prop[offs[l]:offs[l] + o * i].reshape(o, i)
        dz = delta * _dact(cache["z"][l], a)
        grad[offs[l]:offs[l] + o * i] += (dz.T @ x).reshape(-1)
        grad[offs[l] + o * i:offs[l] + o * i + o] += dz.sum(0)
        delta = dz @ W
    return grad, delta


def loss_mean(y, t, kind):
    """trainer.cpp:270-289."""
    if kind == "mse":
        return float(((y - t) ** 2).sum() / y.shape[0])
    zmax = y.max(1, keepdims=True)
    logden = np.log(np.exp(y - zmax).sum(1, keepdims=True))
    mask = t > 0.5
    return float((-(y - zmax - logden) * t * mask).sum() / y.shape[0])


def loss_grad(y, t, kind, denom):
    """trainer.cpp:294-312."""
    if kind == "mse":
        return 2.0 * (y - t) / denom
    zmax = y.max(1, keepdims=True)
    e = np.exp(y - zmax)
    return (e / e.sum(1, keepdims=True) - t) / denom


# --------------------------------------------------------------- replay
class Net:
    def __init__(self, widths, acts, loss):
        self.widths = list(widths)
        self.acts = [ACTS[a] if isinstance(a, (int, np.integer)) else a for a in acts]
        self.loss = LOSSES[loss] if isinstance(loss, (int, np.integer)) else loss


def train_epoch(net, W, N, B, M, lr, x, y, params, mode="timeprest", observe=False,
                layer_math=None):
    """train_epoch (trainer.cpp:642-660) → replay_grid (:388-508) or
    sequential_epoch (:510-553).  `params` is the whole-network flat vector
    (current versions).  Returns dict(params, losses, pinned, consumed, held).

    layer_math (optional) replaces the Linear stage math for other layer
    kinds (oracle/convnet_ref.py): an object with `layers` (per stage),
    `sizes` (per-stage parameter counts), `forward(layers, params, x)` and
    `backward(layers, prop, cache, delta)` with stage_forward /
    stage_backward's contracts; the replay itself is unchanged."""
    global stage_forward, stage_backward
    if layer_math is not None:
        saved = (stage_forward, stage_backward)
        stage_forward, stage_backward = layer_math.forward, layer_math.backward
        try:
            return _train_epoch(net, W, N, B, M, lr, x, y, params, mode, observe,
                                layer_math.sizes, layer_math.layers)
        finally:
            stage_forward, stage_backward = saved
    parts = partition_model(net.widths, W)
    sizes = [sum(net.widths[l] * net.widths[l + 1] + net.widths[l + 1]
                 for l in range(f, f + c)) for f, c in parts]
    layers = [_layers(net.widths, net.acts, f, c) for f, c in parts]
    return _train_epoch(net, W, N, B, M, lr, x, y, params, mode, observe, sizes, layers)


def _train_epoch(net, W, N, B, M, lr, x, y, params, mode, observe, sizes, layers):
    offs = np.cumsum([0] + sizes)
    stores = [{0: params[offs[s]:offs[s + 1]].copy()} for s in range(W)]
    current = [0] * W
    losses, pinned, consumed = [], [], []

    if mode == "sequential":
        for k in range(1, M + 1):
            xin = x[(k - 1) * B:k * B]
            tgt = y[(k - 1) * B:k * B]
            caches = []
            cur = xin
            for s in range(W):
                c = stage_forward(layers[s], stores[s][current[s]], cur)
                caches.append(c)
                cur = c["a"][-1]
            losses.append(loss_mean(cur, tgt, net.loss))
            delta = loss_grad(cur, tgt, net.loss, B)
            for s in range(W - 1, -1, -1):
                p = stores[s][current[s]]
                g, delta = stage_backward(layers[s], p, caches[s], delta)
                stores[s] = {k: p - lr * g}
                current[s] = k
            pinned.append([k - 1])
            consumed.append(k - 1)
        flat = np.concatenate([stores[s][current[s]] for s in range(W)])
        return dict(params=flat, losses=np.array(losses), pinned=pinned,
                    consumed=np.array(consumed), held=None)

    stashed = mode == "pipedream"
    n = 1 if stashed else N
    micro_rows = B // n
    grid = build_schedule(W, N, M, mode)
    led = assign_versions(grid, W, N, M, mode)
    iv, _ = retention_timeline(grid, led, W, M, mode)
    pin = {(int(p[0]), int(p[1])): int(p[3]) for p in led["pins"]}
    fwd, deltas, mini_loss = {}, {}, {}
    H = grid.shape[1]
    held = np.zeros((H, W, M + 1), np.int32) if observe else None
    logs = {}
    for t in range(1, H + 1):
        for s in range(W):
            for v in list(stores[s]):
                freed = int(iv[s, v, 2])
                if freed != 0 and freed <= t:
                    del stores[s][v]
        for s in range(1, W + 1):
            kind, k, j = (int(v) for v in grid[s - 1, t - 1])
            if kind == IDLE:
                continue
            if kind == FWD:
                ver = pin[(k, j)]
                if s == 1:
                    first = (k - 1) * B + ((j - 1) * micro_rows if j > 0 else 0)
                    inp = x[first:first + micro_rows]
                else:
                    inp = fwd[(k, j, s - 1)]["a"][-1]
                fwd[(k, j, s)] = stage_forward(layers[s - 1], stores[s - 1][ver], inp)
                continue
            parts_c = [fwd[(k, 0 if stashed else jj, s)] for jj in range(1, n + 1)]
            stacked = {"input": np.concatenate([c["input"] for c in parts_c]),
                       "z": [np.concatenate([c["z"][l] for c in parts_c])
                             for l in range(len(layers[s - 1]))],
                       "a": [np.concatenate([c["a"][l] for c in parts_c])
                             for l in range(len(layers[s - 1]))]}
            if s == W:
                tot = 0.0
                for jj in range(1, n + 1):
                    first = (k - 1) * B + (jj - 1) * micro_rows
                    tot += loss_mean(parts_c[jj - 1]["a"][-1], y[first:first + micro_rows],
                                     net.loss)
                mini_loss[k] = tot / n
                tgt = y[(k - 1) * B:k * B]
                delta = loss_grad(stacked["a"][-1], tgt, net.loss, B)
            else:
                delta = deltas.pop((k, s))
            prop = stores[s - 1][pin[(k, 0)]] if stashed else stores[s - 1][current[s - 1]]
            g, d_in = stage_backward(layers[s - 1], prop, stacked, delta)
            for jj in range(1, n + 1):
                fwd.pop((k, 0 if stashed else jj, s), None)
            stores[s - 1][k] = stores[s - 1][current[s - 1]] - lr * g
            current[s - 1] = k
            if s > 1:
                deltas[(k, s - 1)] = d_in
            else:
                logs[k] = (mini_loss[k], [pin[(k, 0 if stashed else jj)] for jj in range(1, n + 1)],
                           int(led["update_source"][k - 1]))
        if observe:
            for s in range(W):
                for v in stores[s]:
                    held[t - 1, s, v] = 1
    for k in range(1, M + 1):
        losses.append(logs[k][0])
        pinned.append(logs[k][1])
        consumed.append(logs[k][2])
    flat = np.concatenate([stores[s][current[s]] for s in range(W)])
    return dict(params=flat, losses=np.array(losses), pinned=pinned,
                consumed=np.array(consumed), held=held, grid=grid, ledger=led)


def network_loss(net, params, x, y):
    """trainer.cpp:662-668."""
    c = stage_forward(_layers(net.widths, net.acts, 0, len(net.widths) - 1), params, x)
    return loss_mean(c["a"][-1], y, net.loss)


def network_gradient(net, params, x, y):
    """trainer.cpp:670-679."""
    layers = _layers(net.widths, net.acts, 0, len(net.widths) - 1)
    c = stage_forward(layers, params, x)
    g, _ = stage_backward(layers, params, c, loss_grad(c["a"][-1], y, net.loss, x.shape[0]))
    return g
