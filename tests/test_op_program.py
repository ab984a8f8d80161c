"""The session's op program on the host (plan-only, no GPU): the
PIPESIM_DUMP_OPS listing, and transitive pruning of cross-stream waits
(PIPESIM_PRUNE_EDGES) removing waits only -- the same kernels in the same
order on every stream -- and fusing the latency-bound stages' layers
(PIPESIM_FWD_CHAIN / PIPESIM_DGRAD_CHAIN) on C1's stage 2."""
import os
import subprocess
import sys
from collections import Counter

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = """
import sys
sys.path.insert(0, {root!r})
from paper_2410_14312_b200 import pipesim as P
net = P.NetworkSpec({widths!r}, {acts!r}, 'softmax_cross_entropy')
P.plan_memory(net, {W}, {N}, {B}, {M}, mode={mode!r})
"""


def _dump(tmp_path, name, env_extra, widths=(784, 512, 256, 10), acts=("relu", "relu", "linear"),
          W=2, N=4, B=256, M=12, mode="timeprest"):
    path = tmp_path / f"{name}.txt"
    env = dict(os.environ, PIPESIM_DUMP_OPS=str(path), **env_extra)
    code = CODE.format(root=ROOT, widths=list(widths), acts=list(acts), W=W, N=N, B=B, M=M,
                       mode=mode)
    subprocess.run([sys.executable, "-c", code], env=env, check=True, capture_output=True)
    return [line.split() for line in path.read_text().splitlines()]


def _kernels_per_stream(ops):
    per = {}
    for o in ops:
        if o[2] not in ("wait", "record", "mark"):
            per.setdefault(o[1], []).append(o[2])
    return per


@pytest.mark.parametrize("mode", ["timeprest", "pipedream"])
def test_pruning_removes_only_waits(tmp_path, mode):
    full = _dump(tmp_path, "full", {"PIPESIM_PRUNE_EDGES": "0"}, mode=mode)
    pruned = _dump(tmp_path, "pruned", {"PIPESIM_PRUNE_EDGES": "1"}, mode=mode)
    assert _kernels_per_stream(full) == _kernels_per_stream(pruned)
    nw_full = sum(o[2] == "wait" for o in full)
    nw_pruned = sum(o[2] == "wait" for o in pruned)
    assert 0 < nw_pruned < nw_full


def test_deep_net_program_pruned(tmp_path):
    kw = dict(widths=[256] * 9, acts=["relu"] * 7 + ["linear"], W=8, N=4, B=128, M=10)
    full = _dump(tmp_path, "full", {"PIPESIM_PRUNE_EDGES": "0"}, **kw)
    pruned = _dump(tmp_path, "pruned", {"PIPESIM_PRUNE_EDGES": "1"}, **kw)
    assert _kernels_per_stream(full) == _kernels_per_stream(pruned)
    assert sum(o[2] == "wait" for o in pruned) <= sum(o[2] == "wait" for o in full)


def test_c1_stage2_is_fused(tmp_path):
    ops = _dump(tmp_path, "fused", {})
    kinds = Counter(o[2] for o in ops)
    M = 12
    assert kinds["dgrad_chain"] == M  # one per stage-2 backward
    assert kinds["dgrad"] == 0        # stage 1 needs no delta
    assert kinds["fwd_chain"] >= M    # every stage-2 forward node
    unfused = _dump(tmp_path, "unfused", {"PIPESIM_FWD_CHAIN": "0", "PIPESIM_DGRAD_CHAIN": "0"})
    k2 = Counter(o[2] for o in unfused)
    assert k2["dgrad_chain"] == 0 and k2["fwd_chain"] == 0
    assert k2["dgrad"] == 2 * M
    assert k2["fwd"] == kinds["fwd"] + 2 * kinds["fwd_chain"]


def _hb_graph(ops):
    """Happens-before over op indices: stream order, and record -> wait of
    the same event (every record creates a fresh event)."""
    succ = [[] for _ in ops]
    last_on = {}
    rec_of = {}
    for i, o in enumerate(ops):
        s = o[1]
        if s in last_on:
            succ[last_on[s]].append(i)
        last_on[s] = i
        if o[2] == "record":
            rec_of[o[3]] = i
        elif o[2] == "wait":
            succ[rec_of[o[3]]].append(i)
    return succ, rec_of


def _kernel_index(ops):
    """(stream, n-th kernel on it) <-> op index."""
    fwd, back, count = {}, {}, {}
    for i, o in enumerate(ops):
        if o[2] in ("wait", "record", "mark"):
            continue
        n = count.get(o[1], 0)
        count[o[1]] = n + 1
        fwd[(o[1], n)] = i
        back[i] = (o[1], n)
    return fwd, back


@pytest.mark.parametrize("mode,kw", [
    ("timeprest", {}),
    ("pipedream", {}),
    ("timeprest", dict(widths=[256] * 9, acts=["relu"] * 7 + ["linear"], W=8, N=4, B=128,
                       M=10)),
])
def test_pruned_program_keeps_every_dependency(tmp_path, mode, kw):
    full = _dump(tmp_path, "full", {"PIPESIM_PRUNE_EDGES": "0"}, mode=mode, **kw)
    pruned = _dump(tmp_path, "pruned", {"PIPESIM_PRUNE_EDGES": "1"}, mode=mode, **kw)
    _, f_back = _kernel_index(full)
    p_fwd, _ = _kernel_index(pruned)
    _, f_rec = _hb_graph(full)
    p_succ, _ = _hb_graph(pruned)

    def prev_kernel(ops, i, stream):
        for j in range(i - 1, -1, -1):
            if ops[j][1] == stream and ops[j][0] is not None and ops[j][2] not in (
                    "wait", "record", "mark"):
                return j
        return None

    def next_kernel(ops, i, stream):
        for j in range(i + 1, len(ops)):
            if ops[j][1] == stream and ops[j][2] not in ("wait", "record", "mark"):
                return j
        return None

    reach_cache = {}

    def reaches(a, b):
        key = a
        if key not in reach_cache:
            seen, stack = {a}, [a]
            while stack:
                u = stack.pop()
                for v in p_succ[u]:
                    if v not in seen:
                        seen.add(v)
                        stack.append(v)
            reach_cache[key] = seen
        return b in reach_cache[key]

    checked = 0
    for i, o in enumerate(full):
        if o[2] != "wait":
            continue
        r = f_rec[o[3]]
        producer = prev_kernel(full, r, full[r][1])
        consumer = next_kernel(full, i, o[1])
        if producer is None or consumer is None:
            continue
        a = p_fwd[f_back[producer]]
        b = p_fwd[f_back[consumer]]
        assert reaches(a, b), (full[producer], full[consumer])
        checked += 1
    assert checked > 50


def test_spare_activation_slot_only_for_latency_bound_nets():
    """Latency-bound networks (every layer <= 1024 wide) hold one activation
    slot more per stage where consecutive mini-batches would share one (C1
    stage 2: 1 -> 2); the 16 x 4096 net keeps the minimal colouring."""
    from paper_2410_14312_b200 import pipesim as P
    c1 = P.NetworkSpec([784, 512, 256, 10], ["relu", "relu", "linear"], "softmax_cross_entropy")
    assert list(P.plan_memory(c1, 2, 4, 256, 32)["act_slots"]) == [2, 2]
    c3 = P.NetworkSpec([4096] * 17, ["relu"] * 15 + ["linear"], "softmax_cross_entropy")
    slots = list(P.plan_memory(c3, 8, 8, 1024, 32)["act_slots"])
    assert slots == [3, 3, 3, 2, 2, 2, 2, 1]
