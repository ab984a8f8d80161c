"""Python mirror of the reference's ``pipesim`` API (proj/include/pipesim/*.hpp),
bound to the B200 build through the C ABI (include/pipesim_b200.h).

Same names, argument meaning and error behaviour as the reference:
* plan layer — ``build_nf1b_schedule``, ``assign_versions``, ... — runs in
  the native host library (bit-exact with the reference);
* ``train_epoch`` / ``run_training`` execute the pipeline step on the GPU
  (hand-written sm_100a kernels); there is no CPU fallback.

Exceptions mirror errors.hpp: DomainError (with ``.field``), StructuralError,
InsufficientHorizonError, IntegrityError (``.stage_id``, ``.epoch``), IoError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np

from . import _native as N
from ._native import (DomainError, InsufficientHorizonError, IntegrityError,  # noqa: F401
                      IoError, StructuralError)
from ._session_abi import pb_epoch_out, pb_session_info, pb_train_config

ACTIVATIONS = ("linear", "relu", "tanh", "sigmoid")
LOSSES = ("mse", "softmax_cross_entropy")
SCHEDULE_MODES = ("timeprest", "pipedream")
TRAIN_MODES = ("timeprest", "pipedream", "sequential")

IDLE, FORWARD, BACKWARD = 0, 1, 2


def _L():
    return N.lib()


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# =================================================================== config
@dataclass
class SimConfig:
    """sim_config (config.hpp:32-40)."""
    workers: int = 2
    micro_batches: int = 2
    mini_batches: int = 1
    backward_cost_factor: float = 2.0
    samples_per_mini_batch: int = 64
    seed: int = 0

    def _c(self):
        return N.pb_sim_config(self.workers, self.micro_batches, self.mini_batches,
                               self.backward_cost_factor, self.samples_per_mini_batch,
                               self.seed)


def validate(cfg: SimConfig) -> None:
    """validate (config.hpp:44-62); raises DomainError naming the field."""
    c = cfg._c()
    N.check(_L().pb_validate_config(C.byref(c)))


# =================================================================== schedule
@dataclass(frozen=True)
class Task:
    """task (schedule.hpp:34-44)."""
    kind: int = IDLE
    mini: int = 0
    micro: int = 0

    def is_idle(self):
        return self.kind == IDLE

    def is_forward(self):
        return self.kind == FORWARD

    def is_backward(self):
        return self.kind == BACKWARD


class ScheduleGrid:
    """schedule_grid (schedule.hpp:49-76): worker x slot, 1-based."""

    def __init__(self, cfg: SimConfig, mode: str, cells: Optional[np.ndarray] = None):
        self._cfg = dataclasses.replace(cfg)
        self._mode = mode
        self.cells = (np.zeros((cfg.workers, 0, 3), np.int32) if cells is None
                      else np.ascontiguousarray(cells, np.int32))

    def config(self):
        return self._cfg

    def mode(self):
        return self._mode

    def workers(self):
        return self._cfg.workers

    def horizon(self):
        return self.cells.shape[1]

    def at(self, worker, slot) -> Task:
        if worker < 1 or worker > self.workers() or slot < 1 or slot > self.horizon():
            return Task()
        return Task(*(int(v) for v in self.cells[worker - 1, slot - 1]))

    def put(self, worker, slot, t: Task):
        if slot > self.horizon():
            grow = np.zeros((self.workers(), slot - self.horizon(), 3), np.int32)
            self.cells = np.concatenate([self.cells, grow], axis=1)
        self.cells[worker - 1, slot - 1] = (t.kind, t.mini, t.micro)

    def clear(self, worker, slot):
        if 1 <= worker <= self.workers() and 1 <= slot <= self.horizon():
            self.cells[worker - 1, slot - 1] = 0

    def forward_slot(self, mini, micro, stage):
        row = self.cells[stage - 1]
        hit = np.nonzero((row[:, 0] == FORWARD) & (row[:, 1] == mini) & (row[:, 2] == micro))[0]
        return int(hit[0]) + 1 if len(hit) else 0

    def backward_slot(self, mini, stage):
        row = self.cells[stage - 1]
        hit = np.nonzero((row[:, 0] == BACKWARD) & (row[:, 1] == mini))[0]
        return int(hit[0]) + 1 if len(hit) else 0

    def copy(self):
        return ScheduleGrid(self._cfg, self._mode, self.cells.copy())

    def __eq__(self, other):
        return (isinstance(other, ScheduleGrid) and self.workers() == other.workers()
                and np.array_equal(self.cells, other.cells))

    def _flat(self):
        return np.ascontiguousarray(self.cells, np.int32)


def _mode_id(mode: str) -> int:
    if mode not in SCHEDULE_MODES:
        raise ValueError(f"unknown schedule mode {mode}")
    return SCHEDULE_MODES.index(mode)


def _build(cfg: SimConfig, mode: str) -> ScheduleGrid:
    c = cfg._c()
    h = C.c_int()
    st = _L().pb_schedule_build(C.byref(c), _mode_id(mode), C.byref(h), None, 0)
    if st not in (0, 7):
        N.check(st)
    cells = np.zeros((cfg.workers, h.value, 3), np.int32)
    N.check(_L().pb_schedule_build(C.byref(c), _mode_id(mode), C.byref(h),
                                   cells.ctypes.data_as(C.POINTER(N.pb_task)), h.value))
    return ScheduleGrid(cfg, mode, cells)


def build_nf1b_schedule(cfg: SimConfig) -> ScheduleGrid:
    """build_nf1b_schedule (schedule.hpp:84, schedule.cpp:188-191)."""
    return _build(cfg, "timeprest")


def build_1f1b_schedule(cfg: SimConfig) -> ScheduleGrid:
    """build_1f1b_schedule (schedule.hpp:89, schedule.cpp:193-196)."""
    return _build(cfg, "pipedream")


VIOLATION_KINDS = ("task_invariant", "stage_continuity", "completeness", "backward_priority")


@dataclass
class Violation:
    kind: str
    message: str


@dataclass
class ValidationReport:
    violations: List[Violation] = field(default_factory=list)

    def valid(self):
        return not self.violations


def schedule_document_json(cfg: SimConfig, mode: str = "timeprest") -> str:
    """schedule_document_json(build_*_schedule(cfg), assign_versions(...))
    (export.cpp:78-139): the reference's schedule document, schema 1."""
    c = cfg._c()
    n = C.c_int64(0)
    N.check(_L().pb_schedule_document(C.byref(c), _mode_id(mode), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    N.check(_L().pb_schedule_document(C.byref(c), _mode_id(mode), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def validate_schedule(grid: ScheduleGrid, cfg: SimConfig) -> ValidationReport:
    """validate_schedule (schedule.hpp:108-109)."""
    c = cfg._c()
    n = C.c_int()
    kinds = np.zeros(4096, np.int32)
    msg = C.create_string_buffer(1 << 20)
    cells = grid._flat()
    N.check(_L().pb_schedule_validate(C.byref(c), _mode_id(grid.mode()),
                                      cells.ctypes.data_as(C.POINTER(N.pb_task)),
                                      grid.horizon(), C.byref(n), _ip(kinds), len(kinds),
                                      msg, 1 << 20))
    lines = msg.value.decode().split("\n")
    return ValidationReport([Violation(VIOLATION_KINDS[kinds[i]], lines[i])
                             for i in range(n.value)])


# =================================================================== ledger
@dataclass
class VersionLedger:
    """version_ledger (ledger.hpp:52-65); record arrays are int32 [n][4]."""
    cfg: SimConfig
    mode: str
    commits: np.ndarray          # (version, mini, stage, slot)
    pins: np.ndarray             # (mini, micro, slot, version)
    consumptions: np.ndarray     # (mini, stage, slot, version)
    update_source: np.ndarray
    full_commit_slot: np.ndarray

    def pinned_version(self, mini, micro):
        for p in self.pins:
            if p[0] == mini and p[1] == micro:
                return int(p[3])
        raise StructuralError(f"no pin recorded for mini {mini} micro {micro}")


def assign_versions(grid: ScheduleGrid, cfg: SimConfig) -> VersionLedger:
    """assign_versions (ledger.hpp:70-71)."""
    W, M = cfg.workers, cfg.mini_batches
    units = cfg.micro_batches if grid.mode() == "timeprest" else 1
    commits = np.zeros((max(M * W, 1), 4), np.int32)
    pins = np.zeros((max(M * units, 1), 4), np.int32)
    cons = np.zeros((max(M * W, 1), 4), np.int32)
    us = np.zeros(max(M, 1), np.int32)
    fcs = np.zeros(M + 1, np.int32)
    c = cfg._c()
    cells = grid._flat()
    N.check(_L().pb_assign_versions(
        C.byref(c), _mode_id(grid.mode()), cells.ctypes.data_as(C.POINTER(N.pb_task)),
        grid.horizon(), commits.ctypes.data_as(C.POINTER(N.pb_commit)),
        pins.ctypes.data_as(C.POINTER(N.pb_pin)), cons.ctypes.data_as(C.POINTER(N.pb_consume)),
        _ip(us), _ip(fcs)))
    return VersionLedger(dataclasses.replace(cfg), grid.mode(), commits[:M * W], pins[:M * units],
                         cons[:M * W], us[:M], fcs)


def measure_version_difference(ledger: VersionLedger, strict: bool = True) -> int:
    """measure_version_difference (ledger.hpp:77-78)."""
    c = ledger.cfg._c()
    v = C.c_int()
    us = np.ascontiguousarray(ledger.update_source, np.int32)
    if len(us) == 0:
        us = np.zeros(1, np.int32)
    N.check(_L().pb_measure_version_difference(C.byref(c), _ip(us), int(strict), C.byref(v)))
    return v.value


def closed_form_v(workers: int, micro_batches: int) -> int:
    """closed_form_v: floor((W+N-2)/N) (ledger.hpp:81)."""
    v = C.c_int()
    N.check(_L().pb_closed_form_v(workers, micro_batches, C.byref(v)))
    return v.value


def forward_span(workers, micro_batches, mini_ordinal) -> int:
    v = C.c_int()
    N.check(_L().pb_forward_span(workers, micro_batches, mini_ordinal, C.byref(v)))
    return v.value


def backward_span(workers) -> int:
    v = C.c_int()
    N.check(_L().pb_backward_span(workers, C.byref(v)))
    return v.value


def overlap_condition(workers, micro_batches) -> bool:
    v = C.c_int()
    N.check(_L().pb_overlap_condition(workers, micro_batches, C.byref(v)))
    return bool(v.value)


@dataclass
class SequenceDecomposition:
    sequences: List[List[int]]
    version_difference_measured: int


def decompose_sequences(ledger: VersionLedger, mini_batches: int) -> SequenceDecomposition:
    """decompose_sequences (ledger.hpp:101-102)."""
    c = ledger.cfg._c()
    us = np.ascontiguousarray(ledger.update_source, np.int32)
    n = C.c_int()
    vm = C.c_int()
    lens = np.zeros(max(mini_batches, 1), np.int32)
    minis = np.zeros(max(mini_batches, 1), np.int32)
    N.check(_L().pb_decompose_sequences(C.byref(c), _ip(us), mini_batches, C.byref(n),
                                        _ip(lens), _ip(minis), C.byref(vm)))
    seqs, pos = [], 0
    for i in range(n.value):
        seqs.append([int(v) for v in minis[pos:pos + lens[i]]])
        pos += lens[i]
    return SequenceDecomposition(seqs, vm.value)


@dataclass
class RetentionTimeline:
    """retention_timeline (ledger.hpp:110-117): intervals [W][M+1] of
    (version, retained_from_slot, freed_at_slot)."""
    intervals: np.ndarray
    peak_concurrent: List[int]
    horizon: int

    @property
    def per_stage(self):
        return self.intervals

    def retained_count(self, stage, slot):
        iv = self.intervals[stage - 1]
        return int(((iv[:, 1] <= slot) & (slot < iv[:, 2])).sum())

    def live(self, stage, slot):
        iv = self.intervals[stage - 1]
        return {int(v) for v, a, b in iv if a <= slot < b}


def build_retention_timeline(ledger: VersionLedger, grid: ScheduleGrid) -> RetentionTimeline:
    """build_retention_timeline (ledger.hpp:119-120)."""
    if grid.mode() != ledger.mode or grid.config().mini_batches != ledger.cfg.mini_batches:
        raise StructuralError("ledger does not match grid")
    cfg = ledger.cfg
    c = cfg._c()
    iv = np.zeros((cfg.workers, cfg.mini_batches + 1, 3), np.int32)
    peak = np.zeros(cfg.workers, np.int32)
    cells = grid._flat()
    pins = np.ascontiguousarray(ledger.pins, np.int32)
    N.check(_L().pb_retention_timeline(C.byref(c), _mode_id(grid.mode()),
                                       cells.ctypes.data_as(C.POINTER(N.pb_task)),
                                       grid.horizon(), pins.ctypes.data_as(C.POINTER(N.pb_pin)),
                                       iv.ctypes.data_as(C.POINTER(N.pb_interval)), _ip(peak)))
    return RetentionTimeline(iv, [int(p) for p in peak], grid.horizon())


def staleness_report(ledger: VersionLedger) -> List[int]:
    """staleness_report (ledger.hpp:138); staleness per consumption record."""
    c = ledger.cfg._c()
    out = np.zeros(len(ledger.consumptions), np.int32)
    commits = np.ascontiguousarray(ledger.commits, np.int32)
    cons = np.ascontiguousarray(ledger.consumptions, np.int32)
    N.check(_L().pb_staleness(C.byref(c), commits.ctypes.data_as(C.POINTER(N.pb_commit)),
                              cons.ctypes.data_as(C.POINTER(N.pb_consume)), _ip(out)))
    return [int(v) for v in out]


# =================================================================== model
@dataclass
class LayerSpec:
    """layer_spec (trainer.hpp:50-55)."""
    in_: int
    out: int
    act: str = "linear"

    def param_count(self):
        return self.out * self.in_ + self.out


@dataclass
class NetworkSpec:
    """network_spec (trainer.hpp:57-64)."""
    widths: List[int]
    activations: List[str]
    loss: str = "mse"

    def layer_count(self):
        return len(self.widths) - 1

    def layer(self, i):
        return LayerSpec(self.widths[i], self.widths[i + 1], self.activations[i])

    def param_count(self):
        return sum(self.layer(i).param_count() for i in range(self.layer_count()))

    def _c(self):
        w = np.ascontiguousarray(self.widths, np.int32)
        a = np.ascontiguousarray([ACTIVATIONS.index(x) for x in self.activations], np.int32)
        spec = N.pb_net_spec(self.layer_count(), _ip(w), _ip(a), LOSSES.index(self.loss))
        spec._keep = (w, a)
        return spec


@dataclass
class StageModel:
    """stage_model (trainer.hpp:71-84)."""
    stage_id: int
    first_layer: int
    layers: List[LayerSpec]
    version_store: Dict[int, np.ndarray] = field(default_factory=dict)
    current_version: int = 0

    def param_count(self):
        return sum(l.param_count() for l in self.layers)

    def params(self, version):
        if version not in self.version_store:
            raise StructuralError(f"stage {self.stage_id} does not hold version {version}")
        return self.version_store[version]

    def current_params(self):
        return self.params(self.current_version)


def partition_model(spec: NetworkSpec, workers: int) -> List[StageModel]:
    """partition_model (trainer.hpp:89-90)."""
    c = spec._c()
    fl = np.zeros(max(workers, 1), np.int32)
    nl = np.zeros(max(workers, 1), np.int32)
    N.check(_L().pb_partition_model(C.byref(c), workers, _ip(fl), _ip(nl)))
    return [StageModel(s + 1, int(fl[s]),
                       [spec.layer(l) for l in range(fl[s], fl[s] + nl[s])])
            for s in range(workers)]


def init_network_params(spec: NetworkSpec, seed: int) -> np.ndarray:
    """init_network_params (trainer.hpp:94-95)."""
    c = spec._c()
    out = np.zeros(spec.param_count())
    N.check(_L().pb_init_network_params(C.byref(c), seed, _dp(out), len(out)))
    return out


def load_network_params(stages: List[StageModel], flat, version: int) -> None:
    """load_network_params (trainer.hpp:99-100)."""
    flat = np.asarray(flat, np.float64)
    off = 0
    for st in stages:
        n = st.param_count()
        if off + n > len(flat):
            raise StructuralError("parameter vector shorter than the network")
        st.version_store = {version: flat[off:off + n].copy()}
        st.current_version = version
        off += n
    if off != len(flat):
        raise StructuralError("parameter vector longer than the network")


def gather_network_params(stages: List[StageModel]) -> np.ndarray:
    """gather_network_params (trainer.hpp:102-103)."""
    return np.concatenate([st.current_params() for st in stages]) if stages else np.zeros(0)


def digest_values(values) -> str:
    v = np.ascontiguousarray(values, np.float64)
    out = C.create_string_buffer(17)
    N.check(_L().pb_params_digest(_dp(v), len(v), out))
    return out.value.decode()


def params_digest(stages: List[StageModel]) -> str:
    """params_digest (trainer.hpp:106): FNV-1a over shortest decimals."""
    return digest_values(gather_network_params(stages))


@dataclass
class Dataset:
    """dataset (trainer.hpp:108-111): row-major x and y."""
    x: np.ndarray
    y: np.ndarray


def make_synthetic_task(samples: int, seed: int) -> Dataset:
    """make_synthetic_task (trainer.hpp:115)."""
    x = np.zeros((samples, 2))
    y = np.zeros((samples, 2))
    N.check(_L().pb_make_synthetic_task(samples, seed, _dp(x), _dp(y)))
    return Dataset(x, y)


def make_classification_task(rows, features, classes, seed=7, as_labels=False,
                             dtype=np.float64):
    """Synthetic data of SURVEY §8(d) (x ~ U[0,1), labels rng() % C)."""
    x64 = np.zeros((rows, features)) if dtype == np.float64 else None
    x32 = np.zeros((rows, features), np.float32) if dtype == np.float32 else None
    labels = np.zeros(rows, np.int32)
    N.check(_L().pb_make_classification_task(
        rows, features, classes, seed,
        _dp(x64) if x64 is not None else None,
        x32.ctypes.data_as(C.POINTER(C.c_float)) if x32 is not None else None, _ip(labels)))
    x = x64 if x64 is not None else x32
    if as_labels:
        return x, labels
    y = np.zeros((rows, classes), dtype)
    y[np.arange(rows), labels] = 1.0
    return Dataset(x, y)


@dataclass
class TrainConfig:
    """train_config (trainer.hpp:117-126)."""
    net: NetworkSpec
    workers: int = 2
    micro_batches: int = 2
    mini_batch_size: int = 20
    mini_batches: int = 10
    epochs: int = 1
    learning_rate: float = 0.05
    seed: int = 1


@dataclass
class MiniLog:
    """mini_log (trainer.hpp:133-139)."""
    mini: int = 0
    loss: float = 0.0
    pinned: List[int] = field(default_factory=list)
    consumed: int = 0
    checksum: str = ""


@dataclass
class EpochLog:
    """epoch_log (trainer.hpp:141-147)."""
    epoch: int = 0
    minis: List[MiniLog] = field(default_factory=list)
    final_checksum: str = ""
    # B200 extras (not in the reference): device-observed version trace
    device_ms: float = 0.0
    dev_fwd: Optional[np.ndarray] = None
    dev_bwd: Optional[np.ndarray] = None
    dev_current: Optional[np.ndarray] = None

    def to_text(self) -> str:
        """epoch_log::to_text (trainer.cpp:628-640)."""
        out = []
        for m in self.minis:
            out.append(f"epoch {self.epoch} mini {m.mini} loss {format_double(m.loss)} pinned"
                       + "".join(f" {p}" for p in m.pinned)
                       + f" consumed {m.consumed} checksum {m.checksum}\n")
        out.append(f"epoch {self.epoch} final checksum {self.final_checksum}\n")
        return "".join(out)


def format_double(v: float) -> str:
    """format_double (text.hpp): std::to_chars shortest round trip."""
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    r = repr(float(v))
    neg = r.startswith("-")
    r = r.lstrip("-")
    mant, _, exp = r.partition("e")
    exp = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    raw = ip + fp
    stripped = raw.lstrip("0")
    point = len(ip) + exp - (len(raw) - len(stripped))
    digits = stripped.rstrip("0") or "0"
    nd = len(digits)
    sexp = point - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + \
        ("-" if sexp < 0 else "+") + f"{abs(sexp):02d}"
    if point <= 0:
        fix = "0." + "0" * (-point) + digits
    elif point > nd:
        # trailing zeros would be needed: v is an integer, and std::to_chars
        # prints its exact digits (same length, zero difference)
        fix = str(abs(int(v)))
    elif point == nd:
        fix = digits
    else:
        fix = digits[:point] + "." + digits[point:]
    return ("-" if neg else "") + (fix if len(fix) <= len(sci) else sci)


# ------------------------------------------------------------ GPU sessions
TIMED_KERNELS = (None, "fwd", "dgrad", "wgrad")
TRANSPORTS = ("nccl", "ipc")
PRECISIONS = ("bf16", "fp32")  # bf16 tensor cores / fp32 FFMA verify mode


class Session:
    """Resident pipeline session (C ABI pb_session_*): weights, version pools
    and activation slots of every stage stay in HBM across epochs."""

    def __init__(self, net: NetworkSpec, workers, micro_batches, mini_batch_size,
                 mini_batches, learning_rate, mode="timeprest", device=0, use_graph=True,
                 snapshots=False, fwd_merge=0, rank=0, world=1, nccl_ids=b"",
                 timed_kernel=None, transport="nccl", precision="bf16", digests=False):
        if mode not in TRAIN_MODES:
            raise DomainError(f"unknown training mode: {mode}", "mode")
        self.net = net
        self.W, self.N, self.B, self.M = workers, micro_batches, mini_batch_size, mini_batches
        self.mode = mode
        self.units = micro_batches if mode == "timeprest" else 1
        cfg = pb_train_config(workers, micro_batches, mini_batch_size, mini_batches,
                              float(learning_rate), TRAIN_MODES.index(mode), device,
                              int(use_graph), int(snapshots), int(fwd_merge),
                              TIMED_KERNELS.index(timed_kernel),
                              TRANSPORTS.index(transport), PRECISIONS.index(precision),
                              int(digests))
        spec = net._c()
        h = C.c_void_p()
        if getattr(net, "layer_net", False):  # convnet.ConvNetSpec
            N.check(_L().pb_session_create_layers(C.byref(spec), C.byref(cfg), rank, world,
                                                  bytes(nccl_ids), len(nccl_ids), C.byref(h)))
        elif world > 1:
            N.check(_L().pb_session_create_dist(C.byref(spec), C.byref(cfg), rank, world,
                                                bytes(nccl_ids), len(nccl_ids), C.byref(h)))
        else:
            N.check(_L().pb_session_create(C.byref(spec), C.byref(cfg), C.byref(h)))
        self.rank, self.world = rank, world
        self._h = h
        self.snapshots = snapshots
        self.param_count = net.param_count()
        W = workers
        self._pool = np.zeros(W, np.int32)
        self._acts = np.zeros(W, np.int32)
        self._fl = np.zeros(W, np.int32)
        self._nl = np.zeros(W, np.int32)
        info = pb_session_info(0, 0, 0, 0, 0, _ip(self._pool), _ip(self._acts), _ip(self._fl),
                               _ip(self._nl))
        N.check(_L().pb_session_info_get(h, C.byref(info)))
        self.horizon = info.horizon
        self.kernels_per_epoch = info.kernels_per_epoch
        self.device_bytes = info.device_bytes
        self.pool_sizes = [int(v) for v in self._pool]
        self.act_slots = [int(v) for v in self._acts]
        self.stage_sizes = []
        for s in range(W):
            self.stage_sizes.append(sum(net.layer(l).param_count()
                                        for l in range(self._fl[s], self._fl[s] + self._nl[s])))

    def close(self):
        if getattr(self, "_h", None):
            _L().pb_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_params(self, flat):
        flat = np.ascontiguousarray(flat, np.float64)
        N.check(_L().pb_session_load_params(self._h, _dp(flat), len(flat)))

    def read_params(self) -> np.ndarray:
        out = np.zeros(self.param_count)
        N.check(_L().pb_session_read_params(self._h, _dp(out), len(out)))
        return out

    def snapshot(self, stage, version) -> np.ndarray:
        out = np.zeros(self.stage_sizes[stage - 1])
        N.check(_L().pb_session_snapshot(self._h, stage, version, _dp(out), len(out)))
        return out

    def read_version(self, stage, version) -> np.ndarray:
        """Committed weights of a version retained after the epoch (M and
        M-1 without snapshots; any committed version with snapshots)."""
        out = np.zeros(self.stage_sizes[stage - 1])
        N.check(_L().pb_session_read_version(self._h, stage, version, _dp(out), len(out)))
        return out

    @staticmethod
    def _dtype(a, labels=False):
        if labels:
            return 2
        return 0 if a.dtype == np.float64 else 1

    def upload(self, x, y, y_labels=False):
        x = np.ascontiguousarray(x)
        y = np.ascontiguousarray(y)
        if x.dtype not in (np.float64, np.float32):
            x = x.astype(np.float64)
        if y_labels:
            y = y.astype(np.int32)
        elif y.dtype not in (np.float64, np.float32):
            y = y.astype(np.float64)
        self._keep = (x, y)
        N.check(_L().pb_session_upload(self._h, x.ctypes.data, self._dtype(x), y.ctypes.data,
                                       self._dtype(y, y_labels)))

    def train_epoch_host(self, x_ptr: int, x_dtype: str, y_ptr: int, y_dtype: str):
        """One epoch from host buffers (pb_session_train_epoch): with
        page-locked buffers the upload is streamed inside the epoch (mini-batch
        k's rows copied while earlier ones compute).  x_dtype: "f64"|"f32";
        y_dtype: "f64"|"f32"|"labels"."""
        M, U, W = self.M, self.units, self.W
        r = dict(mini_loss=np.zeros(M), pinned=np.zeros(M * U, np.int32),
                 consumed=np.zeros(M, np.int32), dev_fwd=np.zeros(M * U * W, np.int32),
                 dev_bwd=np.zeros(M * W, np.int32), dev_current=np.zeros(W, np.int32))
        out = pb_epoch_out(_dp(r["mini_loss"]), _ip(r["pinned"]), _ip(r["consumed"]),
                           _ip(r["dev_fwd"]), _ip(r["dev_bwd"]), _ip(r["dev_current"]), 0.0)
        codes = {"f64": 0, "f32": 1, "labels": 2, "bf16": 3}
        N.check(_L().pb_session_train_epoch(self._h, C.c_void_p(x_ptr), codes[x_dtype],
                                            C.c_void_p(y_ptr), codes[y_dtype], C.byref(out)))
        r["device_ms"] = out.device_ms
        r["pinned"] = r["pinned"].reshape(M, U)
        r["dev_fwd"] = r["dev_fwd"].reshape(M, U, W)
        r["dev_bwd"] = r["dev_bwd"].reshape(M, W)
        return r

    def ipc_export(self) -> bytes:
        """This rank's IPC connection blob (transport="ipc")."""
        n = C.c_int64(0)
        N.check(_L().pb_session_ipc_export(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        N.check(_L().pb_session_ipc_export(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def ipc_connect(self, blobs):
        """Connect with every rank's blob (list indexed by rank)."""
        lens = (C.c_int64 * len(blobs))(*[len(b) for b in blobs])
        N.check(_L().pb_session_ipc_connect(self._h, b"".join(blobs), lens, len(blobs)))

    def trace_document(self) -> str:
        """The last epoch's schedule document with device-observed versions
        (pins; timeprest consumptions), in the reference's JSON schema."""
        n = C.c_int64(0)
        N.check(_L().pb_session_trace_document(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        N.check(_L().pb_session_trace_document(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def kernel_times_ms(self):
        """Device durations of the timed GEMM kind's launches in the last
        epoch (Session(timed_kernel=...)), from CUDA events recorded on the
        launch stream inside the epoch (inside the graph)."""
        return self.kernel_timeline()[0]

    def kernel_timeline(self):
        """(durations ms, algorithmic flops) of the timed GEMM kind's launches
        in the last epoch, in issue order."""
        n = C.c_int(0)
        N.check(_L().pb_session_kernel_times(self._h, None, None, 0, C.byref(n)))
        ms = np.zeros(max(1, n.value), np.float32)
        fl = np.zeros(max(1, n.value), np.float64)
        N.check(_L().pb_session_kernel_times(self._h, ms.ctypes.data_as(C.POINTER(C.c_float)),
                                             fl.ctypes.data_as(C.POINTER(C.c_double)),
                                             n.value, C.byref(n)))
        return ms[:n.value], fl[:n.value]

    def profile_epoch(self, max_nodes: int = 1 << 16):
        """One epoch without the CUDA graph, timed per node on the stage
        streams (the native path, with timing events).  Returns run_epoch's
        dict plus `profile`: makespan_ms, per-stage busy_ms, the node timeline
        and bubble = 1 - sum(busy) / (W * makespan) over this GPU's stages."""
        from ._session_abi import pb_epoch_profile
        M, U, W = self.M, self.units, self.W
        r = dict(mini_loss=np.zeros(M), pinned=np.zeros(M * U, np.int32),
                 consumed=np.zeros(M, np.int32), dev_fwd=np.zeros(M * U * W, np.int32),
                 dev_bwd=np.zeros(M * W, np.int32), dev_current=np.zeros(W, np.int32))
        out = pb_epoch_out(_dp(r["mini_loss"]), _ip(r["pinned"]), _ip(r["consumed"]),
                           _ip(r["dev_fwd"]), _ip(r["dev_bwd"]), _ip(r["dev_current"]), 0.0)
        busy = np.zeros(W, np.float32)
        cols = {k: np.zeros(max_nodes, np.int32) for k in ("stage", "fwd", "mini", "lo", "hi")}
        t0 = np.zeros(max_nodes, np.float32)
        t1 = np.zeros(max_nodes, np.float32)
        fp = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
        prof = pb_epoch_profile(0.0, fp(busy), max_nodes, 0, _ip(cols["stage"]),
                                _ip(cols["fwd"]), _ip(cols["mini"]), _ip(cols["lo"]),
                                _ip(cols["hi"]), fp(t0), fp(t1))
        N.check(_L().pb_session_profile_epoch(self._h, C.byref(out), C.byref(prof)))
        r["device_ms"] = out.device_ms
        r["pinned"] = r["pinned"].reshape(M, U)
        r["dev_fwd"] = r["dev_fwd"].reshape(M, U, W)
        r["dev_bwd"] = r["dev_bwd"].reshape(M, W)
        n = min(prof.n_nodes, max_nodes)
        local = busy >= 0
        mk = float(prof.makespan_ms)
        r["profile"] = dict(
            makespan_ms=mk, busy_ms=busy.tolist(),
            bubble=float(1.0 - busy[local].sum() / (local.sum() * mk)) if mk > 0 else None,
            nodes=[dict(stage=int(cols["stage"][i]), fwd=bool(cols["fwd"][i]),
                        mini=int(cols["mini"][i]), micro=(int(cols["lo"][i]), int(cols["hi"][i])),
                        start_ms=float(t0[i]), end_ms=float(t1[i])) for i in range(n)])
        return r

    def digests(self):
        """The M + 1 in-epoch digests of the last epoch (digests=True): the
        per-mini-batch checksums (mini_log::checksum), then the final one."""
        buf = C.create_string_buffer(17 * (self.M + 1))
        N.check(_L().pb_session_digests(self._h, buf, self.M + 1))
        return [buf.raw[17 * i:17 * i + 16].decode() for i in range(self.M + 1)]

    def params_digest(self, version=None):
        """params_digest of every stage's `version` (default M: after an
        epoch), computed on the device."""
        out = C.create_string_buffer(17)
        N.check(_L().pb_session_params_digest(self._h, self.M if version is None else version,
                                              out))
        return out.value.decode()

    def run_epoch(self):
        M, U, W = self.M, self.units, self.W
        r = dict(mini_loss=np.zeros(M), pinned=np.zeros(M * U, np.int32),
                 consumed=np.zeros(M, np.int32), dev_fwd=np.zeros(M * U * W, np.int32),
                 dev_bwd=np.zeros(M * W, np.int32), dev_current=np.zeros(W, np.int32))
        out = pb_epoch_out(_dp(r["mini_loss"]), _ip(r["pinned"]), _ip(r["consumed"]),
                           _ip(r["dev_fwd"]), _ip(r["dev_bwd"]), _ip(r["dev_current"]), 0.0)
        N.check(_L().pb_session_run_epoch(self._h, C.byref(out)))
        r["device_ms"] = out.device_ms
        r["pinned"] = r["pinned"].reshape(M, U)
        r["dev_fwd"] = r["dev_fwd"].reshape(M, U, W)
        r["dev_bwd"] = r["dev_bwd"].reshape(M, W)
        return r


def nccl_unique_ids(world: int) -> bytes:
    """2*(world-1) NCCL unique ids (one per pipeline boundary and direction);
    made on rank 0 and shared with the other ranks by the caller."""
    out = b""
    for _ in range(2 * (world - 1)):
        buf = C.create_string_buffer(128)
        N.check(_L().pb_nccl_unique_id(buf))
        out += buf.raw[:128]
    return out


def plan_transfers(net: NetworkSpec, workers, micro_batches, mini_batch_size, mini_batches,
                   mode="timeprest", rank=0, world=1, fwd_merge=0):
    """The point-to-point transfers rank `rank` issues in one epoch, in order:
    list of (kind 'send'|'recv', direction 0 act / 1 delta, peer, bytes).
    Host only (no GPU)."""
    cfg = pb_train_config(workers, micro_batches, mini_batch_size, mini_batches, 0.05,
                          TRAIN_MODES.index(mode), 0, 0, 0, int(fwd_merge))
    spec = net._c()
    n = C.c_int()
    N.check(_L().pb_plan_transfers(C.byref(spec), C.byref(cfg), rank, world, C.byref(n),
                                   None, None, None, None, 0))
    k = np.zeros(max(n.value, 1), np.int32)
    d = np.zeros_like(k)
    p = np.zeros_like(k)
    b = np.zeros(max(n.value, 1), np.int64)
    N.check(_L().pb_plan_transfers(C.byref(spec), C.byref(cfg), rank, world, C.byref(n),
                                   _ip(k), _ip(d), _ip(p), b.ctypes.data_as(C.POINTER(C.c_int64)),
                                   n.value))
    return [("send" if k[i] else "recv", int(d[i]), int(p[i]), int(b[i])) for i in range(n.value)]


def plan_memory(net: NetworkSpec, workers, micro_batches, mini_batch_size, mini_batches,
                mode="timeprest", rank=0, world=1, precision="bf16"):
    """Device bytes the session holds per stage, from its own arena layout
    (host only, no GPU): dict of numpy arrays `weight_bytes`, `act_bytes`,
    `pool` (weight versions held at peak), `act_slots` (mini-batch
    activation sets held at peak).  The measured counterpart of the slot
    model's memory_footprint (proj/src/metrics.cpp:73-101)."""
    cfg = pb_train_config(workers, micro_batches, mini_batch_size, mini_batches, 0.05,
                          TRAIN_MODES.index(mode), 0, 0, 0)
    cfg.precision = 1 if precision == "fp32" else 0
    spec = net._c()
    W = int(workers)
    wb = np.zeros(W, np.int64)
    ab = np.zeros(W, np.int64)
    pool = np.zeros(W, np.int32)
    acts = np.zeros(W, np.int32)
    i64p = C.POINTER(C.c_int64)
    N.check(_L().pb_plan_memory(C.byref(spec), C.byref(cfg), rank, world,
                                wb.ctypes.data_as(i64p), ab.ctypes.data_as(i64p), _ip(pool),
                                _ip(acts)))
    return {"weight_bytes": wb, "act_bytes": ab, "pool": pool, "act_slots": acts}


_SESSIONS: Dict[tuple, Session] = {}


class b200:
    """Execution knobs of the GPU build (not part of the reference API)."""
    device = int(os.environ.get("PIPESIM_B200_DEVICE", "0"))
    use_graph = True
    # per-mini-batch checksums are computed on the device inside the epoch
    digest = "automatic"         # "automatic" | "every_mini" | "final_only"
    digest_auto_limit = 1 << 40  # params; automatic above it: final only
    precision = "bf16"           # "bf16" (tensor cores) | "fp32" (FFMA verify mode)


def _session_for(cfg: TrainConfig, mode: str, snapshots: bool, digests: bool = False) -> Session:
    key = (tuple(cfg.net.widths), tuple(cfg.net.activations), cfg.net.loss, cfg.workers,
           cfg.micro_batches, cfg.mini_batch_size, cfg.mini_batches, float(cfg.learning_rate),
           mode, snapshots, digests, b200.device, b200.use_graph, b200.precision)
    s = _SESSIONS.get(key)
    if s is None:
        if len(_SESSIONS) > 8:
            for v in _SESSIONS.values():
                v.close()
            _SESSIONS.clear()
        s = Session(cfg.net, cfg.workers, cfg.micro_batches, cfg.mini_batch_size,
                    cfg.mini_batches, cfg.learning_rate, mode, b200.device, b200.use_graph,
                    snapshots, precision=b200.precision, digests=digests)
        _SESSIONS[key] = s
    return s


def _check_train_config(cfg: TrainConfig, data: Dataset):
    """check_train_config (trainer.cpp:351-370)."""
    if cfg.mini_batch_size < 1 or cfg.mini_batches < 1:
        raise DomainError("mini-batch count/size must be >= 1", "mini_batches")
    if cfg.micro_batches < 1:
        raise DomainError("micro-batch count must be >= 1", "micro_batches")
    if cfg.mini_batch_size % cfg.micro_batches != 0:
        raise DomainError(f"mini-batch size {cfg.mini_batch_size} is not divisible by "
                          f"micro-batch count {cfg.micro_batches}", "mini_batch_size")
    rows = np.asarray(data.x).shape[0]
    if rows != cfg.mini_batches * cfg.mini_batch_size:
        raise StructuralError(f"dataset holds {rows} rows, expected M*Ms = "
                              f"{cfg.mini_batches * cfg.mini_batch_size}")
    if np.asarray(data.x).shape[1] != cfg.net.widths[0] or \
            np.asarray(data.y).shape[1] != cfg.net.widths[-1]:
        raise StructuralError("dataset width does not match the network")


def train_epoch(stages: List[StageModel], data: Dataset, cfg: TrainConfig, mode: str,
                epoch: int, observer: Optional[Callable] = None) -> EpochLog:
    """train_epoch (trainer.hpp:159-161) — the pipeline step on B200.

    stages are mutated in place like the reference: version 0 := the current
    weights (rebase), then one committed version per mini-batch; after return
    version_store holds exactly the versions the retention rule keeps live.
    """
    _check_train_config(cfg, data)
    if len(stages) != cfg.workers:
        raise StructuralError("stage count does not match workers")
    if mode not in TRAIN_MODES:
        raise DomainError(f"unknown training mode: {mode}", "mode")
    if mode != "sequential":
        validate(SimConfig(cfg.workers, cfg.micro_batches, cfg.mini_batches,
                           samples_per_mini_batch=cfg.mini_batch_size, seed=cfg.seed))
    P = cfg.net.param_count()
    want = b200.digest
    if want == "automatic":
        want = "every_mini" if P <= b200.digest_auto_limit else "final_only"
    snaps = observer is not None
    if mode != "sequential" and not snaps:
        # retained versions older than M-1 (1F1B stashes) are read from snapshots
        sc0 = SimConfig(cfg.workers, cfg.micro_batches, cfg.mini_batches,
                        samples_per_mini_batch=cfg.mini_batch_size)
        g0 = _build(sc0, mode)
        t0 = build_retention_timeline(assign_versions(g0, sc0), g0)
        snaps = any(b > t0.horizon and v < cfg.mini_batches - 1
                    for iv in t0.intervals for v, a, b in iv)
    sess = _session_for(cfg, mode, snaps, want == "every_mini")
    sess.load_params(gather_network_params(stages))
    sess.upload(data.x, data.y)
    r = sess.run_epoch()
    M, W = cfg.mini_batches, cfg.workers
    final = sess.read_params()

    # device-observed versions must equal the ledger (bit-exact trace)
    pins = r["pinned"]
    if not (np.array_equal(r["dev_fwd"], np.repeat(pins[:, :, None], W, axis=2))
            and np.all(r["dev_current"] == M)):
        raise StructuralError("device version trace diverged from the ledger")

    offs = np.cumsum([0] + sess.stage_sizes)
    log = EpochLog(epoch=epoch, device_ms=r["device_ms"], dev_fwd=r["dev_fwd"],
                   dev_bwd=r["dev_bwd"], dev_current=r["dev_current"])

    grid = ledger = timeline = None
    if mode != "sequential":
        sc = SimConfig(W, cfg.micro_batches, M, samples_per_mini_batch=cfg.mini_batch_size)
        grid = _build(sc, mode)
        ledger = assign_versions(grid, sc)
        timeline = build_retention_timeline(ledger, grid)

    # checksums: computed on the device (digest_dev.hpp) -- in the epoch after
    # every stage-1 commit (trainer.cpp:492-501), or the final one now
    dig = sess.digests() if want == "every_mini" else None
    for k in range(1, M + 1):
        log.minis.append(MiniLog(k, float(r["mini_loss"][k - 1]),
                                 [int(v) for v in r["pinned"][k - 1]],
                                 int(r["consumed"][k - 1]), dig[k - 1] if dig else ""))
    log.final_checksum = dig[M] if dig else sess.params_digest(M)

    # install the final state into the stage objects
    for s, st in enumerate(stages):
        cur = final[offs[s]:offs[s + 1]].copy()
        store = {M: cur}
        if timeline is not None:
            for v, a, b in timeline.intervals[s]:
                if b > timeline.horizon and v != M:
                    # retained past the horizon (trainer.cpp:420-429): M-1 is
                    # always readable, older 1F1B stashes need snapshots
                    store[int(v)] = sess.read_version(s + 1, int(v))
        st.version_store = store
        st.current_version = M

    if observer is not None and timeline is not None:
        # replay of the plan's retention timeline with the committed snapshots
        H = timeline.horizon
        for t in range(1, H + 1):
            view = []
            for s, st in enumerate(stages):
                live = timeline.live(s + 1, t)
                cur_v = max(live) if live else 0
                vs = {v: sess.snapshot(s + 1, v) for v in live}
                view.append(StageModel(st.stage_id, st.first_layer, st.layers, vs, cur_v))
            observer(t, view)
    return log


def network_loss(spec: NetworkSpec, params, data: Dataset) -> float:
    """network_loss (trainer.hpp:169-170) on B200: a single-stage sequential
    forward with learning rate 0."""
    rows = np.asarray(data.x).shape[0]
    s = Session(spec, 1, 1, rows, 1, 0.0, "sequential", b200.device, False, False)
    try:
        s.load_params(params)
        s.upload(data.x, data.y)
        return float(s.run_epoch()["mini_loss"][0])
    finally:
        s.close()


# ================================================================ checkpoint
def checkpoint_filename(stage_id: int, epoch: int) -> str:
    """checkpoint_filename (checkpoint.hpp:44)."""
    return f"stage-{stage_id}-epoch-{epoch}.ckpt"


def checkpoint_stage(stage: StageModel, loss: str, epoch: int, path: str) -> None:
    """checkpoint_stage (checkpoint.hpp:29-31): the reference's text format
    (checkpoint.cpp:39-67), written by the native library."""
    lay = np.ascontiguousarray([[l.in_, l.out, ACTIVATIONS.index(l.act)] for l in stage.layers],
                               np.int32)
    p = np.ascontiguousarray(stage.current_params(), np.float64)
    N.check(_L().pb_checkpoint_stage(stage.stage_id, stage.first_layer, len(stage.layers),
                                     _ip(lay), stage.current_version, _dp(p), len(p),
                                     LOSSES.index(loss), epoch, os.fsencode(path)))


@dataclass
class RestoredStage:
    """restored_stage (checkpoint.hpp:33-38)."""
    stage: StageModel
    loss: str
    epoch: int


def restore_stage(path: str, expected_stage: int = 0, expected_epoch: int = 0,
                  max_layers: int = 4096, max_values: int = 0) -> RestoredStage:
    """restore_stage (checkpoint.hpp:40-42): strict parse, digest check,
    IntegrityError on a missing / truncated / tampered / mismatched file."""
    if max_values <= 0:
        max_values = max(1, os.path.getsize(path) // 2) if os.path.exists(path) else 1
    info = N.pb_restored_stage()
    lay = np.zeros((max_layers, 3), np.int32)
    vals = np.zeros(max_values)
    N.check(_L().pb_restore_stage(os.fsencode(path), expected_stage, expected_epoch,
                                  C.byref(info), _ip(lay), max_layers, _dp(vals), len(vals)))
    layers = [LayerSpec(int(a), int(b), ACTIVATIONS[int(c)]) for a, b, c in lay[:info.n_layers]]
    st = StageModel(info.stage_id, info.first_layer, layers,
                    {info.version: vals[:info.n_values].copy()}, info.version)
    return RestoredStage(st, LOSSES[info.loss], info.epoch)


@dataclass
class TrainRunResult:
    """train_run_result (trainer.hpp:175-183)."""
    logs: List[EpochLog]
    first_epoch: int
    final_checksum: str


def run_training(cfg: TrainConfig, mode: str, data: Dataset, checkpoint_dir: str = "",
                 resume: bool = False) -> TrainRunResult:
    """run_training (trainer.hpp:185-188; trainer.cpp:704-758): epochs of
    train_epoch on B200, a checkpoint per stage after every epoch, and resume
    from the newest epoch that has any stage file (a missing sibling stage
    file is an IntegrityError)."""
    _check_train_config(cfg, data)
    stages = partition_model(cfg.net, cfg.workers)
    load_network_params(stages, init_network_params(cfg.net, cfg.seed), 0)
    first = 1
    if resume and checkpoint_dir:
        newest = 0
        for e in range(cfg.epochs, 0, -1):
            if any(os.path.exists(os.path.join(checkpoint_dir, checkpoint_filename(s, e)))
                   for s in range(1, cfg.workers + 1)):
                newest = e
                break
        if newest > 0:
            for s in range(1, cfg.workers + 1):
                path = os.path.join(checkpoint_dir, checkpoint_filename(s, newest))
                if not os.path.exists(path):
                    raise IntegrityError(f"resume refused: checkpoint for stage {s} epoch "
                                         f"{newest} is missing", s, newest)
                r = restore_stage(path, s, newest, max_values=stages[s - 1].param_count())
                stages[s - 1].version_store = {0: r.stage.current_params()}
                stages[s - 1].current_version = 0
            first = newest + 1
    logs = []
    for e in range(first, cfg.epochs + 1):
        logs.append(train_epoch(stages, data, cfg, mode, e))
        if checkpoint_dir:
            os.makedirs(checkpoint_dir, exist_ok=True)
            for st in stages:
                checkpoint_stage(st, cfg.net.loss, e,
                                 os.path.join(checkpoint_dir,
                                              checkpoint_filename(st.stage_id, e)))
    return TrainRunResult(logs, first, params_digest(stages))
