"""Host-side mirror of the reference's hot-path API (gqsgd::, proj/include/gqsgd).

Names, argument meaning and error classes follow the reference so callers
(and the parity tests) read like proj/tests/*.cpp:

    reference (C++)                          here (CUDA through libgq_b200.so)
    ---------------------------------------  --------------------------------------
    GqsgdConfig        algorithm.hpp:21-32   GqsgdConfig
    standard_lane_width algorithm.cpp:22-29  standard_lane_width / plan_path
    check_width        exp_arith.cpp:24-41   check_width
    local_norm_stat    norms.cpp:52-62       local_norm_stats (all shards, one launch)
    norm_allreduce_inproc collectives.cpp:210 global_norm
    quantize_shard+encode quantizer.cpp:8-48 quantize_shard (returns wire lanes)
    allreduce_inproc   collectives.cpp:155   allreduce_inproc (fused schedule replay)
                                             allreduce_schedule (event interpreter)
    PayloadOps/IntSumOps/TokenReduceOps      PayloadOps/IntSumOps/TokenReduceOps
                       collectives.hpp:39-105  (device plugin: gq_combine_lanes)
    tree/ring_schedule topology.cpp:19-72    tree_schedule / ring_schedule
    chunk_lane_range   topology.cpp:99-106   chunk_lane_range
    decode_dense_*     algorithm.cpp:84-110  decode
    gqsgd_mean         algorithm.cpp:127-228 gqsgd_mean (dense and cfg.sparse)
    to_sparse+serialize_sparse               sparse_payload
    accumulate_sparse  quantizer.cpp:92-110  sparse_accumulate
    baseline_mean      algorithm.cpp:303-340 baseline_mean

Tensors are torch CUDA tensors (torch is used only for device memory and
streams). Every public call synchronises and raises the reference's
exception class on error; `InprocSync` is the allocation-free, sync-free
engine the benchmark drives.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import torch

from . import _lib
from ._lib import (GQ_NORM_INF, DomainError, InvalidArgument, LaneOverflow,  # noqa: F401
                   RuntimeFailure, check, lib, ptr_array)

NORM_INF = GQ_NORM_INF


class LevelKind(IntEnum):
    Standard = 0
    Exponential = 1


class TopologyKind(IntEnum):
    Tree = 0
    Ring = 1


@dataclass(frozen=True)
class NormSpec:
    q: int = NORM_INF
    p: int = NORM_INF


@dataclass
class GqsgdConfig:
    """gqsgd::GqsgdConfig (algorithm.hpp:21-32); dense paths only."""
    workers: int = 4
    scheme: LevelKind = LevelKind.Exponential
    s: int = 7
    norm: NormSpec = field(default_factory=NormSpec)
    sparse: bool = False
    width_bits: int = 8
    topo: TopologyKind = TopologyKind.Tree
    seed: int = 1

    def to_c(self) -> _lib.GqConfig:
        if self.sparse:
            raise InvalidArgument("the sparse allgather path has no dense plan (use sparse_lane_width)")
        return _lib.GqConfig(self.workers, int(self.scheme), self.s, self.norm.q, self.norm.p,
                             self.width_bits, int(self.topo), 0, self.seed)


@dataclass
class Plan:
    lane_width: int
    shift: int
    m: int
    max_e: int


@dataclass
class MeanResult:
    """gqsgd::MeanResult (algorithm.hpp:36-44) for the device path."""
    mean: torch.Tensor            # fp32 [d], identical for every worker
    norm: float
    lane_width_used: int
    stats: torch.Tensor           # per-worker norm statistics (f64)
    summed_lanes: torch.Tensor    # aggregated wire lanes (uint8)


def ceil_log2(v: int) -> int:
    """exp_arith.cpp:8-17"""
    if v == 0:
        raise InvalidArgument("ceil_log2(0)")
    return (v - 1).bit_length()


def prescale_shift(n: int) -> int:
    """exp_arith.cpp:19-22"""
    if n == 0:
        raise InvalidArgument("worker count must be >= 1")
    return ceil_log2(2 * n)


def check_width(kind: LevelKind, s: int, n: int, width_bits: int) -> bool:
    """exp_arith.cpp:24-41 (width_bits > 32 is refused for both kinds, so
    standard_lane_width never reaches its 64-bit candidate)"""
    if s == 0 or n == 0 or width_bits < 2 or width_bits > 32:
        return False
    cap = 1 << (width_bits - 1)
    if kind == LevelKind.Standard:
        return n * (s + 1) <= cap
    return s + 1 + ceil_log2(n) <= cap


def plan_path(cfg: GqsgdConfig) -> Plan:
    """plan_path (algorithm.cpp:40-67) as the device library applies it."""
    p = _lib.GqPlan()
    c = cfg.to_c()
    check(lib().gq_plan_path(C.byref(c), C.byref(p)))
    return Plan(p.lane_width, p.shift, p.m, p.max_e)


def standard_lane_width(s: int, n: int, at_least: int) -> int | None:
    """algorithm.cpp:22-29 (plus the 4-bit extension when at_least == 4)."""
    try:
        return plan_path(GqsgdConfig(workers=n, scheme=LevelKind.Standard, s=s,
                                     width_bits=at_least)).lane_width
    except InvalidArgument:
        return None


def lane_bytes(d: int, width: int) -> int:
    return int(lib().gq_lane_bytes(d, width))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.GQ_DTYPE_F32
    if t.dtype == torch.float64:
        return _lib.GQ_DTYPE_F64
    raise InvalidArgument("gradients must be float32 or float64")


def _check_shards(shards) -> tuple[int, int]:
    if len(shards) == 0:
        raise InvalidArgument("shard count does not match the worker count")
    d = shards[0].numel()
    dt = _dtype_code(shards[0])
    for x in shards:
        if not x.is_cuda or not x.is_contiguous():
            raise InvalidArgument("shards must be contiguous CUDA tensors")
        if x.numel() != d:
            raise InvalidArgument("shard dimensions disagree")
        if _dtype_code(x) != dt:
            raise InvalidArgument("shard dtypes disagree")
    return d, dt


class _ErrWord:
    """One device uint32 error word per device (the C-ABI `err`)."""
    _words: dict[int, torch.Tensor] = {}

    @classmethod
    def get(cls, device: torch.device) -> torch.Tensor:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        w = cls._words.get(idx)
        if w is None:
            w = torch.zeros(1, dtype=torch.int32, device=f"cuda:{idx}")
            cls._words[idx] = w
        return w


def _sync_check(err: torch.Tensor) -> None:
    check(lib().gq_check(err.data_ptr(), _stream()))


def local_norm_stats(shards, spec: NormSpec = NormSpec()) -> torch.Tensor:
    """local_norm_stat (norms.cpp:52-62) of every shard -> f64 device tensor."""
    stats, _ = global_norm(shards, spec, fold=False)
    return stats


def global_norm(shards, spec: NormSpec = NormSpec(), fold: bool = True):
    """Per-worker stats and the tree-folded global scale
    (norm_allreduce_inproc, collectives.cpp:210-233)."""
    d, dt = _check_shards(shards)
    n = len(shards)
    dev = shards[0].device
    err = _ErrWord.get(dev)
    ws = torch.zeros(int(lib().gq_norm_workspace_bytes(n, d)), dtype=torch.uint8, device=dev)
    stats = torch.empty(n, dtype=torch.float64, device=dev)
    norm = torch.empty(1, dtype=torch.float64, device=dev)
    arr = ptr_array([x.data_ptr() for x in shards])
    check(lib().gq_norm(arr, dt, n, d, spec.q, spec.p, stats.data_ptr(),
                        norm.data_ptr() if fold else None, ws.data_ptr(), err.data_ptr(), _stream()))
    _sync_check(err)
    return stats, (norm if fold else None)


def combine_norm_stats(stats: torch.Tensor, spec: NormSpec = NormSpec()) -> torch.Tensor:
    """Tree-order fold + root of device stats (norms.cpp:64-75 via the tree)."""
    norm = torch.empty(1, dtype=torch.float64, device=stats.device)
    check(lib().gq_norm_combine(stats.data_ptr(), stats.numel(), spec.q, spec.p,
                                norm.data_ptr(), _stream()))
    torch.cuda.current_stream().synchronize()
    return norm


def _norm_tensor(norm, device) -> torch.Tensor:
    if isinstance(norm, torch.Tensor):
        return norm.to(device=device, dtype=torch.float64).reshape(1)
    return torch.tensor([float(norm)], dtype=torch.float64, device=device)


def quantize_shard(x: torch.Tensor, norm, kind: LevelKind, s: int, seed: int, worker: int,
                   round: int, width_bits: int = 8, n_total: int = 1) -> torch.Tensor:
    """quantize_shard (quantizer.cpp:8-48) + lane encoding (algorithm.cpp:69-82 /
    exp_arith.cpp:126-160): returns the worker's wire lanes (uint8 tensor of
    lane_bytes(d, width_bits) bytes; the payload is the first ceil(d*w/8))."""
    d, dt = _check_shards([x])
    dev = x.device
    err = _ErrWord.get(dev)
    nt = _norm_tensor(norm, dev)
    out = torch.zeros(lane_bytes(d, width_bits), dtype=torch.uint8, device=dev)
    ids = (C.c_uint32 * 1)(worker)
    check(lib().gq_quantize(ptr_array([x.data_ptr()]), dt, 1, ids, d, nt.data_ptr(), int(kind), s,
                            n_total, width_bits, seed, round, ptr_array([out.data_ptr()]),
                            err.data_ptr(), _stream()))
    _sync_check(err)
    return out


def allreduce_inproc(lanes, d: int, kind: LevelKind, width_bits: int, s: int,
                     topo: TopologyKind = TopologyKind.Tree, seed: int = 1, round: int = 0,
                     lane_begin: int = 0, lane_end: int | None = None) -> torch.Tensor:
    """allreduce_inproc (collectives.cpp:155-190) with IntSumOps / TokenReduceOps:
    returns the aggregated lanes every worker holds (lanes [lane_begin, lane_end))."""
    n = len(lanes)
    dev = lanes[0].device
    err = _ErrWord.get(dev)
    end = d if lane_end is None else lane_end
    out = torch.zeros(lane_bytes(d, width_bits), dtype=torch.uint8, device=dev)
    check(lib().gq_reduce_lanes(ptr_array([t.data_ptr() for t in lanes]), n, d, lane_begin, end,
                                int(kind), width_bits, s, int(topo), seed, round, None,
                                out.data_ptr(), None, None, 0.0, err.data_ptr(), _stream()))
    _sync_check(err)
    return out


def decode(lanes: torch.Tensor, d: int, norm, kind: LevelKind, s: int, n: int,
           width_bits: int, param: torch.Tensor | None = None, lr: float = 0.0) -> torch.Tensor:
    """decode_dense_std / decode_dense_exp (algorithm.cpp:84-110) -> fp32 mean;
    with `param`, also param -= lr * mean (trainer.cpp:335)."""
    dev = lanes.device
    err = _ErrWord.get(dev)
    nt = _norm_tensor(norm, dev)
    out = torch.empty(d, dtype=torch.float32, device=dev)
    check(lib().gq_dequant(lanes.data_ptr(), 0, d, nt.data_ptr(), int(kind), s, n, width_bits,
                           out.data_ptr(), param.data_ptr() if param is not None else None,
                           float(lr), err.data_ptr(), _stream()))
    _sync_check(err)
    return out


# ---------------------------------------------------------------------------
# Schedules (topology.cpp:19-106) and the PayloadOps plugin (collectives.hpp:39-48)
# ---------------------------------------------------------------------------
REDUCE, COPY = 0, 1


@dataclass(frozen=True)
class CommEvent:
    """gqsgd::CommEvent (topology.hpp:24-30)."""
    step: int
    src: int
    dst: int
    op: int = REDUCE
    chunk: int = 0


@dataclass
class Schedule:
    """gqsgd::Schedule (topology.hpp:32-37)."""
    workers: int
    steps: int = 0
    chunks: int = 1
    events: list = field(default_factory=list)


def tree_schedule(workers: int) -> Schedule:
    """Recursive halving onto rank 0, then the mirrored broadcast (topology.cpp:19-43)."""
    if workers == 0:
        raise InvalidArgument("worker count must be >= 1")
    sched = Schedule(workers, 0, 1)
    if workers == 1:
        return sched
    height = ceil_log2(workers)
    for t in range(height):
        span = 1 << t
        for r in range(span, workers, 2 * span):
            sched.events.append(CommEvent(t, r, r - span, REDUCE, 0))
    for t in range(height):
        span = 1 << (height - 1 - t)
        for r in range(0, workers - span, 2 * span):
            sched.events.append(CommEvent(height + t, r, r + span, COPY, 0))
    sched.steps = 2 * height
    return sched


def ring_schedule(workers: int) -> Schedule:
    """Reduce-scatter then allgather around the ring, n chunks (topology.cpp:45-72)."""
    if workers == 0:
        raise InvalidArgument("worker count must be >= 1")
    n = workers
    sched = Schedule(n, 0, n)
    if n == 1:
        return sched
    for t in range(n - 1):
        for r in range(n):
            sched.events.append(CommEvent(t, r, (r + 1) % n, REDUCE, (r + n - t % n) % n))
    for t in range(n - 1):
        for r in range(n):
            sched.events.append(CommEvent(n - 1 + t, r, (r + 1) % n, COPY, (r + 1 + n - t % n) % n))
    sched.steps = 2 * (n - 1)
    return sched


def make_schedule(kind: TopologyKind, workers: int) -> Schedule:
    """topology.cpp:74-77"""
    return tree_schedule(workers) if kind == TopologyKind.Tree else ring_schedule(workers)


def chunk_lane_range(lanes: int, chunks: int, c: int) -> tuple[int, int]:
    """topology.cpp:99-106"""
    if chunks == 0 or c >= chunks:
        raise InvalidArgument("bad chunk index")
    return lanes * c // chunks, lanes * (c + 1) // chunks


@dataclass
class TrafficReport:
    """gqsgd::TrafficReport (collectives.hpp:19-34), payload bytes only."""
    bytes_sent: list = field(default_factory=list)
    total_bytes: int = 0
    messages: int = 0
    steps: int = 0
    reduce_invocations: int = 0

    def add_send(self, worker: int, nbytes: int) -> None:
        if worker >= len(self.bytes_sent):
            self.bytes_sent.extend([0] * (worker + 1 - len(self.bytes_sent)))
        self.bytes_sent[worker] += nbytes
        self.total_bytes += nbytes
        self.messages += 1


class PayloadOps:
    """gqsgd::PayloadOps (collectives.hpp:39-48): element-typed combining of
    raw lanes, a pure function of (acc, in, round, step, dst, elem_offset).
    Here acc / in are CUDA uint8 tensors (views) and combine() is one
    gq_combine_lanes launch; device errors surface at the next check()."""
    kind: int
    width_bits: int
    s: int = 1
    n: int = 1
    seed: int = 1

    def lane_bytes(self) -> int:
        return self.width_bits // 8

    def combine(self, acc: torch.Tensor, inp: torch.Tensor, round: int, step: int, dst: int,
                elem_offset: int, err: torch.Tensor | None = None, stream: int | None = None) -> None:
        if acc.numel() != inp.numel():
            raise InvalidArgument("payload spans differ in size")
        lanes = acc.numel() * 8 // self.width_bits
        e = err if err is not None else _ErrWord.get(acc.device)
        check(lib().gq_combine_lanes(acc.data_ptr(), inp.data_ptr(), lanes, elem_offset, self.kind,
                                     self.width_bits, self.s, self.n, self.seed, round, step, dst,
                                     e.data_ptr(), _stream() if stream is None else stream))


class IntSumOps(PayloadOps):
    """IntSumOps (collectives.hpp:52-63, collectives.cpp:60-81) on the device."""

    def __init__(self, width_bits: int):
        if width_bits not in (8, 16, 32, 64):
            raise InvalidArgument("integer lane width must be 8, 16, 32, or 64 bits")
        self.kind, self.width_bits = 0, width_bits


class TokenReduceOps(PayloadOps):
    """TokenReduceOps (collectives.hpp:92-105, collectives.cpp:125-153) on the
    device: the k draw keyed (round, step<<32|dst, lane) with the given seed."""

    def __init__(self, s: int, n: int, width_bits: int, seed: int):
        if width_bits not in (8, 16, 32):
            raise InvalidArgument("token lane width must be 8, 16, or 32 bits")
        if not check_width(LevelKind.Exponential, s, n, width_bits):
            raise InvalidArgument("refused configuration: exponent range does not fit the lane width")
        self.kind, self.width_bits, self.s, self.n, self.seed = 1, width_bits, s, n, seed


def allreduce_schedule(payloads, sched: Schedule, ops: PayloadOps, round: int):
    """allreduce_inproc (collectives.cpp:155-190) driven event by event with a
    device PayloadOps: any schedule, the reference's interpreter semantics
    (the fused replay in allreduce_inproc()/gq_reduce_lanes is the fast path
    for the tree and ring). Payloads are modified in place; returns the
    TrafficReport after synchronising and raising device errors."""
    n = sched.workers
    if len(payloads) != n:
        raise InvalidArgument("payload count does not match the schedule")
    lb = ops.lane_bytes()
    nbytes = payloads[0].numel() if payloads else 0
    for p in payloads:
        if p.numel() != nbytes or nbytes % lb:
            raise InvalidArgument("payloads must share a lane-aligned size")
    lanes = nbytes // lb
    rep = TrafficReport(bytes_sent=[0] * n, steps=sched.steps)
    err = _ErrWord.get(payloads[0].device)
    for ev in sched.events:
        b, e = chunk_lane_range(lanes, sched.chunks, ev.chunk)
        dst = payloads[ev.dst][b * lb:e * lb]
        src = payloads[ev.src][b * lb:e * lb]
        if ev.op == REDUCE:
            if e > b:
                ops.combine(dst, src, round, ev.step, ev.dst, b, err)
            rep.reduce_invocations += 1
        else:
            dst.copy_(src)
        rep.add_send(ev.src, (e - b) * lb)
    _sync_check(err)
    return rep


class InprocSync:
    """Preallocated n-worker gradient sync on one device: the engine behind
    gqsgd_mean and the benchmark. `run()` only launches (3 kernels, no sync,
    no allocation); call `check()` to surface device errors."""

    def __init__(self, cfg: GqsgdConfig, d: int, device, dtype=torch.float32, kdraws: bool = True):
        self.cfg = cfg
        self.c_cfg = cfg.to_c()
        self.plan = plan_path(cfg)
        self.d = d
        self.device = torch.device(device)
        self.dtype_code = _lib.GQ_DTYPE_F32 if dtype == torch.float32 else _lib.GQ_DTYPE_F64
        n = cfg.workers
        lb = lane_bytes(d, self.plan.lane_width)
        self.lane_bufs = [torch.zeros(lb, dtype=torch.uint8, device=self.device) for _ in range(n)]
        self.result_lanes = torch.zeros(lb, dtype=torch.uint8, device=self.device)
        self.mean = torch.zeros(d, dtype=torch.float32, device=self.device)
        self.stats = torch.zeros(n, dtype=torch.float64, device=self.device)
        self.norm = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.workspace = torch.zeros(int(lib().gq_norm_workspace_bytes(n, d)), dtype=torch.uint8,
                                     device=self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._lane_arr = ptr_array([b.data_ptr() for b in self.lane_bufs])
        self._setup_kdraws(kdraws)

    def _setup_kdraws(self, use: bool) -> None:
        """Exponential tree path: the k draws are filled by the norm launch
        (gq_norm_kdraws) and read by the reduce (gq_reduce_lanes_kdraws)."""
        self.kd = None
        cfg = self.cfg
        device_orders = cfg.norm.q in (2, NORM_INF, _lib.GQ_NORM_L2_SEQUENTIAL) and cfg.norm.p in (2, NORM_INF)
        if not use or not device_orders:  # other orders take gq_norm's host step
            return
        spec = _lib.GqKdraws(None, cfg.workers, int(cfg.scheme), self.plan.lane_width, cfg.s, int(cfg.topo), 0,
                             0, self.d, cfg.seed, 0)
        nbytes = int(lib().gq_kdraws_bytes(C.byref(spec)))
        if nbytes:
            self.kbuf = torch.empty(nbytes // 4, dtype=torch.int32, device=self.device)
            spec.buf = self.kbuf.data_ptr()
            self.kd = spec
            self._ids = (C.c_uint32 * cfg.workers)(*range(cfg.workers))

    def run(self, shards, round: int, param: torch.Tensor | None = None, lr: float = 0.0,
            write_mean: bool = True, write_lanes: bool = True, stream: int | None = None) -> None:
        arr = ptr_array([x.data_ptr() for x in shards])
        sp = _stream() if stream is None else stream
        if self.kd is not None:
            L, cfg, kd, n = lib(), self.cfg, self.kd, self.cfg.workers
            kd.round = round
            check(L.gq_norm_kdraws(arr, self.dtype_code, n, self.d, cfg.norm.q, cfg.norm.p, self.stats.data_ptr(),
                                   self.norm.data_ptr(), self.workspace.data_ptr(), self.err.data_ptr(),
                                   C.byref(kd), sp))
            check(L.gq_quantize(arr, self.dtype_code, n, self._ids, self.d, self.norm.data_ptr(), int(cfg.scheme),
                                cfg.s, n, self.plan.lane_width, cfg.seed, round, self._lane_arr,
                                self.err.data_ptr(), sp))
            check(L.gq_reduce_lanes_kdraws(
                self._lane_arr, n, self.d, 0, self.d, int(cfg.scheme), self.plan.lane_width, cfg.s, int(cfg.topo),
                cfg.seed, round, self.norm.data_ptr(), self.result_lanes.data_ptr() if write_lanes else None,
                self.mean.data_ptr() if write_mean else None, param.data_ptr() if param is not None else None,
                float(lr), self.err.data_ptr(), C.byref(kd), sp))
            return
        check(lib().gq_mean_inproc(
            arr, self.dtype_code, self.d, C.byref(self.c_cfg), round, self._lane_arr,
            self.result_lanes.data_ptr() if write_lanes else None,
            self.mean.data_ptr() if write_mean else None,
            param.data_ptr() if param is not None else None, float(lr),
            self.stats.data_ptr(), self.norm.data_ptr(), self.workspace.data_ptr(),
            self.err.data_ptr(), _stream() if stream is None else stream))

    def check(self) -> None:
        check(lib().gq_check(self.err.data_ptr(), _stream()))

    def graph(self, shards, first_round: int, param: torch.Tensor | None = None, lr: float = 0.0,
              write_mean: bool = True, write_lanes: bool = True) -> "SyncGraph":
        """Capture the whole sync for these shard buffers as one CUDA graph;
        each SyncGraph.launch() is run(shards, round) for round = first_round,
        first_round + 1, ... (the round lives in device memory)."""
        return SyncGraph(self, shards, first_round, param, lr, write_mean, write_lanes)


class SyncGraph:
    """gq_graph_mean_inproc: norm (+ k draws) -> quantize -> reduce/decode ->
    round += 1 as a single graph launch (small-d syncs are launch-bound)."""

    def __init__(self, eng: InprocSync, shards, first_round: int, param, lr: float, write_mean: bool,
                 write_lanes: bool):
        self.eng = eng
        self.handle = None
        self.round = torch.tensor([first_round], dtype=torch.int64, device=eng.device)
        self._keep = (list(shards), param)
        self._arr = ptr_array([x.data_ptr() for x in shards])
        h = C.c_void_p()
        check(lib().gq_graph_mean_inproc(
            self._arr, eng.dtype_code, eng.d, C.byref(eng.c_cfg), self.round.data_ptr(), eng._lane_arr,
            eng.result_lanes.data_ptr() if write_lanes else None, eng.mean.data_ptr() if write_mean else None,
            param.data_ptr() if param is not None else None, float(lr), eng.stats.data_ptr(), eng.norm.data_ptr(),
            eng.workspace.data_ptr(), eng.kbuf.data_ptr() if eng.kd is not None else None, eng.err.data_ptr(),
            C.byref(h)))
        self.handle = h

    def launch(self, stream: int | None = None) -> None:
        check(lib().gq_graph_launch(self.handle, _stream() if stream is None else stream))

    def __del__(self):
        try:
            if self.handle:
                lib().gq_graph_destroy(self.handle)
        except Exception:
            pass


# ---------------------------------------------------------------------------
# the sparse allgather path (cfg.sparse; quantizer.cpp:59-110, serialize.cpp:114-192,
# algorithm.cpp:112-123,187-200)
# ---------------------------------------------------------------------------
def sparse_lane_width(width_bits: int, s: int) -> int:
    """validate_level_width (serialize.cpp:114-122)."""
    if width_bits not in (8, 16, 32):
        raise InvalidArgument("level lane width must be 8, 16, or 32 bits")
    if width_bits < 32 and s > (1 << width_bits) - 1:
        raise InvalidArgument("level index does not fit the lane width")
    return width_bits


def _quantize32(x: torch.Tensor, dt: int, norm: torch.Tensor, kind: int, s: int, seed: int, worker: int,
                round: int, n_total: int, err: torch.Tensor) -> torch.Tensor:
    d = x.numel()
    lanes = torch.zeros(lane_bytes(d, 32), dtype=torch.uint8, device=x.device)
    ids = (C.c_uint32 * 1)(worker)
    check(lib().gq_quantize(ptr_array([x.data_ptr()]), dt, 1, ids, d, norm.data_ptr(), kind, s, n_total, 32,
                            seed, round, ptr_array([lanes.data_ptr()]), err.data_ptr(), _stream()))
    return lanes


def sparse_payload(x: torch.Tensor, norm, kind: LevelKind, s: int, seed: int, worker: int, round: int,
                   width_bits: int = 8) -> torch.Tensor:
    """serialize_sparse(to_sparse(quantize_shard(...))) on the device: the
    worker's sparse wire payload as a uint8 CUDA tensor (byte-identical to the
    reference's)."""
    d, dt = _check_shards([x])
    w = sparse_lane_width(width_bits, s)
    dev = x.device
    err = _ErrWord.get(dev)
    nt = _norm_tensor(norm, dev)
    lanes = _quantize32(x, dt, nt, int(kind), s, seed, worker, round, 1, err)
    payload = torch.zeros(int(lib().gq_sparse_payload_bytes(d, w)) + 16, dtype=torch.uint8, device=dev)
    ws = torch.zeros(int(lib().gq_sparse_workspace_bytes(d)), dtype=torch.uint8, device=dev)
    nnz = torch.zeros(1, dtype=torch.int32, device=dev)
    check(lib().gq_sparse_encode(lanes.data_ptr(), d, int(kind), s, 1, w, nt.data_ptr(), payload.data_ptr(),
                                 ws.data_ptr(), nnz.data_ptr(), _stream()))
    _sync_check(err)
    return payload[:int(lib().gq_sparse_payload_bytes(int(nnz.item()), w))]


def sparse_accumulate(payloads, d: int, kind: LevelKind, s: int, width_bits: int, n: int | None = None,
                      out_f64: bool = False) -> torch.Tensor:
    """accumulate_sparse over received payloads in rank order, then / n
    (decode_sparse_set, algorithm.cpp:112-123)."""
    dev = payloads[0].device
    err = _ErrWord.get(dev)
    acc = torch.zeros(d, dtype=torch.float64, device=dev)
    for p in payloads:
        check(lib().gq_sparse_accumulate(p.data_ptr(), p.numel(), int(kind), s, width_bits, d, acc.data_ptr(),
                                         err.data_ptr(), _stream()))
    out = torch.empty(d, dtype=torch.float64 if out_f64 else torch.float32, device=dev)
    check(lib().gq_sparse_finish(acc.data_ptr(), d, n or len(payloads), None if out_f64 else out.data_ptr(),
                                 out.data_ptr() if out_f64 else None, None, 0.0, _stream()))
    _sync_check(err)
    return out


def _gqsgd_mean_sparse(shards, cfg: GqsgdConfig, round: int) -> MeanResult:
    d, dt = _check_shards(shards)
    n = cfg.workers
    w = sparse_lane_width(cfg.width_bits, cfg.s)
    stats, norm = global_norm(shards, cfg.norm)
    dev = shards[0].device
    err = _ErrWord.get(dev)
    lanes = [_quantize32(x, dt, norm, int(cfg.scheme), cfg.s, cfg.seed, r, round, n, err)
             for r, x in enumerate(shards)]
    mean = torch.empty(d, dtype=torch.float32, device=dev)
    check(lib().gq_sparse_mean_inproc(ptr_array([l.data_ptr() for l in lanes]), n, d, int(cfg.scheme), cfg.s, n,
                                      norm.data_ptr(), mean.data_ptr(), None, _stream()))
    _sync_check(err)
    return MeanResult(mean, float(norm.item()), w, stats, None)


def gqsgd_mean(shards, cfg: GqsgdConfig, round: int, param: torch.Tensor | None = None,
               lr: float = 0.0) -> MeanResult:
    """gqsgd_mean (algorithm.cpp:127-228), Transport::Inproc semantics, on one
    device: shards[r] is worker r's gradient (CUDA tensor, fp32 or fp64)."""
    d, _ = _check_shards(shards)
    if len(shards) != cfg.workers:
        raise InvalidArgument("shard count does not match the worker count")
    if cfg.sparse:
        if param is not None:
            raise InvalidArgument("the fused SGD epilogue is on the dense paths")
        return _gqsgd_mean_sparse(shards, cfg, round)
    eng = InprocSync(cfg, d, shards[0].device, shards[0].dtype)
    eng.run(shards, round, param=param, lr=lr)
    eng.check()
    return MeanResult(eng.mean, float(eng.norm.item()), eng.plan.lane_width, eng.stats,
                      eng.result_lanes)


def baseline_mean(shards) -> torch.Tensor:
    """baseline_mean (algorithm.cpp:303-340) on one device, tree schedule."""
    d, dt = _check_shards(shards)
    if dt != _lib.GQ_DTYPE_F32:
        raise InvalidArgument("the fp32 baseline takes float32 shards")
    out = torch.empty(d, dtype=torch.float32, device=shards[0].device)
    check(lib().gq_baseline_mean_inproc(ptr_array([x.data_ptr() for x in shards]), len(shards), d,
                                        0, out.data_ptr(), _stream()))
    torch.cuda.current_stream().synchronize()
    return out
