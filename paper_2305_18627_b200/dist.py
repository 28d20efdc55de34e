"""Multi-GPU gradient sync: one process per GPU, each rank a set of workers.

This is `gqsgd_mean_worker` (algorithm.cpp:230-301) for ranks that each host
n/N of the n workers, with the TCP mesh (transport.cpp) replaced by
collectives over NVLink (torch.distributed / NCCL as plumbing) and every
per-element step in the sm_100a kernels of libgq_b200.so:

  1. norm      gq_norm on the local shards (stats only), all_gather of the
               n_local f64 stats, gq_norm_combine walks the reference tree over
               all n stats in worker order (collectives.cpp:210-233) -> every
               rank holds the identical global scale;
  2. quantize  gq_quantize of the local workers (keys use the GLOBAL worker id,
               quantizer.cpp:42) into their lane buffers;
  3. exchange  "p2p" (<= 16 GPUs, the default when ranks can map each
               other): no NCCL on the lane path - quantize stores each lane
               slice straight into its owner's receive row for that worker
               (CUDA-IPC peer pointers over NVLink), epoch
               flags (system-scope release/acquire) order the phases, and the
               slice reduce stores its result into every peer's summed buffer
               (the all_gather fused into the reduce epilogue);
               "sparse" (cfg.sparse): serialize_sparse of each local worker,
               all_gather of the payload sizes then of the (padded) payloads,
               accumulate_sparse in rank order (algorithm.cpp:187-200);
               "pull" (the NCCL route, any kind/width; "auto" picks it when the
               ranks cannot map each other's memory): the lanes are cut into N
               equal word-aligned slices; all_to_all_single sends slice j of
               each local worker to rank j; rank g replays the reference
               schedule on slice g over all n workers (gq_reduce_slice: k draws
               keyed by the global lane, collectives.cpp:132-146) and
               all_gather_into_tensor assembles the summed lanes everywhere.
               "nccl_sum" (standard, w in {8, 32}): rank-local partial integer
               sums (gq_reduce_lanes) then one all_reduce(int8|int32, sum);
               exact because integer sums are order-free and plan_path's
               admission rules out intermediate overflow (collectives.cpp:76-78);
  4. decode    gq_dequant of the summed lanes (+ the SGD update, trainer.cpp:335).

The per-element arithmetic never depends on N, so the N-rank result is
bit-identical to the single-device simulation (gqsgd_mean / InprocSync) and to
the reference. DESIGN.md §5.

The kernels and the collectives are reached through two small interfaces
(`DeviceKernels`, `TorchComm`) so the host logic above can be exercised on CPU
by the tests with gloo and an oracle-backed kernel set (tests/dist_fakes.py).
"""
from __future__ import annotations

import ctypes as C
import os

import torch
import torch.distributed as dist

from . import _lib
from ._lib import InvalidArgument, check, lib, ptr_array
from .gqsgd import GqsgdConfig, LevelKind, NormSpec, Plan, lane_bytes, plan_path, sparse_lane_width

SLICE_UNIT_LANES = 128  # slice boundaries: 16-byte aligned for every lane width, float4-aligned mean


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class _Done:
    """Work handle of a collective that already completed (synchronous comms)."""

    def wait(self) -> None:
        return None


DONE = _Done()


class TorchComm:
    """torch.distributed collectives (NCCL on GPUs, gloo in CPU tests). With
    async_op=True they return the Work handle: NCCL runs the collective on its
    own stream after the current stream's prior work, and work.wait() makes
    the current stream (not the host) wait for it, so the caller can queue
    compute for the next bucket in between."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_into_tensor(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        w = dist.all_gather_into_tensor(out, inp, group=self.group, async_op=async_op)
        return w if async_op else DONE

    def all_to_all_single(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        w = dist.all_to_all_single(out, inp, group=self.group, async_op=async_op)
        return w if async_op else DONE

    def all_reduce_sum(self, t: torch.Tensor, async_op: bool = False):
        w = dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=async_op)
        return w if async_op else DONE

    def all_gather_object(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self) -> None:
        dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# kernels (the product path: libgq_b200.so, no fallback)
# ---------------------------------------------------------------------------
class DeviceKernels:
    """The sm_100a kernels through the C ABI. Tensor arguments are CUDA
    tensors or views; every call is stream-ordered on `stream` and does not
    synchronise (except `check`)."""

    def __init__(self, device: torch.device, stream: torch.cuda.Stream | None = None):
        if device.type != "cuda":
            raise InvalidArgument("DeviceKernels needs a CUDA device; there is no CPU fallback")
        self.L = lib()
        self.device = device
        self.stream = stream or torch.cuda.current_stream(device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self._ws: torch.Tensor | None = None

    @property
    def sp(self) -> int:
        return self.stream.cuda_stream

    def _workspace(self, n: int, d: int) -> torch.Tensor:
        need = int(self.L.gq_norm_workspace_bytes(n, d))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def norm_stats(self, shards, spec: NormSpec, stats_out: torch.Tensor) -> None:
        n, d = len(shards), shards[0].numel()
        dt = _lib.GQ_DTYPE_F32 if shards[0].dtype == torch.float32 else _lib.GQ_DTYPE_F64
        check(self.L.gq_norm(ptr_array([x.data_ptr() for x in shards]), dt, n, d, spec.q, spec.p,
                             stats_out.data_ptr(), None, self._workspace(n, d).data_ptr(),
                             self.err.data_ptr(), self.sp))

    def norm_combine(self, stats_all: torch.Tensor, spec: NormSpec, norm_out: torch.Tensor) -> None:
        check(self.L.gq_norm_combine(stats_all.data_ptr(), stats_all.numel(), spec.q, spec.p,
                                     norm_out.data_ptr(), self.sp))

    def quantize(self, shards, worker_ids, norm: torch.Tensor, cfg: GqsgdConfig, width: int,
                 round: int, lanes_out) -> None:
        n_local, d = len(shards), shards[0].numel()
        dt = _lib.GQ_DTYPE_F32 if shards[0].dtype == torch.float32 else _lib.GQ_DTYPE_F64
        ids = (C.c_uint32 * n_local)(*worker_ids)
        check(self.L.gq_quantize(ptr_array([x.data_ptr() for x in shards]), dt, n_local, ids, d,
                                 norm.data_ptr(), int(cfg.scheme), cfg.s, cfg.workers, width,
                                 cfg.seed, round, ptr_array([t.data_ptr() for t in lanes_out]),
                                 self.err.data_ptr(), self.sp))

    def reduce_slice(self, slices, d: int, lane_begin: int, lane_end: int, cfg: GqsgdConfig,
                     width: int, round: int, out_slice: torch.Tensor) -> None:
        check(self.L.gq_reduce_slice(ptr_array([t.data_ptr() for t in slices]), len(slices), d,
                                     lane_begin, lane_end, int(cfg.scheme), width, cfg.s,
                                     int(cfg.topo), cfg.seed, round, None, out_slice.data_ptr(),
                                     None, None, 0.0, self.err.data_ptr(), self.sp))

    def reduce_local(self, lanes, d: int, cfg: GqsgdConfig, width: int, round: int,
                     out: torch.Tensor) -> None:
        """Integer partial sum of the local workers' lanes (standard only)."""
        check(self.L.gq_reduce_lanes(ptr_array([t.data_ptr() for t in lanes]), len(lanes), d, 0, d,
                                     int(cfg.scheme), width, cfg.s, 0, cfg.seed, round, None,
                                     out.data_ptr(), None, None, 0.0, self.err.data_ptr(), self.sp))

    def dequant(self, lanes: torch.Tensor, d: int, norm: torch.Tensor, cfg: GqsgdConfig, width: int,
                mean_out: torch.Tensor | None, param: torch.Tensor | None, lr: float) -> None:
        src = lanes if isinstance(lanes, int) else lanes.data_ptr()  # p2p: raw symmetric buffer
        check(self.L.gq_dequant(src, 0, d, norm.data_ptr(), int(cfg.scheme), cfg.s,
                                cfg.workers, width,
                                mean_out.data_ptr() if mean_out is not None else None,
                                param.data_ptr() if param is not None else None, float(lr),
                                self.err.data_ptr(), self.sp))

    # the sparse allgather path (cfg.sparse)
    def sparse_encode(self, lanes32: torch.Tensor, d: int, cfg: GqsgdConfig, width: int, norm: torch.Tensor,
                      payload: torch.Tensor, workspace: torch.Tensor, nnz_slot: torch.Tensor) -> None:
        check(self.L.gq_sparse_encode(lanes32.data_ptr(), d, int(cfg.scheme), cfg.s, cfg.workers, width,
                                      norm.data_ptr(), payload.data_ptr(), workspace.data_ptr(),
                                      nnz_slot.data_ptr(), self.sp))

    def sparse_accumulate(self, payload: torch.Tensor, nbytes: int, cfg: GqsgdConfig, width: int, d: int,
                          acc: torch.Tensor) -> None:
        check(self.L.gq_sparse_accumulate(payload.data_ptr(), nbytes, int(cfg.scheme), cfg.s, width, d,
                                          acc.data_ptr(), self.err.data_ptr(), self.sp))

    def dequant_f64(self, lanes, d: int, norm: torch.Tensor, cfg: GqsgdConfig, width: int,
                    out: torch.Tensor) -> None:
        """decode_dense_std / decode_dense_exp (algorithm.cpp:84-110) in f64."""
        src = lanes if isinstance(lanes, int) else lanes.data_ptr()
        check(self.L.gq_dequant_f64(src, 0, d, norm.data_ptr(), int(cfg.scheme), cfg.s, cfg.workers, width,
                                    out.data_ptr(), self.err.data_ptr(), self.sp))

    def sparse_finish(self, acc: torch.Tensor, d: int, n: int, mean_out, param, lr: float,
                      mean64_out=None) -> None:
        check(self.L.gq_sparse_finish(acc.data_ptr(), d, n, mean_out.data_ptr() if mean_out is not None else None,
                                      mean64_out.data_ptr() if mean64_out is not None else None,
                                      param.data_ptr() if param is not None else None, float(lr), self.sp))

    def sparse_workspace_bytes(self, d: int) -> int:
        return int(self.L.gq_sparse_workspace_bytes(d))

    def check(self) -> tuple[int, str]:
        rc = self.L.gq_check(self.err.data_ptr(), self.sp)
        return rc, (self.L.gq_last_error().decode() if rc else "")


# ---------------------------------------------------------------------------
class DistSync:
    """Preallocated multi-rank gradient sync (gqsgd_mean_worker semantics).

    `run(shards, round)` takes this rank's n_local shards (workers
    rank*n_local ... in order), leaves the decoded mean in `self.mean` (and
    applies the SGD step to `param` when given); no allocation, no host sync
    beyond what the collectives imply. `check()` raises the reference's
    exception class on every rank if any rank saw a device error.
    """

    def __init__(self, cfg: GqsgdConfig, d: int, comm=None, kernels=None, device=None,
                 exchange: str = "auto", dtype=torch.float32, share_p2p: "DistSync | None" = None):
        """share_p2p: another DistSync of the same d whose peer-memory
        communicator this one reuses (its steps must be stream-ordered with the
        owner's, as BucketedSync arranges); the owner keeps the buffers."""
        self.cfg = cfg
        self._p2p_owner = None
        self.comm = comm or TorchComm()
        self.world, self.rank = self.comm.world, self.comm.rank
        n = cfg.workers
        if n % self.world:
            raise InvalidArgument("worker count must be a multiple of the number of ranks")
        self.n_local = n // self.world
        self.worker_ids = list(range(self.rank * self.n_local, (self.rank + 1) * self.n_local))
        if cfg.sparse:  # the allgather path (algorithm.cpp:187-200, :272-282)
            exchange = "sparse"
            self.plan = None
            self.width = w = sparse_lane_width(cfg.width_bits, cfg.s)
        else:
            self.plan: Plan = plan_path(cfg)
            self.width = w = self.plan.lane_width
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        if exchange == "auto":  # peer memory between the GPUs of one node, else NCCL all_to_all
            exchange = "p2p" if (self.world <= 16 and self.device.type == "cuda") else "pull"
        if exchange not in ("pull", "nccl_sum", "sparse", "p2p"):
            raise InvalidArgument(f"unknown exchange {exchange!r}")
        if exchange == "nccl_sum" and not (cfg.scheme == LevelKind.Standard and w in (8, 32)):
            raise InvalidArgument("nccl_sum needs standard lanes of 8 or 32 bits "
                                  "(token reduce has no NCCL operator)")
        self.exchange = exchange
        self.d = d
        self.kernels = kernels or DeviceKernels(self.device)
        dev = self.device

        if exchange == "p2p" and self.world > 16:
            raise InvalidArgument("the peer-memory exchange maps at most 16 GPUs")
        self.lanes = []
        self.host_waits = False
        if exchange == "p2p":
            ok = True
            try:
                self._setup_geometry(exchange)
                if share_p2p is not None and getattr(share_p2p, "_comm", None) and share_p2p.d == d:
                    self._share_p2p(share_p2p)
                else:
                    self._setup_p2p()
            except _lib.GqError:
                ok = False
            # every rank must agree: if any rank could not map its peers
            # (no CUDA IPC / peer access), all fall back to the NCCL exchange
            if not all(self.comm.all_gather_object(ok)):
                self._release_p2p()
                exchange = self.exchange = "pull"
        if exchange != "p2p":
            self._setup_geometry(exchange)
        if exchange == "pull":
            N = self.world
            self.recv = [torch.zeros(N * self.slice_bytes, dtype=torch.uint8, device=dev)
                         for _ in range(self.n_local)]
            # worker w's slice g arrives from rank w // n_local in recv[w % n_local]
            self.slice_views = [self.recv[wk % self.n_local][(wk // self.n_local) * self.slice_bytes:
                                                             (wk // self.n_local + 1) * self.slice_bytes]
                                for wk in range(n)]
            g = self.rank
            self.my_slice = self.summed[g * self.slice_bytes:(g + 1) * self.slice_bytes]
            self.send = [t[:N * self.slice_bytes] for t in self.lanes]
        if exchange == "sparse":
            self.pay_cap = int(lib().gq_sparse_payload_bytes(d, w))
            self.payloads = torch.zeros(self.n_local, self.pay_cap, dtype=torch.uint8, device=dev)
            self.sws = torch.zeros(self.kernels.sparse_workspace_bytes(d), dtype=torch.uint8, device=dev)
            self.nnz_local = torch.zeros(self.n_local, dtype=torch.int32, device=dev)
            self.nnz_all = torch.zeros(n, dtype=torch.int32, device=dev)
            self.acc = torch.zeros(d, dtype=torch.float64, device=dev)
        self.stats_local = torch.zeros(self.n_local, dtype=torch.float64, device=dev)
        self.stats_all = torch.zeros(n, dtype=torch.float64, device=dev)
        self.norm = torch.zeros(1, dtype=torch.float64, device=dev)
        self.mean = torch.zeros(d, dtype=torch.float32, device=dev)

    def _setup_geometry(self, exchange: str) -> None:
        """Slice geometry (pull / p2p exchange): N equal slices of slice_lanes
        lanes; rank g owns lanes [g*slice_lanes, (g+1)*slice_lanes) of d."""
        N, d, w, dev = self.world, self.d, self.width, self.device
        unit = 1024 if exchange == "p2p" else SLICE_UNIT_LANES  # whole 4 KiB quantize chunks per slice
        self.slice_lanes = max(unit, -(-d // (N * unit)) * unit)
        self.slice_bytes = self.slice_lanes * w // 8
        self.buf_bytes = max(N * self.slice_bytes, lane_bytes(d, w))
        if exchange == "sparse":  # 32-bit lanes carry (sign, level index) into the encoder
            self.buf_bytes = lane_bytes(d, 32)
        # p2p: the lanes live in the communicator's symmetric buffers
        self.lanes = [torch.zeros(self.buf_bytes, dtype=torch.uint8, device=dev)
                      for _ in range(self.n_local if exchange != "p2p" else 0)]
        self.summed = torch.zeros(self.buf_bytes, dtype=torch.uint8, device=dev)
        g = self.rank
        self.lane_begin = min(d, g * self.slice_lanes)
        self.lane_end = min(d, (g + 1) * self.slice_lanes)

    # -- peer-memory exchange (exchange="p2p") -------------------------------
    def _setup_p2p(self) -> None:
        """A native communicator (gq_comm_*, csrc/gq_comm.cu) owns the
        symmetric buffers; this rank's bootstrap blob is all-gathered over the
        process group (like an NCCL unique id) and every rank maps its peers
        (CUDA IPC across processes, plain pointers between threads)."""
        L = lib()
        ptr = C.c_void_p()
        cfg = self.cfg.to_c()
        check(L.gq_comm_init(self.rank, self.world, C.byref(cfg), self.d, C.byref(ptr)))
        self._comm = ptr.value
        hb = int(L.gq_comm_handle_bytes())
        h = (C.c_char * hb)()
        check(L.gq_comm_handle(self._comm, h))
        blobs = self.comm.all_gather_object(bytes(h))
        allh = (C.c_char * (hb * self.world)).from_buffer_copy(b"".join(blobs))
        check(L.gq_comm_connect(self._comm, allh))
        info = _lib.GqCommInfo()
        check(L.gq_comm_info_get(self._comm, C.byref(info)))
        if info.slice_lanes != self.slice_lanes or info.lane_width != self.width:
            raise _lib.RuntimeFailure("communicator geometry disagrees with the host plan")
        if self.device.index is not None and info.device != self.device.index:
            raise _lib.RuntimeFailure(f"communicator buffers landed on cuda:{info.device}, not {self.device} "
                                      "(set the current device before creating DistSync)")
        self.p_summed = int(L.gq_comm_summed(self._comm))
        self.host_waits = bool(info.host_wait)  # a peer shares this GPU: no graph capture
        self.p2p_bytes = self.world * self.slice_bytes

    def _share_p2p(self, owner: "DistSync") -> None:
        """Reuse `owner`'s communicator: same symmetric buffers and flags, so
        the two syncs' steps must not overlap (one stream, or the flag chain
        of consecutive steps orders them: a rank reuses a buffer only after
        every peer signalled it consumed the previous step's contents)."""
        self._p2p_owner = owner
        self._comm = owner._comm
        self.p_summed = owner.p_summed
        self.host_waits = owner.host_waits
        self.p2p_bytes = owner.p2p_bytes

    def _p2p_quantize(self, shards, round: int) -> None:
        k = self.kernels
        dt = _lib.GQ_DTYPE_F32 if shards[0].dtype == torch.float32 else _lib.GQ_DTYPE_F64
        check(lib().gq_comm_quantize(self._comm, ptr_array([x.data_ptr() for x in shards]), dt,
                                     self.norm.data_ptr(), round, k.err.data_ptr(), k.sp))

    def _p2p_exchange(self, round: int) -> None:
        k = self.kernels
        check(lib().gq_allreduce_lanes(self._comm, None, round, None, k.err.data_ptr(), k.sp))

    def make_graph(self, shards, first_round: int, param: torch.Tensor | None = None, lr: float = 0.0,
                   write_mean: bool = True, round_step: int = 1) -> "CommGraph":
        """The whole p2p step on fixed buffers as one CUDA graph
        (gq_comm_graph): each launch() is run(shards, round) with the round
        kept on the device and advanced by round_step per launch."""
        if self.exchange != "p2p":
            raise InvalidArgument("graph capture covers the peer-memory exchange")
        return CommGraph(self, shards, first_round, param, lr, write_mean, round_step)

    def _release_p2p(self) -> None:
        if getattr(self, "_comm", None) and getattr(self, "_p2p_owner", None) is None:
            lib().gq_comm_destroy(self._comm)
        self._comm = None

    def __del__(self):
        try:
            self._release_p2p()
        except Exception:
            pass

    # -- phases ------------------------------------------------------------
    # Each exchange step is split into "issue" and "finish" halves so a
    # bucket pipeline (BucketedSync) can queue other buckets' compute while a
    # collective is in flight; run() calls them back to back.
    def _coll(self, fn, *a, async_op: bool = False):
        w = fn(*a, async_op=async_op) if async_op else fn(*a)
        return w if w is not None else DONE

    def norm_issue(self, shards, async_op: bool = False, round: int = 0):
        if self.exchange == "p2p":  # stats stored into every peer, tree fold on each rank; the same
            k = self.kernels        # pass precomputes this round's k draws of the rank's slice
            dt = _lib.GQ_DTYPE_F32 if shards[0].dtype == torch.float32 else _lib.GQ_DTYPE_F64
            check(lib().gq_comm_norm(self._comm, ptr_array([x.data_ptr() for x in shards]), dt, round,
                                     self.norm.data_ptr(), k.err.data_ptr(), k.sp))
            return DONE
        self.kernels.norm_stats(shards, self.cfg.norm, self.stats_local)
        return self._coll(self.comm.all_gather_into_tensor, self.stats_all, self.stats_local, async_op=async_op)

    def norm_finish(self, work) -> None:
        work.wait()
        if self.exchange != "p2p":
            self.kernels.norm_combine(self.stats_all, self.cfg.norm, self.norm)

    def norm_phase(self, shards, round: int = 0) -> None:
        self.norm_finish(self.norm_issue(shards, round=round))

    def quantize_phase(self, shards, round: int) -> None:
        if self.exchange == "p2p":
            self._p2p_quantize(shards, round)
            return
        self.kernels.quantize(shards, self.worker_ids, self.norm, self.cfg,
                              32 if self.exchange == "sparse" else self.width, round, self.lanes)

    def _sparse_exchange(self) -> None:
        """serialize_sparse per local worker, all_gather of the payloads (padded
        to the largest; sizes exchanged first), rank-ordered accumulate_sparse."""
        k, cfg, d, w = self.kernels, self.cfg, self.d, self.width
        for i in range(self.n_local):
            k.sparse_encode(self.lanes[i], d, cfg, w, self.norm, self.payloads[i], self.sws,
                            self.nnz_local[i:i + 1])
        self.comm.all_gather_into_tensor(self.nnz_all, self.nnz_local)
        sizes = [16 + 4 * c + (c + 7) // 8 + c * (w // 8) for c in self.nnz_all.cpu().tolist()]
        cap = max(sizes)
        send = self.payloads[:, :cap].contiguous()
        recv = torch.empty(self.world * self.n_local, cap, dtype=torch.uint8, device=self.device)
        self.comm.all_gather_into_tensor(recv.view(-1), send.view(-1))
        self.acc.zero_()
        for wk in range(cfg.workers):  # rank order: worker wk is row wk
            k.sparse_accumulate(recv[wk], sizes[wk], cfg, w, d, self.acc)

    def exchange_issue(self, round: int, async_op: bool = False):
        k, cfg, d, w = self.kernels, self.cfg, self.d, self.width
        if self.exchange == "sparse":
            self._sparse_exchange()
            return [DONE]
        if self.exchange == "p2p":
            self._p2p_exchange(round)
            return [DONE]
        if self.exchange == "pull":
            return [self._coll(self.comm.all_to_all_single, self.recv[i], self.send[i], async_op=async_op)
                    for i in range(self.n_local)]
        if self.n_local == 1:
            self.summed.copy_(self.lanes[0])
        else:
            k.reduce_local(self.lanes, d, cfg, w, round, self.summed)
        view = self.summed.view(torch.int8) if w == 8 else self.summed.view(torch.int32)
        return [self._coll(self.comm.all_reduce_sum, view, async_op=async_op)]

    def exchange_mid(self, works, round: int, async_op: bool = False):
        for wk in works:
            wk.wait()
        if self.exchange != "pull":
            return DONE
        if self.lane_end > self.lane_begin:
            self.kernels.reduce_slice(self.slice_views, self.d, self.lane_begin, self.lane_end, self.cfg,
                                      self.width, round, self.my_slice)
        return self._coll(self.comm.all_gather_into_tensor, self.summed[:self.world * self.slice_bytes],
                          self.my_slice, async_op=async_op)

    def exchange_phase(self, round: int) -> None:
        self.exchange_mid(self.exchange_issue(round), round).wait()

    def decode_phase(self, param=None, lr: float = 0.0, write_mean: bool = True) -> None:
        if param is None and not write_mean:
            return
        if self.exchange == "sparse":
            self.kernels.sparse_finish(self.acc, self.d, self.cfg.workers, self.mean if write_mean else None,
                                       param, lr)
            return
        src = self.p_summed if self.exchange == "p2p" else self.summed
        self.kernels.dequant(src, self.d, self.norm, self.cfg, self.width,
                             self.mean if write_mean else None, param, lr)

    def decode_f64(self, out: torch.Tensor) -> None:
        """This step's mean as the reference's doubles (f64 gradients: the
        decoders of algorithm.cpp:84-110 are f64), written into `out`."""
        if out.dtype != torch.float64 or out.numel() != self.d:
            raise InvalidArgument("decode_f64 writes a float64 tensor of d elements")
        if self.exchange == "sparse":
            self.kernels.sparse_finish(self.acc, self.d, self.cfg.workers, None, None, 0.0, mean64_out=out)
            return
        src = self.p_summed if self.exchange == "p2p" else self.summed
        self.kernels.dequant_f64(src, self.d, self.norm, self.cfg, self.width, out)

    def run(self, shards, round: int, param: torch.Tensor | None = None, lr: float = 0.0,
            write_mean: bool = True, marks=None) -> None:
        """marks: optional list of 5 CUDA events recorded on the kernel stream
        at the phase boundaries (norm | quantize | exchange | decode)."""
        if len(shards) != self.n_local:
            raise InvalidArgument("shard count does not match the workers of this rank")
        mark = (lambda i: marks[i].record(self.kernels.stream)) if marks else (lambda i: None)
        mark(0)
        self.norm_phase(shards, round)
        mark(1)
        self.quantize_phase(shards, round)
        mark(2)
        self.exchange_phase(round)
        mark(3)
        self.decode_phase(param, lr, write_mean)
        mark(4)

    def check(self) -> None:
        if self.exchange == "p2p":  # every rank's error word over peer memory, same status everywhere
            check(lib().gq_sync(self._comm, self.kernels.err.data_ptr(), self.kernels.sp))
            return
        rc, msg = self.kernels.check()
        results = self.comm.all_gather_object((rc, msg))
        for r, (code, m) in enumerate(results):
            if code:
                raise _lib._EXC.get(code, _lib.RuntimeFailure)(f"rank {r}: {m}")

    @property
    def summed_payload(self) -> torch.Tensor:
        if self.exchange == "p2p":  # the summed lanes live in the symmetric buffer
            L, k = lib(), self.kernels
            check(L.gq_memcpy(self.summed.data_ptr(), self.p_summed, self.p2p_bytes, k.sp))
            check(L.gq_stream_sync(k.sp))
        return self.summed[:(self.d * self.width + 7) // 8]


class CommGraph:
    """A captured DistSync step (see DistSync.make_graph)."""

    def __init__(self, sync: DistSync, shards, first_round: int, param, lr: float, write_mean: bool,
                 round_step: int = 1):
        self.sync = sync
        self.handle = None
        self.round = torch.tensor([first_round], dtype=torch.int64, device=sync.device)
        self._keep = (list(shards), param)
        dt = _lib.GQ_DTYPE_F32 if shards[0].dtype == torch.float32 else _lib.GQ_DTYPE_F64
        h = C.c_void_p()
        check(lib().gq_comm_graph(sync._comm, ptr_array([x.data_ptr() for x in shards]), dt,
                                  sync.mean.data_ptr() if write_mean else None, None,
                                  param.data_ptr() if param is not None else None, float(lr),
                                  self.round.data_ptr(), round_step, sync.kernels.err.data_ptr(), C.byref(h)))
        self.handle = h

    def launch(self, stream: int | None = None) -> None:
        check(lib().gq_graph_launch(self.handle, self.sync.kernels.sp if stream is None else stream))

    def __del__(self):
        try:
            if self.handle:
                lib().gq_graph_destroy(self.handle)
        except Exception:
            pass


class BucketedSync:
    """Several buckets (each its own reference call / round) synchronised as
    one software pipeline: every phase is issued for all buckets before the
    next phase, with the collectives asynchronous, so the NCCL transfer of
    bucket b (stats all_gather, lane all_to_all, summed-lane all_gather) runs
    under the kernels of bucket b+1 on the compute stream. This is how a DDP
    step with many gradient buckets overlaps communication with compute.
    Results are the per-bucket DistSync results (bit-identical to run())."""

    # peer-memory communicators per bucket size (bucket b uses lane b % COMM_LANES)
    COMM_LANES = int(os.environ.get("GQ_COMM_LANES", "3"))

    def __init__(self, cfg: GqsgdConfig, sizes, comm=None, kernels=None, device=None,
                 exchange: str = "auto"):
        self.comm = comm or TorchComm()
        # p2p: the buckets share COMM_LANES communicators per distinct size
        # (C4: 2 for the 6,553,600-element buckets + 1 for the tail) instead of
        # one symmetric allocation + IPC maps per bucket; bucket b uses the
        # communicator of lane b % COMM_LANES, whose steps stay ordered (one
        # stream per lane in graph replays, bucket order in run()).
        self.syncs, owners = [], {}
        for b, db in enumerate(sizes):
            key = (db, b % self.COMM_LANES)
            s = DistSync(cfg, db, comm=self.comm, kernels=kernels, device=device, exchange=exchange,
                         share_p2p=owners.get(key))
            if s.exchange == "p2p" and s._p2p_owner is None:
                owners[key] = s
            self.syncs.append(s)
        self.kernels = self.syncs[0].kernels if self.syncs else kernels
        self.async_ok = isinstance(self.comm, TorchComm)
        self.communicators = len(owners)

    def run(self, bucket_shards, rounds, params=None, lr: float = 0.0, write_mean: bool = True,
            marks=None) -> None:
        """bucket_shards[b]: this rank's shards of bucket b; rounds[b]: its
        round; params[b]: optional SGD parameter view. marks: 5 boundary events
        around the phases of bucket 0 (as DistSync.run)."""
        a = self.async_ok
        S = self.syncs
        nb = len(S)
        mark = (lambda i: marks[i].record(self.kernels.stream)) if marks else (lambda i: None)
        if nb and S[0].exchange == "p2p":
            # every p2p step is device work on one stream: bucket after bucket
            # (shared communicators need exactly that order)
            for b in range(nb):
                S[b].run(bucket_shards[b], rounds[b], param=params[b] if params is not None else None, lr=lr,
                         write_mean=write_mean, marks=marks if b == 0 else None)
            return
        mark(0)
        wn = [S[b].norm_issue(bucket_shards[b], async_op=a, round=rounds[b]) for b in range(nb)]
        wx = []
        for b in range(nb):
            S[b].norm_finish(wn[b])
            if b == 0:
                mark(1)
            S[b].quantize_phase(bucket_shards[b], rounds[b])
            if b == 0:
                mark(2)
            wx.append(S[b].exchange_issue(rounds[b], async_op=a))
        wg = [S[b].exchange_mid(wx[b], rounds[b], async_op=a) for b in range(nb)]
        for b in range(nb):
            wg[b].wait()
            if b == 0:
                mark(3)
            S[b].decode_phase(params[b] if params is not None else None, lr, write_mean)
            if b == 0:
                mark(4)

    def check(self) -> None:
        for s in self.syncs:
            s.check()


def gqsgd_mean_dist(shards, cfg: GqsgdConfig, round: int, param=None, lr: float = 0.0,
                    exchange: str = "auto", comm=None) -> torch.Tensor:
    """One synchronous call: this rank's shards -> the decoded mean every rank
    holds (gqsgd_mean_worker, algorithm.cpp:230-301). Allocates per call; the
    benchmark and training loops keep a DistSync instead."""
    d = shards[0].numel()
    eng = DistSync(cfg, d, comm=comm, device=shards[0].device, exchange=exchange,
                   dtype=shards[0].dtype)
    eng.run(shards, round, param=param, lr=lr)
    eng.check()
    return eng.mean
