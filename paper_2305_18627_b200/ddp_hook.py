"""PyTorch DDP communication hook running the Global-QSGD sync.

    model = DDP(model, device_ids=[rank])
    state = GqsgdHookState(GqsgdConfig(scheme=LevelKind.Standard, s=15, width_bits=8, seed=42))
    model.register_comm_hook(state, gqsgd_hook)

Each DDP gradient bucket of each step is one reference call (gqsgd_mean_worker,
algorithm.cpp:230-301, with this rank as worker `rank` of `world`): global
norm -> quantize -> lane exchange -> decode, all through dist.DistSync and the
sm_100a kernels. Bucket b of step t uses round = t * ROUND_STRIDE + b so every
bucket has its own dither / k-draw keys and any (step, bucket) replays exactly
(SURVEY §7 hard part 7). The hook writes the decoded mean into the bucket (DDP
expects the averaged gradient) and returns a completed CUDA-aware future.
With `overlap=True` (default on GPUs) the sync of a bucket runs on a
dedicated stream that first waits for the bucket's gradients, so it overlaps
the backward kernels of the layers still being differentiated; DDP's wait on
the future orders the optimizer after it. The host never waits.
Device errors (NaN/Inf gradients, overflow) are raised every `check_every`
steps, or on demand with state.check().
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from ._lib import InvalidArgument
from .dist import DeviceKernels, DistSync, TorchComm
from .gqsgd import GqsgdConfig

ROUND_STRIDE = 1 << 16  # rounds reserved per step (> any bucket count)


class GqsgdHookState:
    def __init__(self, cfg: GqsgdConfig, process_group=None, exchange: str = "auto",
                 check_every: int = 0, kernels_factory=None, overlap: bool = True):
        self.cfg = cfg
        self.overlap = overlap
        self.streams: dict = {}
        self.pg = process_group
        self.exchange = exchange
        self.check_every = check_every
        self.kernels_factory = kernels_factory  # tests: CPU oracle kernels; default: the device
        self.step = 0
        self.syncs: dict = {}
        self.comm = None

    def _sync_for(self, bucket_index: int, buf: torch.Tensor) -> DistSync:
        key = (bucket_index, buf.numel(), buf.device)
        s = self.syncs.get(key)
        if s is None:
            if self.comm is None:
                self.comm = TorchComm(self.pg)
            cfg = GqsgdConfig(**{**self.cfg.__dict__, "workers": self.comm.world})
            kernels = self.kernels_factory(buf.device) if self.kernels_factory else None
            side = self.side_stream(buf.device)
            if kernels is None and side is not None:
                kernels = DeviceKernels(buf.device, side)
            s = DistSync(cfg, buf.numel(), comm=self.comm, kernels=kernels, device=buf.device,
                         exchange=self.exchange)
            self.syncs[key] = s
        return s

    def side_stream(self, device):
        """The stream bucket syncs run on (None: the current stream)."""
        if not (self.overlap and device.type == "cuda" and self.kernels_factory is None):
            return None
        st = self.streams.get(device)
        if st is None:
            st = self.streams[device] = torch.cuda.Stream(device)
        return st

    def check(self) -> None:
        for s in self.syncs.values():
            s.check()


def gqsgd_hook(state: GqsgdHookState, bucket: dist.GradBucket) -> torch.futures.Future:
    buf = bucket.buffer()
    if buf.dtype not in (torch.float32, torch.float64):
        raise InvalidArgument("the gqsgd hook takes fp32 / fp64 gradient buckets")
    idx = bucket.index()
    if idx >= ROUND_STRIDE:
        raise InvalidArgument("more DDP buckets than ROUND_STRIDE")
    sync = state._sync_for(idx, buf)
    side = state.side_stream(buf.device)
    rnd = state.step * ROUND_STRIDE + idx
    def sync_into_buffer():
        if buf.dtype == torch.float64:  # the reference's f64 decode, straight into the bucket
            sync.run([buf], rnd, write_mean=False)
            sync.decode_f64(buf)
        else:
            sync.run([buf], rnd)
            buf.copy_(sync.mean)

    if side is None:
        sync_into_buffer()
        fut: torch.futures.Future = torch.futures.Future()
        fut.set_result(buf)
    else:
        side.wait_stream(torch.cuda.current_stream(buf.device))  # the bucket's gradients are ready
        with torch.cuda.stream(side):
            sync_into_buffer()
            fut = torch.futures.Future(devices=[buf.device])
            fut.set_result(buf)  # records the completion event on the side stream
    if bucket.is_last():
        state.step += 1
        if state.check_every and state.step % state.check_every == 0:
            state.check()
    return fut
