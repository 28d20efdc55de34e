"""TEST INFRASTRUCTURE — CPU stand-ins for the multi-rank host logic tests.

`OracleKernels` implements DistSync's kernel interface with the C oracle
(oracle/gq_oracle.c) on CPU tensors, so the host-side logic of
paper_2305_18627_b200/dist.py (worker placement, slice geometry, the
all_to_all / all_gather layout, stats exchange, round keys) runs under gloo
with world_size > 1 in this container. It is never used on the product path
(DistSync defaults to DeviceKernels, which has no CPU fallback).

`ThreadComm` runs N virtual ranks as threads of one process (one GPU in the
-m gpu tests), implementing the same collectives by copies.
"""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import torch


class OracleKernels:
    def __init__(self, oracle):
        self.o = oracle

    def norm_stats(self, shards, spec, stats_out):
        for i, x in enumerate(shards):
            stats_out[i] = self.o.local_norm_stat(x.double().numpy(), spec.q, spec.p)

    def norm_combine(self, stats_all, spec, norm_out):
        norm_out[0] = self.o.norm_tree_combine(stats_all.numpy(), spec.q, spec.p)

    def quantize(self, shards, worker_ids, norm, cfg, width, round, lanes_out):
        nv = float(norm[0])
        for x, wk, out in zip(shards, worker_ids, lanes_out):
            sign, idx = self.o.quantize(x.double().numpy(), nv, int(cfg.scheme), cfg.s, cfg.seed, wk,
                                        round)
            enc = self.o.encode(int(cfg.scheme), cfg.s, cfg.workers, width, sign, idx)
            out.zero_()
            out[:enc.size] = torch.from_numpy(enc)

    def reduce_slice(self, slices, d, lane_begin, lane_end, cfg, width, round, out_slice):
        n = len(slices)
        nb = (d * width + 7) // 8
        full = np.zeros((n, nb + 16), dtype=np.uint8)
        b0 = lane_begin * width // 8
        b1 = (lane_end * width + 7) // 8
        for r, sl in enumerate(slices):
            full[r, b0:b1] = sl[:b1 - b0].numpy()
        res = self.o.allreduce_inproc(full[:, :nb], d, int(cfg.scheme), width, cfg.s, int(cfg.topo),
                                      cfg.seed, round)
        out_slice.zero_()
        out_slice[:b1 - b0] = torch.from_numpy(res[0, b0:b1].copy())

    def reduce_local(self, lanes, d, cfg, width, round, out):
        nb = (d * width + 7) // 8
        full = np.stack([t[:nb].numpy() for t in lanes])
        res = self.o.allreduce_inproc(full, d, int(cfg.scheme), width, cfg.s, 0, cfg.seed, round)
        out.zero_()
        out[:nb] = torch.from_numpy(res[0].copy())

    def dequant(self, lanes, d, norm, cfg, width, mean_out, param, lr):
        nb = (d * width + 7) // 8
        m = self.o.decode(int(cfg.scheme), lanes[:nb].numpy(), d, float(norm[0]), cfg.s, cfg.workers,
                          width).astype(np.float32)
        if mean_out is not None:
            mean_out.copy_(torch.from_numpy(m))
        if param is not None:
            p = param.numpy()
            p[:] = p - np.float32(lr) * m

    # sparse allgather path (numpy restatement of serialize_sparse /
    # accumulate_sparse on the oracle's quantized levels)
    def sparse_workspace_bytes(self, d):
        return 1

    def _level(self, kind, i, s):
        return (s - i) / s if kind == 0 else 2.0 ** -i

    def sparse_encode(self, lanes32, d, cfg, width, norm, payload, ws, nnz_slot):
        lanes = lanes32[:4 * d].numpy().view(np.int32) if d else np.zeros(0, np.int32)
        kind, s = int(cfg.scheme), cfg.s
        shift = (2 * cfg.workers - 1).bit_length()
        if kind == 0:
            nzm = lanes != 0
            idx = s - np.abs(lanes)
        else:
            e = lanes.view(np.uint32) & 0x7FFFFFFF
            nzm = e != 0
            idx = e.astype(np.int64) - shift
        neg = (lanes.view(np.uint32) >> 31).astype(bool)
        j = np.flatnonzero(nzm).astype(np.uint32)
        nnz = j.size
        bits = np.zeros((nnz + 7) // 8, dtype=np.uint8)
        for k in np.flatnonzero(neg[nzm]):
            bits[k // 8] |= np.uint8(1 << (k % 8))
        lv = idx[nzm].astype(np.uint32).view(np.uint8).reshape(-1, 4)[:, :width // 8].reshape(-1)
        body = b"".join([np.float64(float(norm[0])).tobytes(), np.uint32(d).tobytes(), np.uint32(nnz).tobytes(),
                         j.tobytes(), bits.tobytes(), lv.tobytes()])
        payload.zero_()
        payload[:len(body)] = torch.frombuffer(bytearray(body), dtype=torch.uint8)
        nnz_slot[0] = nnz

    def sparse_accumulate(self, payload, nbytes, cfg, width, d, acc):
        b = payload[:nbytes].numpy().tobytes()
        norm = np.frombuffer(b[:8], np.float64)[0]
        nnz = int(np.frombuffer(b[12:16], np.uint32)[0])
        j = np.frombuffer(b[16:16 + 4 * nnz], np.uint32)
        bm = np.frombuffer(b[16 + 4 * nnz:16 + 4 * nnz + (nnz + 7) // 8], np.uint8)
        off = 16 + 4 * nnz + (nnz + 7) // 8
        lb = width // 8
        raw = np.frombuffer(b[off:off + nnz * lb], np.uint8).reshape(nnz, lb)
        li = np.zeros(nnz, np.uint32)
        for t in range(lb):
            li |= raw[:, t].astype(np.uint32) << (8 * t)
        a = acc.numpy()
        for k in range(nnz):
            sg = -norm if (bm[k // 8] >> (k % 8)) & 1 else norm
            a[j[k]] = a[j[k]] + sg * self._level(int(cfg.scheme), int(li[k]), cfg.s)

    def sparse_finish(self, acc, d, n, mean_out, param, lr):
        m = (acc.numpy() / n).astype(np.float32)
        if mean_out is not None:
            mean_out.copy_(torch.from_numpy(m))
        if param is not None:
            p = param.numpy()
            p[:] = p - np.float32(lr) * m

    def check(self):
        return 0, ""


class ThreadComm:
    """N virtual ranks as threads sharing one process; collectives by copies.
    For CUDA tensors every deposit is preceded by a device synchronize."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.sh = shared
        self.rank = rank
        self.world = shared.world

    @classmethod
    def group(cls, world):
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def _sync(self, t):
        if isinstance(t, torch.Tensor) and t.is_cuda:
            torch.cuda.synchronize(t.device)

    def _exchange(self, obj):
        self._sync(obj)
        self.sh.slots[self.rank] = obj
        self.sh.barrier.wait()
        got = list(self.sh.slots)
        return got

    def _done(self):
        self.sh.barrier.wait()

    def all_gather_into_tensor(self, out, inp):
        got = self._exchange(inp)
        k = inp.numel()
        for r, t in enumerate(got):
            out[r * k:(r + 1) * k].copy_(t)
        self._sync(out)
        self._done()

    def all_to_all_single(self, out, inp):
        got = self._exchange(inp)
        k = inp.numel() // self.world
        for r, t in enumerate(got):
            out[r * k:(r + 1) * k].copy_(t[self.rank * k:(self.rank + 1) * k])
        self._sync(out)
        self._done()

    def all_reduce_sum(self, t):
        got = self._exchange(t.clone())
        acc = got[0].clone()
        for g in got[1:]:
            acc += g
        t.copy_(acc)
        self._sync(t)
        self._done()

    def all_gather_object(self, obj):
        got = self._exchange(obj)
        self._done()
        return got

    def barrier(self):
        self.sh.barrier.wait()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def gloo_worker(rank, world, port, cases, q):
    """Spawned per rank: run every case through DistSync over gloo with the
    oracle-backed kernels; put (rank, results) on q."""
    import torch.distributed as dist

    from oracle.bind import Oracle
    from paper_2305_18627_b200.dist import DistSync, TorchComm
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind, NormSpec, TopologyKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        out = []
        for c in cases:
            x = o.gaussian_shards(c["n"], c["d"], c["data_seed"]).astype(np.float32)
            cfg = GqsgdConfig(workers=c["n"], scheme=LevelKind(c["kind"]), s=c["s"],
                              width_bits=c["width"], topo=TopologyKind(c["topo"]), seed=c["seed"],
                              norm=NormSpec(c.get("q", 0xFFFFFFFF), c.get("p", 0xFFFFFFFF)),
                              sparse=c.get("sparse", False))
            eng = DistSync(cfg, c["d"], comm=TorchComm(), kernels=OracleKernels(o),
                           device="cpu", exchange=c.get("exchange", "pull"))
            mine = [torch.from_numpy(x[w].copy()) for w in eng.worker_ids]
            param = torch.ones(c["d"], dtype=torch.float32) if c.get("sgd") else None
            eng.run(mine, c["round"], param=param, lr=0.5)
            eng.check()
            out.append(dict(mean=eng.mean.numpy().copy(), norm=float(eng.norm[0]),
                            summed=None if cfg.sparse else eng.summed_payload.numpy().copy(),
                            param=None if param is None else param.numpy().copy(),
                            width=eng.width))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def ddp_gloo_worker(rank, world, port, q):
    """Spawned per rank: a tiny model under DDP (gloo, CPU) with gqsgd_hook
    and the oracle kernels, 2 steps. Each hook call's input bucket, round and
    output are recorded so the test can check every bucket exactly against
    the oracle's gqsgd_mean over all ranks' inputs."""
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from oracle.bind import Oracle
    from paper_2305_18627_b200.ddp_hook import ROUND_STRIDE, GqsgdHookState, gqsgd_hook
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(), torch.nn.Linear(32, 4))
        ddp = DDP(model, bucket_cap_mb=0.001)  # several buckets
        state = GqsgdHookState(GqsgdConfig(scheme=LevelKind.Exponential, s=7, width_bits=8, seed=5),
                               kernels_factory=lambda dev: OracleKernels(o))
        records = []

        def recording_hook(st, bucket):
            inp = bucket.buffer().detach().clone().numpy()
            rnd = st.step * ROUND_STRIDE + bucket.index()
            fut = gqsgd_hook(st, bucket)
            records.append((bucket.index(), rnd, inp, fut.value().detach().clone().numpy()))
            return fut

        ddp.register_comm_hook(state, recording_hook)
        for step in range(2):
            g = torch.Generator().manual_seed(100 + rank + 10 * step)
            x = torch.randn(8, 16, generator=g)
            ddp.zero_grad()
            ddp(x).pow(2).mean().backward()
        q.put((rank, records, state.step))
    finally:
        dist.destroy_process_group()


def bucketed_gloo_worker(rank, world, port, q):
    """Spawned per rank: dist.BucketedSync over gloo (async collectives) with
    the oracle kernels; three buckets of different sizes, own rounds."""
    import torch.distributed as dist

    from oracle.bind import Oracle
    from paper_2305_18627_b200.dist import BucketedSync, TorchComm
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        sizes = [700, 333, 1024]
        n = 4
        cfg = GqsgdConfig(workers=n, scheme=LevelKind.Exponential, s=7, width_bits=8, seed=21)
        pipe = BucketedSync(cfg, sizes, comm=TorchComm(), kernels=OracleKernels(o), device="cpu")
        data = [o.gaussian_shards(n, sz, 50 + b).astype(np.float32) for b, sz in enumerate(sizes)]
        mine = [[torch.from_numpy(data[b][w].copy()) for w in pipe.syncs[b].worker_ids]
                for b in range(len(sizes))]
        pipe.run(mine, [10, 11, 12])
        pipe.check()
        q.put((rank, [s.mean.numpy().copy() for s in pipe.syncs]))
    finally:
        dist.destroy_process_group()


class StoreComm:
    """Ranks as separate processes on ONE GPU, collectives through a
    torch.distributed TCPStore (host copies). The native communicator maps
    the peers' buffers with CUDA IPC exactly as across GPUs (and, since the
    ranks share one device, waits on the host unless GQ_OPT_COMM_WAIT = 1)."""

    def __init__(self, rank, world, port):
        import torch.distributed as dist
        self.rank, self.world = rank, world
        self.store = dist.TCPStore("127.0.0.1", port, world, rank == 0, timeout=__import__("datetime").timedelta(seconds=120))
        self.seq = 0

    def _xchg(self, payload: bytes):
        import pickle
        self.seq += 1
        self.store.set(f"{self.seq}/{self.rank}", payload)
        out = [self.store.get(f"{self.seq}/{r}") for r in range(self.world)]
        self.barrier()
        return out

    def all_gather_object(self, obj):
        import pickle
        return [pickle.loads(b) for b in self._xchg(pickle.dumps(obj))]

    def all_gather_into_tensor(self, out, inp):
        got = self.all_gather_object(inp.detach().cpu())
        k = inp.numel()
        for r, t in enumerate(got):
            out[r * k:(r + 1) * k].copy_(t.to(out.device))

    def barrier(self):
        self.seq += 1
        self.store.add(f"b{self.seq}", 1)
        while int(self.store.add(f"b{self.seq}", 0)) < self.world:
            pass


def ipc_worker(rank, world, port, case, q):
    """Spawned per rank (all on cuda:0): DistSync(exchange='p2p') with CUDA-IPC
    peer mappings between processes."""
    import torch as T

    from oracle.bind import Oracle
    from paper_2305_18627_b200.dist import DistSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind
    try:
        T.cuda.set_device(0)
        from paper_2305_18627_b200 import _lib
        _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_COMM_WAIT, case.get("wait", 0)))
        o = Oracle()
        n, d = world * case.get("per", 1), case["d"]
        x = o.gaussian_shards(n, d, case["data_seed"]).astype(np.float32)
        comm = StoreComm(rank, world, port)
        cfg = GqsgdConfig(workers=n, scheme=LevelKind(case["kind"]), s=case["s"], width_bits=case["width"],
                          seed=case["seed"])
        eng = DistSync(cfg, d, comm=comm, device=T.device("cuda", 0), exchange="p2p")
        mine = [T.from_numpy(x[w].copy()).cuda() for w in eng.worker_ids]
        if case.get("graph"):  # replays of the captured step: one mean per round
            g = eng.make_graph(mine, case["round"])
            means = []
            for _ in range(case["graph"]):
                g.launch()
                T.cuda.synchronize()
                means.append(eng.mean.cpu().numpy().copy())
            eng.check()
            q.put((rank, means, None))
            comm.barrier()
            return
        if case.get("nan_rank") == rank:
            mine[0][5] = float("nan")
        eng.run(mine, case["round"])
        if case.get("nan_rank") is not None:
            try:
                eng.check()
                q.put((rank, None, "no error raised"))
            except _lib.InvalidArgument as e:
                q.put((rank, "raised", None))
            comm.barrier()
            return
        eng.check()
        T.cuda.synchronize()
        q.put((rank, eng.mean.cpu().numpy(), None))
        comm.barrier()  # keep the mappings alive until every rank is done
    except Exception as e:  # pragma: no cover - surfaced by the test
        q.put((rank, None, repr(e)))
