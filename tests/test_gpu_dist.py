"""The multi-rank path (paper_2305_18627_b200/dist.py) with the real sm_100a
kernels on one B200.

Only one GPU is available to the tests, so N ranks run as N threads of this
process (ThreadComm: the collectives become device copies) on cuda:0, plus a
real single-rank NCCL process group. Every rank's decoded mean and summed
lanes must equal the reference's bits (oracle pinned to the reference;
full-size runs against the reference's own fingerprints).
"""
import hashlib
import os
import threading

import numpy as np
import pytest
import torch

from dist_fakes import ThreadComm, free_port

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFF


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_virtual(x, cfg, world, round, exchange="pull", sgd=False):
    from paper_2305_18627_b200.dist import DeviceKernels, DistSync

    n, d = x.shape
    comms = ThreadComm.group(world)
    out = [None] * world
    errs = []
    dev = torch.device("cuda:0")

    def body(r):
        try:
            torch.cuda.set_device(dev)
            eng = DistSync(cfg, d, comm=comms[r], kernels=DeviceKernels(dev), device=dev,
                           exchange=exchange)
            mine = [torch.from_numpy(x[w].copy()).to(dev) for w in eng.worker_ids]
            param = torch.ones(d, dtype=torch.float32, device=dev) if sgd else None
            eng.run(mine, round, param=param, lr=0.5)
            eng.check()
            torch.cuda.synchronize()
            out[r] = dict(mean=eng.mean.cpu().numpy(), summed=None if cfg.sparse else eng.summed_payload.cpu().numpy(),
                          norm=float(eng.norm.item()),
                          param=None if param is None else param.cpu().numpy())
        except BaseException as e:  # surfaced by the caller
            errs.append(e)
            comms[r].sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return out


CASES = [
    dict(n=8, d=4099, kind=1, s=4, width=4, topo=0, seed=42, round=3, data_seed=12345, world=8),
    dict(n=8, d=4099, kind=1, s=4, width=4, topo=0, seed=42, round=3, data_seed=12345, world=2),
    dict(n=8, d=3000, kind=0, s=15, width=8, topo=1, seed=7, round=0, data_seed=1, world=4),
    dict(n=6, d=2000, kind=1, s=7, width=8, topo=1, seed=8, round=2, data_seed=3, q=2, p=2, world=3, sgd=True),
    dict(n=4, d=5000, kind=0, s=31, width=8, topo=0, seed=6, round=1, data_seed=5, world=4, exchange="nccl_sum"),
    dict(n=4, d=5000, kind=0, s=1000, width=16, topo=0, seed=6, round=1, data_seed=5, world=2),
    dict(n=4, d=999, kind=0, s=1, width=4, topo=0, seed=2, round=4, data_seed=6, world=4),
]


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_virtual_ranks_match_reference(cuda, oracle, ci):
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind, NormSpec, TopologyKind

    c = CASES[ci]
    x = oracle.gaussian_shards(c["n"], c["d"], c["data_seed"]).astype(np.float32)
    cfg = GqsgdConfig(workers=c["n"], scheme=LevelKind(c["kind"]), s=c["s"], width_bits=c["width"],
                      topo=TopologyKind(c["topo"]), seed=c["seed"],
                      norm=NormSpec(c.get("q", INF), c.get("p", INF)))
    out = run_virtual(x, cfg, c["world"], c["round"], c.get("exchange", "pull"), c.get("sgd", False))
    mean, norm, lw, summed = oracle.mean(x.astype(np.float64), c["kind"], c["s"], q=c.get("q", INF),
                                         p=c.get("p", INF), width=c["width"], topo=c["topo"],
                                         seed=c["seed"], round=c["round"])
    for r, o in enumerate(out):
        if c.get("q", INF) == INF:
            assert o["norm"] == norm
            assert np.array_equal(o["summed"], summed), r
            assert np.array_equal(o["mean"], mean.astype(np.float32)), r
        else:  # L2: the norm is within 1e-12; levels checked with the device norm injected
            assert abs(o["norm"] - norm) <= 1e-12 * norm
            m2, _, _, s2 = oracle.mean(x.astype(np.float64), c["kind"], c["s"], q=c["q"], p=c["p"],
                                       width=c["width"], topo=c["topo"], seed=c["seed"],
                                       round=c["round"], norm_override=o["norm"])
            assert np.array_equal(o["summed"], s2), r
            assert np.array_equal(o["mean"], m2.astype(np.float32)), r
            mean = m2
        if c.get("sgd"):
            assert np.array_equal(o["param"], np.float32(1) - np.float32(0.5) * mean.astype(np.float32))


def test_virtual_ranks_full_size_c2(cuda, oracle, fingerprints):
    """C2 at its BASELINE size (d = 2^24, n = 8, 4-bit) over 8 virtual ranks:
    the decoded mean equals the reference's fingerprint."""
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind, TopologyKind

    f = fingerprints["C2_exp_s4_n8_d2^24"]
    x = oracle.gaussian_shards(f["n"], f["d"], f["data_seed"]).astype(np.float32)
    cfg = GqsgdConfig(workers=f["n"], scheme=LevelKind(f["kind"]), s=f["s"], width_bits=4,
                      topo=TopologyKind(f["topo"]), seed=f["seed"])
    out = run_virtual(x, cfg, 8, f["round"])
    for o in out:
        assert o["norm"] == f["norm"]
        assert _sha(o["mean"]) == f["mean_f32_sha"]


@pytest.mark.parametrize("exchange", ["pull", "nccl_sum"])
def test_single_rank_nccl_group(cuda, oracle, exchange):
    """A real NCCL process group (world 1): the TorchComm plumbing end to end."""
    import torch.distributed as dist

    from paper_2305_18627_b200.dist import gqsgd_mean_dist
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        n, d = 4, 10000
        x = oracle.gaussian_shards(n, d, 77).astype(np.float32)
        cfg = GqsgdConfig(workers=n, scheme=LevelKind.Standard, s=31, width_bits=8, seed=5)
        mean = gqsgd_mean_dist([torch.from_numpy(x[w]).to(cuda) for w in range(n)], cfg, 9,
                               exchange=exchange)
        want, _, _, _ = oracle.mean(x.astype(np.float64), 0, 31, width=8, seed=5, round=9)
        assert np.array_equal(mean.cpu().numpy(), want.astype(np.float32))
    finally:
        dist.destroy_process_group()


def test_ddp_comm_hook_single_rank_nccl(cuda, oracle):
    """gqsgd_hook inside real DDP on the GPU (NCCL, world 1): each synced
    bucket equals the device gqsgd_mean of that bucket with the hook's round."""
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2305_18627_b200.ddp_hook import ROUND_STRIDE, GqsgdHookState, gqsgd_hook
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.Tanh(), torch.nn.Linear(256, 8)).to(cuda)
        ddp = DDP(model, device_ids=[0], bucket_cap_mb=0.01)
        state = GqsgdHookState(GqsgdConfig(scheme=LevelKind.Standard, s=15, width_bits=8, seed=3))
        records = []

        def recording_hook(st, bucket):
            inp = bucket.buffer().detach().clone()
            rnd = st.step * ROUND_STRIDE + bucket.index()
            fut = gqsgd_hook(st, bucket)
            fut.wait()  # CUDA-aware future: the current stream waits for the side-stream sync
            records.append((rnd, inp, fut.value().detach().clone()))
            return fut

        ddp.register_comm_hook(state, recording_hook)
        for step in range(3):
            x = torch.randn(32, 64, device=cuda)
            ddp.zero_grad()
            ddp(x).pow(2).mean().backward()
        torch.cuda.synchronize()
        state.check()
        assert state.step == 3 and len(records) >= 3
        for rnd, inp, out in records:
            want, _, _, _ = oracle.mean(inp.double().cpu().numpy()[None, :], 0, 15, width=8, seed=3, round=rnd)
            assert np.array_equal(out.cpu().numpy(), want.astype(np.float32))
    finally:
        dist.destroy_process_group()


def test_ddp_comm_hook_float64_buckets(cuda, oracle):
    """An fp64 model: the hook decodes in f64 (algorithm.cpp:84-110), so each
    synced bucket equals the reference's doubles bit for bit, not fl32 of them."""
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2305_18627_b200.ddp_hook import ROUND_STRIDE, GqsgdHookState, gqsgd_hook
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        torch.manual_seed(1)
        model = torch.nn.Sequential(torch.nn.Linear(32, 128), torch.nn.Tanh(), torch.nn.Linear(128, 4)).to(cuda)
        model = model.double()
        ddp = DDP(model, device_ids=[0], bucket_cap_mb=0.01)
        state = GqsgdHookState(GqsgdConfig(scheme=LevelKind.Exponential, s=7, width_bits=8, seed=4))
        records = []

        def recording_hook(st, bucket):
            inp = bucket.buffer().detach().clone()
            rnd = st.step * ROUND_STRIDE + bucket.index()
            fut = gqsgd_hook(st, bucket)
            fut.wait()
            records.append((rnd, inp, fut.value().detach().clone()))
            return fut

        ddp.register_comm_hook(state, recording_hook)
        for step in range(2):
            x = torch.randn(16, 32, device=cuda, dtype=torch.float64)
            ddp.zero_grad()
            ddp(x).pow(2).mean().backward()
        torch.cuda.synchronize()
        state.check()
        assert len(records) >= 2
        for rnd, inp, out in records:
            assert out.dtype == torch.float64
            want, _, _, _ = oracle.mean(inp.cpu().numpy()[None, :], 1, 7, width=8, seed=4, round=rnd)
            assert np.array_equal(out.cpu().numpy(), want)
    finally:
        dist.destroy_process_group()


def test_bucketed_pipeline_single_rank_nccl(cuda, oracle):
    """BucketedSync on a real NCCL group with asynchronous collectives."""
    import torch.distributed as dist

    from paper_2305_18627_b200.dist import BucketedSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        sizes = [5000, 1234, 9999]
        n = 4
        cfg = GqsgdConfig(workers=n, scheme=LevelKind.Exponential, s=4, width_bits=4, seed=8)
        pipe = BucketedSync(cfg, sizes, device=cuda)
        data = [oracle.gaussian_shards(n, sz, 70 + b).astype(np.float32) for b, sz in enumerate(sizes)]
        pipe.run([[torch.from_numpy(data[b][w]).to(cuda) for w in range(n)] for b in range(3)], [5, 6, 7])
        pipe.check()
        for b in range(3):
            want, _, _, _ = oracle.mean(data[b].astype(np.float64), 1, 4, width=4, seed=8, round=5 + b)
            assert np.array_equal(pipe.syncs[b].mean.cpu().numpy(), want.astype(np.float32))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,s,width,world", [(0, 2, 8, 4), (1, 7, 16, 2)])
def test_virtual_ranks_sparse_allgather(cuda, oracle, reference, kind, s, width, world):
    """cfg.sparse over N virtual ranks: encode, all_gather of sizes and padded
    payloads, rank-ordered accumulate == the reference's gqsgd_mean(sparse)."""
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    if reference is None:
        pytest.skip("reference library not built")
    n, d = 4, 2500
    x = oracle.gaussian_shards(n, d, 321).astype(np.float32)
    cfg = GqsgdConfig(workers=n, scheme=LevelKind(kind), s=s, width_bits=width, seed=13, sparse=True)
    out = run_virtual(x, cfg, world, 6, sgd=True)
    want, wnorm, _ = reference.mean_sparse(x.astype(np.float64), kind, s, width=width, seed=13, round=6)
    for o in out:
        assert o["norm"] == wnorm
        assert np.array_equal(o["mean"], want.astype(np.float32))
        assert np.array_equal(o["param"], np.float32(1) - np.float32(0.5) * want.astype(np.float32))


@pytest.mark.parametrize("kind,s,width,world,d,per", [(1, 4, 4, 8, 100003, 1), (0, 15, 8, 4, 50000, 1),
                                                      (1, 7, 8, 2, 1234, 1), (0, 31, 16, 2, 70001, 1),
                                                      (1, 4, 4, 2, 60001, 4), (0, 7, 8, 4, 9000, 2)])
def test_virtual_ranks_peer_memory_exchange(cuda, oracle, kind, s, width, world, d, per):
    """exchange="p2p": quantize stores slices straight into the owners' rows,
    epoch flags, reduce stores the summed slice into every peer (here the
    ranks are threads sharing one B200, so peer pointers are plain device
    pointers; across GPUs they are CUDA-IPC mappings)."""
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    x = oracle.gaussian_shards(world * per, d, 55 + world).astype(np.float32)
    cfg = GqsgdConfig(workers=world * per, scheme=LevelKind(kind), s=s, width_bits=width, seed=12)
    out = run_virtual(x, cfg, world, 8, exchange="p2p", sgd=True)
    mean, norm, lw, summed = oracle.mean(x.astype(np.float64), kind, s, width=width, seed=12, round=8)
    for r, o in enumerate(out):
        assert o["norm"] == norm
        assert np.array_equal(o["summed"], summed), r
        assert np.array_equal(o["mean"], mean.astype(np.float32)), r
        assert np.array_equal(o["param"], np.float32(1) - np.float32(0.5) * mean.astype(np.float32))


def test_virtual_ranks_one_worker_per_rank_large_d(cuda):
    """One worker per rank with the k draws in the norm pass at a large d
    (the N = 8 C2 shape per rank): the norm grid must fit the workspace's
    partials (a one-worker norm with the k draws once asked for two waves of
    blocks, more partials than the workspace holds). Checked against the
    single-device sync of the same shards."""
    from paper_2305_18627_b200 import gqsgd as G
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    d = 1 << 24
    gen = np.random.default_rng(4)
    x = gen.standard_normal((2, d)).astype(np.float32)
    cfg = GqsgdConfig(workers=2, scheme=LevelKind.Exponential, s=4, width_bits=4, seed=21)
    out = run_virtual(x, cfg, 2, 3, exchange="p2p")
    res = G.gqsgd_mean([torch.from_numpy(x[w]).to(cuda) for w in range(2)], cfg, 3)
    want = res.mean.cpu().numpy()
    for r, o in enumerate(out):
        assert o["norm"] == res.norm == float(np.abs(x).max()), r
        assert np.array_equal(o["mean"], want), r


@pytest.mark.parametrize("q", [2, "inf"])
def test_shard_stat_independent_of_n_and_k_draws(cuda, q):
    """A worker's stat (the parallel L2 partial sums included) depends on its
    data and d only: reduced beside 7 others without the k draws, alone with
    them (an N = 8 rank), or beside 3 others with them, the stats are the
    same bits. d is ragged (a scalar tail in the last slice)."""
    import ctypes as C

    from paper_2305_18627_b200 import _lib
    from paper_2305_18627_b200.gqsgd import NORM_INF

    q = NORM_INF if q == "inf" else 2
    L = _lib.lib()
    d = (1 << 24) + 3
    n = 8
    gen = torch.Generator(device=cuda).manual_seed(5)
    xs = [torch.randn(d, device=cuda, generator=gen) for _ in range(n)]
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    ws = torch.zeros(int(L.gq_norm_workspace_bytes(n, d)), dtype=torch.uint8, device=cuda)
    INF = 0xFFFFFFFF
    sp = torch.cuda.current_stream().cuda_stream

    def stats_of(shards, kdraws):
        k = len(shards)
        st = torch.zeros(k, dtype=torch.float64, device=cuda)
        nm = torch.zeros(1, dtype=torch.float64, device=cuda)
        arr = _lib.ptr_array([t.data_ptr() for t in shards])
        if kdraws:
            spec = _lib.GqKdraws(None, n, 1, 4, 4, 0, 0, 0, min(d, 1 << 21), 9, 0)
            kb = int(L.gq_kdraws_bytes(C.byref(spec)))
            buf = torch.empty(max(kb, 4) // 4, dtype=torch.int32, device=cuda)
            spec.buf = buf.data_ptr()
            _lib.check(L.gq_norm_kdraws(arr, 0, k, d, q, INF, st.data_ptr(), nm.data_ptr(), ws.data_ptr(),
                                        err.data_ptr(), C.byref(spec), sp))
        else:
            _lib.check(L.gq_norm(arr, 0, k, d, q, INF, st.data_ptr(), nm.data_ptr(), ws.data_ptr(),
                                 err.data_ptr(), sp))
        torch.cuda.synchronize()
        return st.cpu().numpy()

    base = stats_of(xs, False)
    for r in range(n):
        assert stats_of([xs[r]], True)[0] == base[r], r
    assert np.array_equal(stats_of(xs[:4], True), base[:4])
    assert np.array_equal(stats_of(xs, True), base)
    if q == 2:  # the parallel L2 (f64 partials) against numpy's f64 norm (p = inf: the stat is the norm)
        want = np.array([float(np.sqrt(np.sum(x.double().cpu().numpy() ** 2))) for x in xs])
        assert np.allclose(base, want, rtol=1e-12)


def test_virtual_ranks_peer_memory_exchange_unfolded(cuda, oracle):
    """GQ_OPT_COMM_FOLD = 0: the eager exchange with separate signal kernels
    gives the same bits."""
    from paper_2305_18627_b200 import _lib
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_COMM_FOLD, 0))
    try:
        x = oracle.gaussian_shards(4, 30001, 91).astype(np.float32)
        cfg = GqsgdConfig(workers=4, scheme=LevelKind.Exponential, s=4, width_bits=4, seed=12)
        out = run_virtual(x, cfg, 4, 8, exchange="p2p", sgd=True)
    finally:
        _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_COMM_FOLD, 1))
    mean, norm, lw, summed = oracle.mean(x.astype(np.float64), 1, 4, width=4, seed=12, round=8)
    for r, o in enumerate(out):
        assert o["norm"] == norm and np.array_equal(o["mean"], mean.astype(np.float32)), r


@pytest.mark.parametrize("fold", [1, 0])
def test_world1_comm_graph_replays(cuda, oracle, fold):
    """DistSync(exchange='p2p') at world 1: the captured step (gq_comm_graph)
    replays rounds r, r+1, ... with the eager path's bits - with the exchange
    steps folded into the kernels (default) and as separate kernels
    (GQ_OPT_COMM_FOLD = 0)."""
    from paper_2305_18627_b200 import _lib
    from paper_2305_18627_b200.dist import DeviceKernels, DistSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_COMM_FOLD, fold))
    try:
        _world1_comm_graph(cuda, oracle)
    finally:
        _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_COMM_FOLD, 1))


def _world1_comm_graph(cuda, oracle):
    from paper_2305_18627_b200.dist import DeviceKernels, DistSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    n, d = 4, 30001
    x = oracle.gaussian_shards(n, d, 77).astype(np.float32)
    cfg = GqsgdConfig(workers=n, scheme=LevelKind.Standard, s=15, width_bits=8, seed=5)
    dev = torch.device("cuda:0")
    comm = ThreadComm.group(1)[0]
    eng = DistSync(cfg, d, comm=comm, kernels=DeviceKernels(dev), device=dev, exchange="p2p")
    shards = [torch.from_numpy(x[w].copy()).to(dev) for w in range(n)]
    param = torch.ones(d, dtype=torch.float32, device=dev)
    g = eng.make_graph(shards, 20, param=param, lr=0.5)
    for i in range(3):
        g.launch()
        torch.cuda.synchronize()
        want, _, _, _ = oracle.mean(x.astype(np.float64), 0, 15, width=8, seed=5, round=20 + i)
        assert np.array_equal(eng.mean.cpu().numpy(), want.astype(np.float32)), i
    eng.check()
    assert int(g.round.item()) == 23


def test_bench_two_ranks_on_one_gpu(cuda):
    """bench.py's N-rank path end to end (torchrun, 2 processes): both ranks on
    cuda:0 (gloo plumbing, CUDA-IPC peer exchange with host waits). Timing is
    meaningless here; the JSON line must be complete and its dist_check must
    find every rank bit-identical to the single-device path."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GQ_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--workload", "c1", "--steps", "3", "--warmup", "3", "--no-cpu"]
    p = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 prints one line
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["execution"]["exchange"] == "p2p"
    assert line["dist_check"]["all_ranks_bit_identical_to_single_device"] is True
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
