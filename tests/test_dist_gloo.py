"""Multi-rank host logic of paper_2305_18627_b200/dist.py on CPU.

world_size 2 over gloo (spawned processes, 127.0.0.1), kernels replaced by
the oracle (tests/dist_fakes.py), so what is tested is exactly the host
side: worker placement, slice geometry, the all_to_all / all_gather layout,
the stats exchange + tree fold, and round keys. The result must equal the
reference semantics of gqsgd_mean on the whole problem (the oracle is
pinned to the reference, tests/test_oracle_kat.py). The same DistSync with
the real kernels runs on the GPU in tests/test_gpu_dist.py.
"""
import multiprocessing as mp

import numpy as np
import pytest

from dist_fakes import OracleKernels, ThreadComm, free_port, gloo_worker

INF = 0xFFFFFFFF

CASES = [
    # C2 shape (exponential, 4-bit, tree), ragged d
    dict(n=4, d=1001, kind=1, s=4, width=4, topo=0, seed=42, round=3, data_seed=12345),
    # standard 8-bit over the ring schedule, n_local = 4
    dict(n=8, d=777, kind=0, s=15, width=8, topo=1, seed=7, round=0, data_seed=1),
    # exponential ring, 8-bit, L2 norm, fused SGD
    dict(n=6, d=700, kind=1, s=7, width=8, topo=1, seed=8, round=2, data_seed=3, q=2, p=2, sgd=True),
    # NCCL-style integer all_reduce of rank-local partial sums
    dict(n=4, d=640, kind=0, s=31, width=8, topo=0, seed=6, round=1, data_seed=5, exchange="nccl_sum"),
    # tiny d: rank 1's slice is empty
    dict(n=2, d=100, kind=1, s=7, width=8, topo=0, seed=1, round=0, data_seed=9),
    # the sparse allgather path, standard s=2 and exponential s=7 with SGD
    dict(n=4, d=500, kind=0, s=2, width=8, topo=0, seed=3, round=4, data_seed=11, sparse=True),
    dict(n=6, d=333, kind=1, s=7, width=16, topo=0, seed=4, round=5, data_seed=12, sparse=True, sgd=True),
]


def expected(oracle, c):
    x = oracle.gaussian_shards(c["n"], c["d"], c["data_seed"]).astype(np.float32).astype(np.float64)
    if c.get("sparse"):
        from oracle.bind import reference_or_none
        ref = reference_or_none()
        if ref is None:
            pytest.skip("the sparse path is checked against the compiled reference")
        mean, norm, _ = ref.mean_sparse(x, c["kind"], c["s"], width=c["width"], seed=c["seed"], round=c["round"])
        return mean, norm, c["width"], None
    mean, norm, lw, summed = oracle.mean(x, c["kind"], c["s"], q=c.get("q", INF), p=c.get("p", INF),
                                         width=c["width"], topo=c["topo"], seed=c["seed"],
                                         round=c["round"])
    return mean, norm, lw, summed


@pytest.fixture(scope="module")
def gloo_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=gloo_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, out = q.get(timeout=240)
            res[r] = out
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    return res


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_world2_gloo_equals_reference_semantics(gloo_results, oracle, ci):
    c = CASES[ci]
    mean, norm, lw, summed = expected(oracle, c)
    for r in (0, 1):
        got = gloo_results[r][ci]
        assert got["width"] == lw
        assert got["norm"] == norm
        if summed is not None:
            assert np.array_equal(got["summed"], summed)
        assert np.array_equal(got["mean"], mean.astype(np.float32))
        if c.get("sgd"):
            want = np.float32(1.0) - np.float32(0.5) * mean.astype(np.float32)
            assert np.array_equal(got["param"], want)


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_ranks_threads_equal_reference_semantics(oracle, world):
    """Same host logic with N ranks as threads (ThreadComm), CPU kernels."""
    import threading

    import torch

    from paper_2305_18627_b200.dist import DistSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind, TopologyKind

    c = dict(n=8, d=1500, kind=1, s=4, width=4, topo=0, seed=42, round=11, data_seed=12345)
    x = oracle.gaussian_shards(c["n"], c["d"], c["data_seed"]).astype(np.float32)
    comms = ThreadComm.group(world)
    out = [None] * world
    errs = []

    def body(r):
        try:
            cfg = GqsgdConfig(workers=c["n"], scheme=LevelKind(c["kind"]), s=c["s"], width_bits=c["width"],
                              topo=TopologyKind(c["topo"]), seed=c["seed"])
            eng = DistSync(cfg, c["d"], comm=comms[r], kernels=OracleKernels(oracle), device="cpu")
            eng.run([torch.from_numpy(x[w].copy()) for w in eng.worker_ids], c["round"])
            eng.check()
            out[r] = (eng.mean.numpy().copy(), eng.summed_payload.numpy().copy())
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            comms[r].sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not errs, errs
    mean, norm, lw, summed = expected(oracle, c)
    for r in range(world):
        assert np.array_equal(out[r][1], summed)
        assert np.array_equal(out[r][0], mean.astype(np.float32))


def test_dist_rejects_bad_configs():
    from paper_2305_18627_b200.dist import DistSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, InvalidArgument, LevelKind

    comms = ThreadComm.group(3)
    with pytest.raises(InvalidArgument):  # 4 workers over 3 ranks
        DistSync(GqsgdConfig(workers=4, scheme=LevelKind.Standard, s=15), 100, comm=comms[0],
                 kernels=object(), device="cpu")
    comms = ThreadComm.group(2)
    with pytest.raises(InvalidArgument):  # token reduce has no NCCL operator
        DistSync(GqsgdConfig(workers=4, scheme=LevelKind.Exponential, s=7), 100, comm=comms[0],
                 kernels=object(), device="cpu", exchange="nccl_sum")


def test_bucketed_pipeline_gloo(oracle):
    """dist.BucketedSync (all phases issued bucket by bucket with async
    collectives) gives each bucket's reference result."""
    from dist_fakes import bucketed_gloo_worker
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=bucketed_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, means = q.get(timeout=240)
            res[r] = means
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    sizes = [700, 333, 1024]
    for b, sz in enumerate(sizes):
        x = oracle.gaussian_shards(4, sz, 50 + b).astype(np.float32).astype(np.float64)
        want, _, _, _ = oracle.mean(x, 1, 7, width=8, seed=21, round=10 + b)
        for r in (0, 1):
            assert np.array_equal(res[r][b], want.astype(np.float32)), (b, r)


@pytest.mark.parametrize("exchange", ["p2p", "auto"])
def test_peer_exchange_falls_back_together(oracle, exchange):
    """When the ranks cannot map each other's memory (here: no GPU at all),
    every rank agrees to fall back to the NCCL-style pull exchange and the
    result is unchanged."""
    import threading

    import torch

    from paper_2305_18627_b200.dist import DistSync
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    if torch.cuda.is_available():
        pytest.skip("checks the no-peer-memory fallback")
    world, c = 2, dict(n=4, d=900, kind=1, s=7, width=8, topo=0, seed=5, round=2, data_seed=77)
    x = oracle.gaussian_shards(c["n"], c["d"], c["data_seed"]).astype(np.float32)
    comms = ThreadComm.group(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            cfg = GqsgdConfig(workers=c["n"], scheme=LevelKind(c["kind"]), s=c["s"], width_bits=c["width"],
                              seed=c["seed"])
            eng = DistSync(cfg, c["d"], comm=comms[r], kernels=OracleKernels(oracle), device="cpu",
                           exchange=exchange)
            eng.run([torch.from_numpy(x[w].copy()) for w in eng.worker_ids], c["round"])
            out[r] = (eng.exchange, eng.mean.numpy().copy())
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            comms[r].sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not errs, errs
    mean, _, _, _ = expected(oracle, c)
    for r in range(world):
        assert out[r][0] == "pull"
        assert np.array_equal(out[r][1], mean.astype(np.float32))
