"""The peer-memory exchange across PROCESSES: two ranks on one B200 map each
other's receive / summed / flag buffers with CUDA IPC (gq_ipc_get /
gq_ipc_open) exactly as ranks on different GPUs of an NVSwitch node do, and
synchronise through the system-scope epoch flags."""
import multiprocessing as mp

import numpy as np
import pytest

from dist_fakes import free_port, ipc_worker

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [dict(kind=1, s=4, width=4, d=40000, data_seed=3, seed=5, round=2),
                                  dict(kind=0, s=31, width=8, d=9999, data_seed=4, seed=6, round=7),
                                  dict(kind=1, s=7, width=8, d=30001, data_seed=5, seed=7, round=1, per=3),
                                  # waits in a spinning device kernel (the multi-GPU mode) across processes
                                  dict(kind=1, s=4, width=4, d=65536, data_seed=6, seed=8, round=4, wait=1),
                                  dict(kind=0, s=15, width=8, d=5000, data_seed=7, seed=9, round=5, per=2, wait=1)])
def test_ipc_peer_exchange_two_processes(cuda, oracle, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    world = 2
    procs = [ctx.Process(target=ipc_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, mean, err = q.get(timeout=300)
            assert err is None, err
            res[r] = mean
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    x = oracle.gaussian_shards(world * case.get("per", 1), case["d"], case["data_seed"]).astype(np.float32).astype(np.float64)
    want, _, _, _ = oracle.mean(x, case["kind"], case["s"], width=case["width"], seed=case["seed"], round=case["round"])
    for r in range(world):
        assert np.array_equal(res[r], want.astype(np.float32)), r


def test_ipc_error_reaches_every_rank(cuda):
    """A NaN in rank 1's shard raises invalid_argument on BOTH ranks (gq_sync)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    case = dict(kind=0, s=15, width=8, d=3000, data_seed=8, seed=1, round=0, nan_rank=1)
    procs = [ctx.Process(target=ipc_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, got, err = q.get(timeout=300)
            assert err is None, err
            res[r] = got
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    assert res == {0: "raised", 1: "raised"}


def test_ipc_graph_replays(cuda, oracle):
    """gq_comm_graph across two processes (device-side waits): each replay is
    one step with the next round, bit-identical to the reference."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    case = dict(kind=1, s=4, width=4, d=50001, data_seed=9, seed=3, round=10, wait=1, graph=3, per=2)
    procs = [ctx.Process(target=ipc_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, means, err = q.get(timeout=300)
            assert err is None, err
            res[r] = means
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    x = oracle.gaussian_shards(4, case["d"], case["data_seed"]).astype(np.float32).astype(np.float64)
    for i in range(3):
        want, _, _, _ = oracle.mean(x, 1, 4, width=4, seed=3, round=10 + i)
        for r in (0, 1):
            assert np.array_equal(res[r][i], want.astype(np.float32)), (r, i)


def test_absent_peer_times_out_instead_of_hanging(cuda):
    """A rank whose peer never arrives: every device wait gives up after
    GQ_OPT_COMM_TIMEOUT_S and gq_sync raises the reference's runtime_error
    class instead of the GPU hanging."""
    import ctypes as C
    import time

    import torch

    from paper_2305_18627_b200 import _lib
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    L = _lib.lib()
    d = 4096
    cfg = GqsgdConfig(workers=2, scheme=LevelKind.Standard, s=15, width_bits=8, seed=1).to_c()
    comms = []
    try:
        _lib.check(L.gq_set_option(_lib.GQ_OPT_COMM_WAIT, 1))  # spinning device waits
        _lib.check(L.gq_set_option(_lib.GQ_OPT_COMM_TIMEOUT_S, 1))
        hb = int(L.gq_comm_handle_bytes())
        blobs = (C.c_char * (2 * hb))()
        for r in range(2):
            p = C.c_void_p()
            _lib.check(L.gq_comm_init(r, 2, C.byref(cfg), d, C.byref(p)))
            comms.append(p.value)
            h = (C.c_char * hb)()
            _lib.check(L.gq_comm_handle(p, h))
            C.memmove(C.addressof(blobs) + r * hb, h, hb)
        for c in comms:
            _lib.check(L.gq_comm_connect(c, blobs))
        x = torch.randn(d, device=cuda)
        mean = torch.empty(d, device=cuda)
        err = torch.zeros(1, dtype=torch.int32, device=cuda)
        sp = torch.cuda.current_stream().cuda_stream
        t0 = time.time()
        _lib.check(L.gq_comm_mean(comms[0], _lib.ptr_array([x.data_ptr()]), _lib.GQ_DTYPE_F32, 3, mean.data_ptr(),
                                  None, None, 0.0, None, err.data_ptr(), sp))  # rank 1 never runs
        with pytest.raises(_lib.RuntimeFailure):
            _lib.check(L.gq_sync(comms[0], err.data_ptr(), sp))
        assert time.time() - t0 < 30
    finally:
        L.gq_set_option(_lib.GQ_OPT_COMM_WAIT, 0)
        L.gq_set_option(_lib.GQ_OPT_COMM_TIMEOUT_S, 60)
        torch.cuda.synchronize()
        for c in comms:
            L.gq_comm_destroy(c)
