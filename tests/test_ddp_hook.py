"""The DDP comm hook (paper_2305_18627_b200/ddp_hook.py) on CPU: world 2 over
gloo with the oracle kernels. Every bucket of every step must equal the
reference semantics of gqsgd_mean over both ranks' bucket inputs with
round = step * ROUND_STRIDE + bucket index."""
import multiprocessing as mp

import numpy as np
import pytest

from dist_fakes import ddp_gloo_worker, free_port


@pytest.fixture(scope="module")
def ddp_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=ddp_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            r, records, steps = q.get(timeout=240)
            res[r] = (records, steps)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    return res


def test_ddp_hook_buckets_equal_reference_semantics(ddp_results, oracle):
    (rec0, steps0), (rec1, steps1) = ddp_results[0], ddp_results[1]
    assert steps0 == steps1 == 2
    assert len(rec0) == len(rec1) >= 2  # buckets x 2 steps
    for (i0, r0, in0, out0), (i1, r1, in1, out1) in zip(rec0, rec1):
        assert (i0, r0) == (i1, r1)
        x = np.stack([in0, in1]).astype(np.float64)
        mean, _, _, _ = oracle.mean(x, 1, 7, width=8, seed=5, round=r0)
        assert np.array_equal(out0, mean.astype(np.float32))
        assert np.array_equal(out1, out0)
    rounds = {r for _, r, _, _ in rec0}
    assert len(rounds) == len(rec0)  # every (step, bucket) has its own round
