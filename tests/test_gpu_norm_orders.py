"""General norm orders (norms.cpp:34-75: q, p in 1..16 besides 2 / inf).

The device forms sum_j |x_j|^q per worker with correctly rounded powers over
the d-only partition of the L2 sums; the root pow(acc, 1/q), the p-th power
and the tree fold run on the host with the reference's own libm calls
(gq_capi.cu norm_general). The reference sums std::pow(|x|, q) in element
order and glibc's pow is not correctly rounded, so the stats agree to
rounding (relative 1e-13 here), like the parallel L2 sum; with one element
per worker the sum is exact and the stat is bit-identical.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2305_18627_b200 import gqsgd as G

pytestmark = pytest.mark.gpu
INF = G.NORM_INF


def ref_or_oracle(reference, oracle):
    return reference if reference is not None else oracle


def cr_pow(x: float, q: int) -> float:
    return float(Fraction(abs(x)) ** q)  # correctly rounded |x|^q


def host_stat(nq: float, p: int) -> float:
    if p == INF:
        return nq
    if p == 2:
        return nq * nq
    return math.pow(nq, float(p))


@pytest.mark.parametrize("q,p", [(3, INF), (1, 1), (4, 3), (16, 2), (7, 16), (INF, 3), (2, 5)])
def test_single_element_stats_bit_exact(cuda, q, p):
    """One element per worker: the device sum is the correctly rounded power
    itself, the host applies pow(., 1/q) and the p-th power as norms.cpp."""
    gen = np.random.default_rng(q * 31 + (p if p != INF else 99))
    xs = (gen.standard_normal(6) * 2.0 ** gen.integers(-12, 12, 6)).astype(np.float32)
    shards = [torch.tensor([v], device=cuda) for v in xs]
    stats = G.local_norm_stats(shards, G.NormSpec(q, p)).cpu().numpy()
    for w, v in enumerate(xs.astype(np.float64)):
        if q == INF:
            nq = abs(v)
        elif q == 2:
            nq = math.sqrt(v * v)
        else:
            nq = math.pow(cr_pow(v, q), 1.0 / q)
        assert stats[w] == host_stat(nq, p), (w, v, q, p)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("q,p", [(1, 1), (3, 3), (4, INF), (16, 2), (INF, 3), (2, 7), (5, 16)])
def test_stats_and_global_norm_match_reference(cuda, reference, oracle, dtype, q, p):
    ref = ref_or_oracle(reference, oracle)
    gen = np.random.default_rng(17)
    n, d = 4, 5003
    x = gen.standard_normal((n, d)) * np.array([1.0, 0.5, 3.0, 1e-3])[:, None]
    x = x.astype(np.float32).astype(np.float64)
    shards = [torch.from_numpy(x[w]).to(cuda, dtype) for w in range(n)]
    stats, norm = G.global_norm(shards, G.NormSpec(q, p))
    stats = stats.cpu().numpy()
    want = np.array([ref.local_norm_stat(x[w], q, p) for w in range(n)])
    np.testing.assert_allclose(stats, want, rtol=1e-13, atol=0)
    wn = ref.norm_allreduce_inproc(want, q, p) if hasattr(ref, "norm_allreduce_inproc") else \
        ref.norm_tree_combine(want, q, p)
    assert float(norm.item()) == pytest.approx(wn, rel=1e-13)
    # the device fold of the device stats: the host fold of the same stats, exactly
    assert float(G.combine_norm_stats(torch.from_numpy(stats).to(cuda), G.NormSpec(q, p)).item()) == \
        float(norm.item())


@pytest.mark.parametrize("kind,s,w", [(G.LevelKind.Standard, 15, 8), (G.LevelKind.Exponential, 4, 8)])
def test_sync_with_general_orders_matches_reference(cuda, reference, oracle, kind, s, w):
    ref = ref_or_oracle(reference, oracle)
    gen = np.random.default_rng(5)
    n, d = 4, 3001
    x = gen.standard_normal((n, d)).astype(np.float32).astype(np.float64)
    spec = G.NormSpec(3, 3)
    cfg = G.GqsgdConfig(workers=n, scheme=kind, s=s, width_bits=w, seed=9, norm=spec)
    res = G.gqsgd_mean([torch.from_numpy(x[r]).to(cuda) for r in range(n)], cfg, 2)
    mean, norm, lw = ref.mean(x, int(kind), s, 3, 3, width=w, seed=9, round=2)
    assert res.norm == pytest.approx(norm, rel=1e-13)
    # the same levels wherever the dither is not within ~1e-13 of a boundary
    # (every element here); the decoded values carry the norm's last bits
    np.testing.assert_allclose(res.mean.cpu().numpy().astype(np.float64), mean.astype(np.float32), rtol=1e-6,
                               atol=0)
    nz = mean != 0
    assert np.array_equal(res.mean.cpu().numpy() != 0, nz)


def test_general_orders_refused_where_the_device_folds(cuda):
    from paper_2305_18627_b200 import _lib
    n, d = 2, 1024
    shards = [torch.randn(d, device=cuda) for _ in range(n)]
    cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind.Standard, s=7, width_bits=8, seed=1, norm=G.NormSpec(3, 3))
    eng = G.InprocSync(cfg, d, cuda)
    with pytest.raises(G.InvalidArgument):
        eng.graph(shards, 0)
    for bad in (0, 17):
        with pytest.raises(G.InvalidArgument):
            G.plan_path(G.GqsgdConfig(workers=n, s=7, norm=G.NormSpec(bad, 2)))
    assert _lib.lib() is not None


def test_general_orders_zero_and_nonfinite(cuda):
    """An all-zero worker has stat 0 (pow(0, 1/q) = 0, pow(0, p) = 0); a NaN or
    Inf raises invalid_argument as local_norm_stat does (norms.cpp:52-57)."""
    spec = G.NormSpec(3, 4)
    z = [torch.zeros(4099, device=cuda), torch.ones(4099, device=cuda)]
    stats, norm = G.global_norm(z, spec)
    st = stats.cpu().numpy()
    assert st[0] == 0.0
    assert st[1] == math.pow(math.pow(4099.0, 1.0 / 3), 4.0)
    assert float(norm.item()) == math.pow(st[0] + st[1], 1.0 / 4)
    for bad in (float("nan"), float("inf")):
        x = torch.ones(4099, device=cuda)
        x[1234] = bad
        with pytest.raises(G.InvalidArgument):
            G.global_norm([x, z[1]], spec)
