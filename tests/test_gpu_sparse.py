"""The sparse allgather path (cfg.sparse) on the device vs the unmodified
reference: wire payloads byte for byte (serialize_sparse(to_sparse(...))),
the accumulated mean (accumulate_sparse in rank order / n) in f64 bit for
bit, the fp32 mean as fl32 of it, and malformed payloads -> domain_error."""
import numpy as np
import pytest
import torch

from paper_2305_18627_b200 import gqsgd as G
from paper_2305_18627_b200.gqsgd import DomainError, GqsgdConfig, InvalidArgument, LevelKind, NormSpec

pytestmark = pytest.mark.gpu
INF = 0xFFFFFFFF


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("kind,s,width,d", [(0, 2, 8, 1000), (0, 15, 8, 4099), (0, 300, 16, 777), (1, 7, 8, 5000),
                                            (1, 3, 32, 1), (1, 30, 8, 9000), (0, 1, 8, 64)])
def test_sparse_payload_bytes_equal_reference(cuda, reference, oracle, kind, s, width, d):
    if reference is None:
        pytest.skip("reference library not built")
    x = oracle.gaussian_shards(2, d, 17 + d).astype(np.float32)
    norm = float(np.abs(x).max())
    for r in range(2):
        want = reference.sparse_payload(x[r].astype(np.float64), norm, kind, s, 9, r, 33, width)
        got = G.sparse_payload(dev(x[r]), norm, LevelKind(kind), s, 9, r, 33, width).cpu().numpy()
        assert np.array_equal(got, want), (r, got.size, want.size)


@pytest.mark.parametrize("kind,s,n,width,q", [(0, 2, 4, 8, INF), (1, 7, 3, 8, INF), (0, 15, 8, 8, 2),
                                              (1, 4, 5, 16, INF), (0, 255, 2, 8, INF)])
def test_sparse_gqsgd_mean_equals_reference(cuda, reference, oracle, kind, s, n, width, q):
    if reference is None:
        pytest.skip("reference library not built")
    d = 3001
    x = oracle.gaussian_shards(n, d, 5 + n).astype(np.float32)
    cfg = GqsgdConfig(workers=n, scheme=LevelKind(kind), s=s, width_bits=width, seed=4, sparse=True,
                      norm=NormSpec(q, q))
    res = G.gqsgd_mean([dev(x[r]) for r in range(n)], cfg, 12)
    want, wnorm, _ = reference.mean_sparse(x.astype(np.float64), kind, s, q=q, p=q, width=width, seed=4, round=12)
    if q == INF:
        assert res.norm == wnorm
        assert np.array_equal(res.mean.cpu().numpy(), want.astype(np.float32))
    else:
        assert res.norm == pytest.approx(wnorm, rel=1e-12)
    # the wire path: every worker's payload accumulated in rank order, f64 bit-exact
    pays = [G.sparse_payload(dev(x[r]), res.norm, LevelKind(kind), s, 4, r, 12, width) for r in range(n)]
    acc = G.sparse_accumulate(pays, d, LevelKind(kind), s, width, out_f64=True).cpu().numpy()
    if q == INF:
        assert np.array_equal(acc, want)
    assert np.array_equal(acc.astype(np.float32), res.mean.cpu().numpy())


def test_sparse_errors(cuda, oracle):
    with pytest.raises(InvalidArgument, match="does not fit"):
        G.sparse_lane_width(8, 256)
    x = oracle.gaussian_shards(1, 100, 3).astype(np.float32)
    p = G.sparse_payload(dev(x[0]), float(np.abs(x).max()), LevelKind.Standard, 3, 1, 0, 0, 8)
    bad = p.clone()
    bad[8] = 99  # dim disagrees with d
    with pytest.raises(DomainError):
        G.sparse_accumulate([bad], 100, LevelKind.Standard, 3, 8)
    bad = p.clone()
    bad[16:20] = bad[20:24].clone()  # duplicate index -> not strictly increasing
    with pytest.raises(DomainError):
        G.sparse_accumulate([bad], 100, LevelKind.Standard, 3, 8)
