"""64-bit integer lanes on the device vs the unmodified reference.

What the reference does with 64 bits: standard_lane_width (algorithm.cpp:22-29)
lists a 64-bit candidate, but check_width (exp_arith.cpp:24-41) refuses
width_bits > 32, so gqsgd_mean never plans 64-bit lanes and refuses
n(s+1) > 2^31 - the device plan must refuse the same configurations. The
64-bit lane format itself is live in the reference as the IntSumOps{64}
plugin (collectives.cpp:23-27,60-81; test_collectives.cpp:68-80) and in
encode_dense_std / decode_dense_std's 8-byte case: those are checked byte for
byte here.
"""
import numpy as np
import pytest
import torch

from paper_2305_18627_b200 import gqsgd as G
from paper_2305_18627_b200.gqsgd import GqsgdConfig, LaneOverflow, LevelKind, TopologyKind

pytestmark = pytest.mark.gpu


def dev(a, device="cuda:0"):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def need(reference):
    if reference is None:
        pytest.skip("reference library not built")


def test_plan_refuses_like_the_reference(reference):
    """standard_lane_width walks {8, 16, 32, 64} but check_width refuses
    width_bits > 32 (exp_arith.cpp:26), so the reference never plans 64-bit
    lanes: n(s+1) > 2^31, or an explicit 64-bit request, is refused."""
    need(reference)
    for s, n, at_least in [(15, 8, 64), (1 << 24, 128, 8), ((1 << 31) - 1, 2, 8), (63, 2, 8),
                           (1 << 16, 1 << 5, 16), ((1 << 30) - 1, 2, 16)]:
        want = reference.standard_lane_width(s, n, at_least)
        got = G.standard_lane_width(s, n, at_least)
        assert got == want, (s, n, at_least, got, want)
    with pytest.raises(G.InvalidArgument):
        G.plan_path(GqsgdConfig(workers=8, scheme=LevelKind.Standard, s=15, width_bits=64))
    with pytest.raises(Exception):
        reference.mean(np.zeros((8, 16)), 0, 15, width=64)


@pytest.mark.parametrize("s,n,d,topo", [(15, 8, 3001, 0), (15, 5, 1999, 1), (1 << 24, 128, 257, 0), (3, 3, 5, 0)])
def test_int64_payloads_match_reference(cuda, oracle, reference, s, n, d, topo):
    """encode_dense_std at lane_width 64 (algorithm.cpp:69-82, the encoder's
    own 8-byte case) -> allreduce_inproc with IntSumOps{64} -> decode:
    lanes and summed lanes byte-identical to the reference's encoder and its
    IntSumOps plugin under the same schedule."""
    need(reference)
    x = oracle.gaussian_shards(n, d, 77).astype(np.float32)
    x64 = x.astype(np.float64)
    norm = float(np.abs(x64).max())
    lanes, dev_lanes = [], []
    for r in range(n):
        sign, idx = reference.quantize(x64[r], norm, 0, s, 9, r, 4)
        lanes.append(reference.encode(0, s, n, 64, sign, idx))
        got = G.quantize_shard(dev(x[r]), norm, LevelKind.Standard, s, 9, r, 4, 64, n)
        assert np.array_equal(got.cpu().numpy()[:8 * d], lanes[-1]), r
        dev_lanes.append(got)
    summed = reference.allreduce_inproc(np.stack(lanes), d, 0, 64, s, topo, 9, 4)[0]
    got_sum = G.allreduce_inproc(dev_lanes, d, LevelKind.Standard, 64, s, TopologyKind(topo), 9, 4)
    assert np.array_equal(got_sum.cpu().numpy()[:8 * d], summed)
    # decode_dense_std (algorithm.cpp:84-100) on the int64 sums, f32 and f64 outputs
    v = summed.view(np.int64)
    scale = norm / (float(n) * s)
    want64 = scale * v.astype(np.float64)
    mean = G.decode(got_sum, d, norm, LevelKind.Standard, s, n, 64)
    assert np.array_equal(mean.cpu().numpy(), want64.astype(np.float32))


def test_fused_sgd_64(cuda, oracle):
    """The int64 schedule replay with the fused SGD epilogue (trainer.cpp:335)."""
    n, d, s = 4, 4097, 15
    rng = np.random.default_rng(3)
    vals = [rng.integers(-s, s + 1, d, dtype=np.int64) for _ in range(n)]
    dev_lanes = [dev(np.pad(v.view(np.uint8), (0, 8))) for v in vals]
    norm = 1.5
    p0 = oracle.gaussian_shards(1, d, 6)[0].astype(np.float32)
    param = dev(p0.copy())
    lr = 0.125
    err = G._ErrWord.get(cuda)
    nt = torch.tensor([norm], dtype=torch.float64, device=cuda)
    G.check(G.lib().gq_reduce_lanes(G.ptr_array([t.data_ptr() for t in dev_lanes]), n, d, 0, d, 0, 64, s, 0, 1, 0,
                                    nt.data_ptr(), None, None, param.data_ptr(), lr, err.data_ptr(), G._stream()))
    G._sync_check(err)
    m32 = ((norm / (float(n) * s)) * sum(vals).astype(np.float64)).astype(np.float32)
    exp = (p0 - (np.float32(lr) * m32).astype(np.float32)).astype(np.float32)
    assert np.array_equal(param.cpu().numpy(), exp)


def test_payload_ops_64_match_reference_plugin(cuda, reference):
    need(reference)
    rng = np.random.default_rng(64)
    for trial in range(4):
        lanes = int(rng.integers(1, 2000))
        lim = (1 << 62) - 1
        a = rng.integers(-lim, lim, lanes, dtype=np.int64)
        b = rng.integers(-lim, lim, lanes, dtype=np.int64)
        ab, bb = a.view(np.uint8), b.view(np.uint8)
        want = reference.payload_combine(ab, bb, 0, 0, 64, 1, 2, 1, 0, 0, 0)
        pad = int(rng.integers(0, 5)) * 8
        da = torch.zeros(pad + ab.size + 8, dtype=torch.uint8, device=cuda)
        db = torch.zeros_like(da)
        da[pad:pad + ab.size] = dev(ab)
        db[pad:pad + ab.size] = dev(bb)
        G.IntSumOps(64).combine(da[pad:pad + ab.size], db[pad:pad + ab.size], 0, 0, 0, 0)
        G._sync_check(G._ErrWord.get(cuda))
        assert np.array_equal(da[pad:pad + ab.size].cpu().numpy(), want), trial


def test_int64_overflow_raises(cuda, reference):
    """IntSumOps width 64: __builtin_add_overflow -> overflow_error (collectives.cpp:74-76)."""
    a = np.array([(1 << 62), -5, (1 << 63) - 1], dtype=np.int64)
    b = np.array([(1 << 62), 3, 1], dtype=np.int64)
    if reference is not None:
        with pytest.raises(Exception):
            reference.payload_combine(a.view(np.uint8), b.view(np.uint8), 0, 0, 64, 1, 2, 1, 0, 0, 0)
    da, db = dev(a.view(np.uint8)), dev(b.view(np.uint8))
    G.IntSumOps(64).combine(da, db, 0, 0, 0, 0)
    with pytest.raises(LaneOverflow):
        G._sync_check(G._ErrWord.get(cuda))
    # the schedule replay flags it too (tree: worker 1 into worker 0)
    la = [dev(np.pad(a.view(np.uint8), (0, 8))), dev(np.pad(b.view(np.uint8), (0, 8)))]
    with pytest.raises(LaneOverflow):
        G.allreduce_inproc(la, 3, LevelKind.Standard, 64, 1)


def test_f64_decode_64(cuda, oracle, reference):
    """gq_dequant_f64 on int64 lanes: the reference's decode_dense_std doubles."""
    n, d, s = 3, 1001, 1 << 20
    rng = np.random.default_rng(1)
    v = rng.integers(-n * s, n * s, d, dtype=np.int64)
    lanes = dev(np.pad(v.view(np.uint8), (0, 8)))
    norm = 2.75
    out = torch.zeros(d, dtype=torch.float64, device=cuda)
    nt = torch.tensor([norm], dtype=torch.float64, device=cuda)
    err = G._ErrWord.get(cuda)
    G.check(G.lib().gq_dequant_f64(lanes.data_ptr(), 0, d, nt.data_ptr(), 0, s, n, 64, out.data_ptr(),
                                   err.data_ptr(), G._stream()))
    G._sync_check(err)
    scale = norm / (float(n) * s)
    assert np.array_equal(out.cpu().numpy(), scale * v.astype(np.float64))
