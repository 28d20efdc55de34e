"""Pin the CPU oracle (oracle/gq_oracle.c) before trusting it.

1. The reference's own known-answer tests, transcribed case by case from
   /root/reference/proj/tests/test_{levels,quantizer,exp_arith,collectives,
   topology,algorithm}.cpp (file:line on each test).
2. The golden fixtures produced by the unmodified reference
   (tests/golden/make_golden.py -> golden.npz).
3. When oracle/_ref was built here, a randomized oracle-vs-reference sweep.
"""
import math

import numpy as np
import pytest

INF = 0xFFFFFFFF
STD, EXP = 0, 1


# --- test_levels.cpp -------------------------------------------------------
def test_standard_grid(oracle):  # test_levels.cpp:10-17
    assert list(oracle.levels(STD, 4)) == [1.0, 0.75, 0.5, 0.25, 0.0]


def test_exponential_grid(oracle):  # test_levels.cpp:19-24
    assert list(oracle.levels(EXP, 3)) == [1.0, 0.5, 0.25, 0.0]


def test_bracket_index(oracle):  # test_levels.cpp:37-44
    assert oracle.bracket_index(STD, 4, 1.0) == 0
    assert oracle.bracket_index(STD, 4, 0.0) == 3
    assert oracle.bracket_index(STD, 4, 0.5) == 2
    assert oracle.bracket_index(STD, 4, 0.6) == 1
    assert oracle.bracket_index(STD, 4, 0.1) == 3


def test_random_round_split(oracle):  # test_levels.cpp:46-52
    assert oracle.random_round(STD, 1, 0.5, 0.3) == 0
    assert oracle.random_round(STD, 1, 0.5, 0.5) == 1
    assert oracle.random_round(STD, 1, 0.0, 0.99) == 1
    assert oracle.random_round(STD, 1, 1.0, 0.99) == 0


@pytest.mark.parametrize("kind,s", [(STD, 5), (EXP, 6)])
def test_random_round_unbiased_split_points(oracle, kind, s):  # test_levels.cpp:54-73
    lv = oracle.levels(kind, s)
    for i in range(201):
        y = i / 200.0
        b = oracle.bracket_index(kind, s, y)
        hi, lo = lv[b], lv[b + 1]
        p_up = (y - lo) / (hi - lo)
        assert abs(p_up * hi + (1 - p_up) * lo - y) < 1e-15
        if 0.0 < p_up < 1.0:
            assert oracle.random_round(kind, s, y, p_up * (1.0 - 1e-12)) == b
            assert oracle.random_round(kind, s, y, p_up) == b + 1


# --- test_quantizer.cpp ----------------------------------------------------
def test_grid_points_quantize_deterministically(oracle):  # test_quantizer.cpp:11-24
    sign, idx = oracle.quantize(np.array([2.0, -1.5, 1.0, -0.5, 0.0]), 2.0, STD, 4, 3, 0, 0)
    assert list(idx) == [0, 1, 2, 3, 4]
    assert list(sign) == [1, -1, 1, -1, 1]


def test_zero_shard(oracle):  # test_quantizer.cpp:26-33
    sign, idx = oracle.quantize(np.zeros(4), 0.0, EXP, 3, 3, 1, 9)
    assert list(idx) == [3] * 4 and list(sign) == [1] * 4


def test_precondition_violations(oracle):  # test_quantizer.cpp:35-42
    from oracle.bind import OracleError
    with pytest.raises(OracleError) as e:
        oracle.quantize(np.array([1.0]), 0.0, STD, 2, 1, 0, 0)
    assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        oracle.quantize(np.array([3.0]), 2.0, STD, 2, 1, 0, 0)
    assert e.value.code == 1


def test_keys_reshuffle(oracle):  # test_quantizer.cpp:44-56
    x = np.sin(np.arange(64) + 1.0)
    a = oracle.quantize(x, 1.0, EXP, 5, 17, 2, 5)[1]
    b = oracle.quantize(x, 1.0, EXP, 5, 17, 2, 5)[1]
    c = oracle.quantize(x, 1.0, EXP, 5, 17, 2, 6)[1]
    d = oracle.quantize(x, 1.0, EXP, 5, 17, 3, 5)[1]
    assert np.array_equal(a, b) and not np.array_equal(a, c) and not np.array_equal(a, d)


# --- test_exp_arith.cpp ----------------------------------------------------
def test_ceil_log2_and_prescale(oracle):  # test_exp_arith.cpp:12-26
    assert [oracle.ceil_log2(v) for v in (1, 2, 3, 16, 17, 1 << 40)] == [0, 1, 2, 4, 5, 40]
    assert [oracle.prescale_shift(n) for n in (2, 3, 16, 17)] == [2, 3, 5, 6]


def test_check_width_worked_cases(oracle):  # test_exp_arith.cpp:28-43
    assert oracle.check_width(EXP, 3, 16, 4)
    assert not oracle.check_width(EXP, 4, 16, 4)
    assert not any(oracle.check_width(STD, s, 16, 4) for s in range(1, 65))
    assert oracle.check_width(STD, 7, 16, 8)
    assert not oracle.check_width(STD, 8, 16, 8)
    assert not oracle.check_width(STD, 255, 16, 8)
    assert oracle.check_width(EXP, 123, 16, 8)
    assert not oracle.check_width(EXP, 124, 16, 8)


def test_sample_k_dyadic(oracle):  # test_exp_arith.cpp:45-60
    m = 8
    assert oracle.sample_k(0.6, m) == 1
    assert oracle.sample_k(0.5, m) == 1
    assert oracle.sample_k(0.49999, m) == 2
    assert oracle.sample_k(0.2, m) == 3
    assert oracle.sample_k(2.0 ** -8, m) == 8
    assert oracle.sample_k(2.0 ** -9, m) == 8
    assert oracle.sample_k(0.0, m) == 8
    for j in range(1, m):
        lo = 2.0 ** -j
        assert oracle.sample_k(lo, m) == j
        assert oracle.sample_k(np.nextafter(2.0 * lo, 0.0), m) == j


def _scaled(t):
    return 0 if t[1] == 0 else t[0] * (1 << (20 - t[1]))


def _expect(oracle, a, b, m, max_e):
    acc = 0
    for j in range(1, m + 1):
        pj = (1 << (m - j)) if j < m else 2
        acc += pj * _scaled(oracle.reduce_pair(a, b, j, max_e))
    return acc


def test_reduce_pair_worked_examples(oracle):  # test_exp_arith.cpp:124-142
    m, max_e = 8, 127  # ReduceContext::make(7, 16, 8)
    assert _expect(oracle, (1, 2), (1, 4), m, max_e) == (5 << 16) << m
    assert _expect(oracle, (1, 2), (-1, 4), m, max_e) == (3 << 16) << m
    assert oracle.reduce_pair((1, 3), (1, 3), 1, max_e) == (1, 2)
    assert oracle.reduce_pair((-1, 3), (-1, 3), 5, max_e) == (-1, 2)
    assert oracle.reduce_pair((1, 0), (-1, 6), 1, max_e) == (-1, 6)
    assert oracle.reduce_pair((-1, 6), (1, 0), 3, max_e) == (-1, 6)
    assert oracle.reduce_pair((1, 0), (1, 0), 2, max_e) == (1, 0)
    assert oracle.reduce_pair((1, 4), (-1, 4), 1, max_e) == (1, 0)


def test_reduce_pair_exactly_unbiased(oracle):  # test_exp_arith.cpp:144-164
    m, max_e = 8, 32767  # ReduceContext::make(7, 16, 16)
    for e1 in range(1, 13):
        for e2 in range(1, 13):
            if abs(e1 - e2) > m - 1:
                continue
            for s1 in (1, -1):
                for s2 in (1, -1):
                    if s1 == s2 and (e1 == 1 or e2 == 1):
                        continue
                    want = (_scaled((s1, e1)) + _scaled((s2, e2))) * (1 << m)
                    assert _expect(oracle, (s1, e1), (s2, e2), m, max_e) == want


def test_reduce_pair_guard(oracle):  # test_exp_arith.cpp:179-186
    from oracle.bind import OracleError
    with pytest.raises(OracleError) as e:
        oracle.reduce_pair((1, 1), (1, 1), 1, 127)
    assert e.value.code == 2


def test_token_lanes_pack(oracle):  # test_exp_arith.cpp:188-222
    # shift = 3 for n = 4 (ReduceContext::make(3, 4, 8)); idx {0, 2, 3} -> e {3, 5, 0}
    lanes = oracle.encode(EXP, 3, 4, 8, np.array([1, -1, 1], np.int8), np.array([0, 2, 3], np.uint32))
    assert list(lanes) == [0x03, 0x85, 0x00]
    # frozen bytes 0x7f, 0x85, 0x00 for tokens (+,127), (-,5), zero (n=1: shift 1)
    lanes = oracle.encode(EXP, 127, 1, 8, np.array([1, -1, 1], np.int8),
                          np.array([126, 4, 127], np.uint32))
    assert list(lanes) == [0x7f, 0x85, 0x00]


# --- test_collectives.cpp --------------------------------------------------
def test_int8_lane_sums(oracle):  # test_collectives.cpp:53-66
    from oracle.bind import OracleError
    lanes = np.array([[0xff, 0x05, 0x7e], [0xff, 0xfb, 0x01]], dtype=np.uint8)
    out = oracle.allreduce_inproc(lanes, 3, STD, 8, 1, 0, 0, 0)
    assert list(out[0]) == [0xfe, 0x00, 0x7f]
    with pytest.raises(OracleError) as e:
        oracle.allreduce_inproc(np.array([[0x7f], [0x01]], np.uint8), 1, STD, 8, 1, 0, 0, 0)
    assert e.value.code == 2
    with pytest.raises(OracleError):
        oracle.allreduce_inproc(np.array([[0x80], [0xff]], np.uint8), 1, STD, 8, 1, 0, 0, 0)


def test_token_lane_golden_bytes(oracle):  # test_collectives.cpp:109-118
    lanes = np.array([[0x03, 0x83, 0x00, 0x05, 0x05], [0x03, 0x83, 0x05, 0x00, 0x85]], np.uint8)
    out = oracle.allreduce_inproc(lanes, 5, EXP, 8, 7, 0, 99, 0)  # n=2 tree: one event
    assert list(out[0]) == [0x02, 0x82, 0x05, 0x05, 0x00]


def test_exact_sums_tree_and_ring(oracle):  # test_collectives.cpp:135-170
    shards = np.array([[1, -2, 3, -4, 5, -6], [10, 20, 30, 40, 50, 60],
                       [-7, -7, -7, -7, -7, -7], [100, 0, -100, 0, 100, 0]], dtype=np.int16)
    want = shards.sum(axis=0).astype(np.int16)
    for topo in (0, 1):
        out = oracle.allreduce_inproc(shards.view(np.uint8), 6, STD, 16, 1, topo, 0, 1)
        for r in range(4):
            assert np.array_equal(out[r].view(np.int16), want)


def test_norm_exchange_kat(oracle):  # test_collectives.cpp:199-213
    stats = [9.0, 16.0, 0.25, 144.0]
    assert math.isclose(oracle.norm_tree_combine(stats, 2, 2), 13.009611831257688, rel_tol=1e-12)
    assert oracle.norm_tree_combine(stats, INF, INF) == 144.0


# --- test_topology.cpp -----------------------------------------------------
def test_tree5_events(oracle):  # test_topology.cpp:76-97
    want = [(0, 1, 0, 0, 0), (0, 3, 2, 0, 0), (1, 2, 0, 0, 0), (2, 4, 0, 0, 0),
            (3, 0, 4, 1, 0), (4, 0, 2, 1, 0), (5, 0, 1, 1, 0), (5, 2, 3, 1, 0)]
    assert oracle.schedule(0, 5) == want


def test_ring3_events(oracle):  # test_topology.cpp:125-146
    rs = [(0, 0, 1, 0, 0), (0, 1, 2, 0, 1), (0, 2, 0, 0, 2),
          (1, 0, 1, 0, 2), (1, 1, 2, 0, 0), (1, 2, 0, 0, 1)]
    ev = oracle.schedule(1, 3)
    assert ev[:6] == rs and all(e[3] == 1 for e in ev[6:]) and len(ev) == 12


# --- test_algorithm.cpp ----------------------------------------------------
def test_standard_lane_widths(oracle):  # test_algorithm.cpp:53-63
    assert oracle.standard_lane_width(7, 8, 8) == 8
    assert oracle.standard_lane_width(15, 8, 8) == 8
    assert oracle.standard_lane_width(15, 9, 8) == 16
    assert oracle.standard_lane_width(7, 255, 8) == 16
    assert oracle.standard_lane_width(255, 255, 8) == 32
    assert oracle.standard_lane_width(1, 2, 32) == 32
    assert oracle.standard_lane_width(255, 1 << 24, 8) is None


def test_zero_shards_short_circuit(oracle, golden):  # test_algorithm.cpp:65-77
    mean, norm, lw, _ = oracle.mean(np.zeros((3, 5)), EXP, 7)
    assert norm == 0.0 and np.all(mean == 0.0)


# --- golden fixtures from the unmodified reference --------------------------
def test_rng_bits_golden(oracle, golden):
    data, _ = golden
    for k, want in zip(data["kat/rng_keys"], data["kat/rng_bits"]):
        assert oracle.rng_bits(*[int(v) for v in k]) == int(want)


def test_reduce_pair_golden_table(oracle, golden):
    data, _ = golden
    from oracle.bind import OracleError
    for s1, e1, s2, e2, k, so, eo, err in data["kat/reduce_pair"]:
        if err:
            with pytest.raises(OracleError):
                oracle.reduce_pair((int(s1), int(e1)), (int(s2), int(e2)), int(k), 32767)
        else:
            assert oracle.reduce_pair((int(s1), int(e1)), (int(s2), int(e2)), int(k), 32767) == (so, eo)


def test_oracle_matches_golden_configs(oracle, golden):
    data, meta = golden
    for name, m in meta.items():
        x = data[f"{name}/x"].astype(np.float64)
        mean, norm, lw, summed = oracle.mean(x, m["kind"], m["s"], m["q"], m["p"], m["width"],
                                             m["topo"], m["seed"], m["round"])
        assert lw == m["lane_width"], name
        assert np.array_equal(mean, data[f"{name}/mean"]), name
        if m["q"] == INF:
            assert norm == m["norm"], name
        else:
            assert math.isclose(norm, m["norm"], rel_tol=1e-12), name
        if f"{name}/summed" in data:
            assert np.array_equal(summed, data[f"{name}/summed"]), name
            for r in range(m["n"]):
                sign, idx = oracle.quantize(x[r], m["norm"], m["kind"], m["s"], m["seed"], r, m["round"])
                lanes = oracle.encode(m["kind"], m["s"], m["n"], lw, sign, idx)
                assert np.array_equal(lanes, data[f"{name}/lanes"][r]), (name, r)


def test_gaussian_shards_match_reference(oracle, reference):
    if reference is None:
        pytest.skip("oracle/_ref not built")
    assert np.array_equal(oracle.gaussian_shards(3, 2000, 12345), reference.gaussian_shards(3, 2000, 12345))


def test_oracle_vs_reference_sweep(oracle, reference):
    """Randomized configs (incl. ragged d, ring, L2, 16-bit) vs the reference."""
    if reference is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(0)
    for trial in range(40):
        kind = int(rng.integers(0, 2))
        n = int(rng.integers(1, 10))
        d = int(rng.integers(1, 700))
        topo = int(rng.integers(0, 2))
        width = int(rng.choice([8, 16]))
        s = int(rng.integers(1, 20)) if kind == STD else int(rng.integers(1, 9))
        q, p = [(INF, INF), (2, 2), (INF, 2), (2, INF)][int(rng.integers(0, 4))]
        seed, rnd = int(rng.integers(0, 1 << 62)), int(rng.integers(0, 1000))
        x = reference.gaussian_shards(n, d, 100 + trial).astype(np.float32).astype(np.float64)
        try:
            want = reference.mean(x, kind, s, q, p, width, topo, seed, rnd)
        except Exception as e:
            from oracle.bind import OracleError
            with pytest.raises(OracleError):
                oracle.mean(x, kind, s, q, p, width, topo, seed, rnd)
            continue
        got = oracle.mean(x, kind, s, q, p, width, topo, seed, rnd)
        assert got[2] == want[2]
        if q == INF:
            assert got[1] == want[1]
            assert np.array_equal(got[0], want[0]), (trial, kind, n, d, topo, width, s)


def test_four_bit_equals_eight_bit(oracle):
    """Extension: 4-bit lanes hold the same values as the reference's 8-bit run."""
    x = oracle.gaussian_shards(8, 1001, 12345).astype(np.float32).astype(np.float64)
    m8, n8, w8, s8 = oracle.mean(x, EXP, 4, width=8, seed=42)
    m4, n4, w4, s4 = oracle.mean(x, EXP, 4, width=4, seed=42)
    assert (w8, w4) == (8, 4) and np.array_equal(m8, m4)
    nib = np.zeros(1001, np.uint8)
    nib[0::2] = s4[: (1001 + 1) // 2] & 0xF
    nib[1::2] = s4[: 1001 // 2] >> 4
    tok8 = s8.astype(np.uint8)
    assert np.array_equal((tok8 & 0x7) | ((tok8 >> 7) << 3), nib)


def test_gaussian_range_is_a_column_slice_of_gaussian_shards(oracle, reference, fingerprints):
    """The large fixtures' inputs: columns [j0, j0+cnt) of gaussian_shards
    (verify.cpp:118-128), from the C oracle and the reference shim alike."""
    full = oracle.gaussian_shards(3, 5000, 12345)
    part = oracle.gaussian_range(3, 1234, 2000, 12345)
    assert np.array_equal(full[:, 1234:3234], part)
    if reference is not None:
        assert np.array_equal(reference.gaussian_range(3, 1234, 2000, 12345), part)
        assert np.array_equal(reference.gaussian_shards(3, 5000, 12345), full)
    f = fingerprints["C4_std_s15_n8_bucket51"]
    x = oracle.gaussian_range(f["n"], f["j0"], f["d"], f["data_seed"]).astype(np.float32)
    import hashlib
    assert hashlib.sha256(x.tobytes()).hexdigest() == f["x_sha"]
