"""Known-answer tests of the device counter RNG (gq_rng_draws).

The hot loops never call the reference's bits() literally: quantize and the
token reduce hoist mix64^4(seed, stream, a, b) to the host and evaluate the
last mix64 in a group-shared form (gq_common.cuh elem_mix / token_kword). These
tests pin every form against the reference (rng.hpp:45-61 bits/u01,
exp_arith.cpp:43-50 sample_k and its KATs test_exp_arith.cpp:45-60), on random
keys and on the group-carry corner cases the shared form has to special-case.
"""
import numpy as np
import pytest
import torch

from paper_2305_18627_b200 import gqsgd as G

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1


def mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def prefix(seed, stream, a, b):
    h = mix64(seed ^ 0x517CC1B727220A95)
    h = mix64(h ^ stream)
    h = mix64(h ^ a)
    return mix64(h ^ b)


def draws(cuda, seed, stream, a, b, c0, count, m=8, bits_in=None):
    bits = torch.zeros(count, dtype=torch.int64, device=cuda)
    hi = torch.zeros(count, dtype=torch.int32, device=cuda)
    k = torch.zeros(count, dtype=torch.int32, device=cuda)
    bi = None
    if bits_in is not None:
        bi = torch.from_numpy(np.asarray(bits_in, dtype=np.uint64).view(np.int64)).to(cuda)
    G.check(G.lib().gq_rng_draws(seed, stream, a, b, c0, count, m, bi.data_ptr() if bi is not None else None,
                                 bits.data_ptr(), hi.data_ptr(), k.data_ptr(), G._stream()))
    torch.cuda.synchronize()
    return (bits.cpu().numpy().view(np.uint64), hi.cpu().numpy().view(np.uint32), k.cpu().numpy())


def oracle_or_reference(oracle, reference):
    return reference if reference is not None else oracle


def check_block(cuda, ref, seed, stream, a, b, c0, count, m):
    bits, hi, k = draws(cuda, seed, stream, a, b, c0, count, m)
    for i in range(count):
        c = (c0 + i) & M64
        want = ref.rng_bits(seed, stream, a, b, c)
        assert int(bits[i]) == want, (seed, stream, a, b, c)
        h = int(hi[i])
        assert (want >> 32) == h ^ (h >> 31), c           # H is the pre-xorshift high word
        assert (want >> 41) == h >> 9, c                  # the quantizer's 23 dither bits
        u = ref.u01(seed, stream, a, b, c)
        assert u == (want >> 11) * 2.0 ** -53
        assert int(k[i]) == ref.sample_k(u, m), (c, u, m)


@pytest.mark.parametrize("m", [1, 2, 5, 8, 32, 33, 100])
def test_random_keys_match_reference(cuda, oracle, reference, m):
    ref = oracle_or_reference(oracle, reference)
    rng = np.random.default_rng(m)
    for _ in range(6):
        seed, a, b = (int(x) for x in rng.integers(0, 1 << 63, 3))
        stream = int(rng.integers(0, 5))
        c0 = int(rng.integers(0, 1 << 62))
        check_block(cuda, ref, seed, stream, a, b, c0, 700, m)


def test_group_carry_corners(cuda, oracle, reference):
    """The quad-shared form shares the carry of the low-word add B = b + C0lo
    across a group of 4; groups whose add straddles 2^32 fall back to the
    generic hash. Walk c across every B in [2^32 - 64, 2^32 + 64)."""
    ref = oracle_or_reference(oracle, reference)
    for seed, stream, a, b in [(42, 1, 3, 7), (1, 2, 0, 123456789), (2**63 + 5, 2, 9, 2**40)]:
        p = prefix(seed, stream, a, b)
        plo = p & 0xFFFFFFFF
        for hiword in (0, 0x12345678):
            target_b = (2**32 - 0x7F4A7C15 - 64) & 0xFFFFFFFC
            c_lo = (target_b ^ (plo & ~3)) & 0xFFFFFFFC
            c0 = (hiword << 32) | c_lo
            check_block(cuda, ref, seed, stream, a, b, c0, 128 + 4, 8)
            check_block(cuda, ref, seed, stream, a, b, (c0 - 64) & M64, 64, 3)


def test_sample_k_kats_on_device_bits(cuda, reference, oracle):
    """test_exp_arith.cpp:45-60 through the device's bits -> k map
    (u = (bits >> 11) 2^-53, so bits = u 2^53 << 11 for dyadic-exact u)."""
    ref = oracle_or_reference(oracle, reference)
    m = 8

    def bits_of(u):  # the largest u01 value <= u (u01 values are multiples of 2^-53)
        return int(u * 2.0 ** 53) << 11

    cases = [(0.6, 1), (0.5, 1), (0.49999, 2), (0.2, 3), (2.0 ** -8, 8), (2.0 ** -9, 8), (0.0, 8)]
    for j in range(1, m):
        lo = 2.0 ** -j
        cases.append((lo, j))
        cases.append((np.nextafter(2.0 * lo, 0.0), j))
    bits = [bits_of(u) for u, _ in cases]
    _, _, k = draws(cuda, 0, 0, 0, 0, 0, len(bits), m, bits_in=bits)
    for (u, want), b, got in zip(cases, bits, k):
        ub = (b >> 11) * 2.0 ** -53  # == u except 0.49999, which is not a u01 value (same dyadic class)
        assert int(got) == want == ref.sample_k(ub, m) == ref.sample_k(u, m), (u, want, int(got))
    # the u == 0 tail and u just above 0 for a deep truncation
    _, _, k = draws(cuda, 0, 0, 0, 0, 0, 3, 100, bits_in=[0, 1 << 11, (1 << 11) - 1])
    assert [int(x) for x in k] == [100, 53, 100] == [ref.sample_k(0.0, 100), ref.sample_k(2.0 ** -53, 100),
                                                    ref.sample_k(0.0, 100)]
