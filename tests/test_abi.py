"""CPU-side checks of the C-ABI library (no GPU needed).

- libgq_b200.so loads and exports exactly the entry points include/gq_b200.h
  declares;
- the host-only admission logic (gq_plan_path, gq_lane_bytes) matches the
  reference's plan_path / standard_lane_width / ReduceContext::make cases
  (test_algorithm.cpp:53-63, test_exp_arith.cpp:28-43,91-101) and the oracle.
"""
import re
import subprocess
from pathlib import Path

import pytest

from paper_2305_18627_b200 import _lib
from paper_2305_18627_b200.gqsgd import (GqsgdConfig, InvalidArgument, LevelKind, NormSpec,
                                         check_width, lane_bytes, plan_path, prescale_shift,
                                         standard_lane_width)

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "gq_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\S[^;(]*?\b(gq_\w+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 13
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (gq_\w+)$", out, flags=re.M))
    assert set(syms) == exported
    assert set(_lib.SIGNATURES) == exported
    L = _lib.lib()
    for s in syms:
        assert getattr(L, s) is not None


def test_no_cuda_runtime_dependency_on_path():
    out = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "libcudart" not in out  # cudart is linked statically; only the driver is needed


@pytest.mark.parametrize("s,n,at_least,want", [
    (7, 8, 8, 8), (15, 8, 8, 8), (15, 9, 8, 16), (7, 255, 8, 16), (255, 255, 8, 32),
    (1, 2, 32, 32), (255, 1 << 24, 8, None),
    # extension: packed 4-bit standard lanes when n(s+1) <= 8
    (3, 2, 4, 4), (1, 4, 4, 4), (1, 8, 4, 8),
])
def test_standard_lane_width(s, n, at_least, want):
    if n > _lib.GQ_MAX_WORKERS:
        with pytest.raises(InvalidArgument):
            plan_path(GqsgdConfig(workers=n, scheme=LevelKind.Standard, s=s, width_bits=at_least))
        return
    assert standard_lane_width(s, n, at_least) == want


def test_exponential_admission():
    p = plan_path(GqsgdConfig(workers=16, scheme=LevelKind.Exponential, s=7, width_bits=8))
    assert (p.lane_width, p.m, p.shift, p.max_e) == (8, 8, 5, 127)
    with pytest.raises(InvalidArgument, match="refused configuration"):
        plan_path(GqsgdConfig(workers=16, scheme=LevelKind.Exponential, s=124, width_bits=8))
    with pytest.raises(InvalidArgument):
        plan_path(GqsgdConfig(workers=16, scheme=LevelKind.Exponential, s=7, width_bits=12))
    # C2: 4-bit packed at n=8 admits s <= 4
    assert plan_path(GqsgdConfig(workers=8, scheme=LevelKind.Exponential, s=4, width_bits=4)).lane_width == 4
    with pytest.raises(InvalidArgument):
        plan_path(GqsgdConfig(workers=8, scheme=LevelKind.Exponential, s=5, width_bits=4))
    # 2-bit is refused for every n >= 2 (exp_arith.cpp:27-36)
    with pytest.raises(InvalidArgument):
        plan_path(GqsgdConfig(workers=2, scheme=LevelKind.Exponential, s=1, width_bits=2))


def test_config_errors():
    with pytest.raises(InvalidArgument):
        plan_path(GqsgdConfig(workers=0))
    with pytest.raises(InvalidArgument):
        plan_path(GqsgdConfig(s=0))
    # orders 1..16 besides inf (norm_spec_from_string, norms.cpp:17-30); 0 and 17 refused
    assert plan_path(GqsgdConfig(norm=NormSpec(3, 3))).lane_width == 8
    for bad in ((0, 2), (17, 2), (2, 0), (2, 17)):
        with pytest.raises(InvalidArgument):
            plan_path(GqsgdConfig(norm=NormSpec(*bad)))
    with pytest.raises(InvalidArgument):
        plan_path(GqsgdConfig(sparse=True))


def test_admission_agrees_with_oracle(oracle):
    for kind in (0, 1):
        for n in (1, 2, 3, 4, 8, 16, 100):
            for s in (1, 2, 3, 4, 5, 7, 15, 31, 63, 124, 127, 1000):
                for w in (4, 8, 16, 32):
                    assert check_width(LevelKind(kind), s, n, w) == oracle.check_width(kind, s, n, w)
                    cfg = GqsgdConfig(workers=n, scheme=LevelKind(kind), s=s, width_bits=w)
                    if kind == 0:
                        assert standard_lane_width(s, n, w) == oracle.standard_lane_width(s, n, w)
                    else:
                        if oracle.check_width(kind, s, n, w):
                            assert plan_path(cfg).lane_width == w
                            assert plan_path(cfg).shift == prescale_shift(n) == oracle.prescale_shift(n)
                        else:
                            with pytest.raises(InvalidArgument):
                                plan_path(cfg)


def test_lane_bytes_padding():
    assert lane_bytes(0, 8) == 0
    assert lane_bytes(1, 8) == 16
    assert lane_bytes(33, 4) == 32
    assert lane_bytes(1 << 24, 4) == 1 << 23
    assert lane_bytes(1000, 16) % 16 == 0 and lane_bytes(1000, 16) >= 2000


def test_communicator_argument_checks():
    """gq_comm_* reject bad configurations on the host, before touching a GPU
    (status GQ_ERR_INVALID, the reference's invalid_argument class)."""
    import ctypes as C

    from paper_2305_18627_b200 import _lib
    from paper_2305_18627_b200.gqsgd import GqsgdConfig, LevelKind

    L = _lib.lib()
    assert L.gq_comm_handle_bytes() >= 64
    cfg = GqsgdConfig(workers=4, scheme=LevelKind.Standard, s=15, width_bits=8).to_c()
    out = C.c_void_p()
    for rank, nranks, d in [(0, 0, 100), (2, 2, 100), (0, 17, 100), (0, 3, 100), (0, 2, 0)]:
        assert L.gq_comm_init(rank, nranks, C.byref(cfg), d, C.byref(out)) == _lib.GQ_ERR_INVALID
        assert out.value is None
    bad = GqsgdConfig(workers=16, scheme=LevelKind.Exponential, s=124, width_bits=8).to_c()  # refused width
    assert L.gq_comm_init(0, 2, C.byref(bad), 100, C.byref(out)) == _lib.GQ_ERR_INVALID
    assert b"refused" in L.gq_last_error()
    for fn in (L.gq_comm_quantize, ):
        assert fn(None, None, 0, None, 0, None, None) == _lib.GQ_ERR_INVALID
    assert L.gq_allreduce_lanes(None, None, 0, None, None, None) == _lib.GQ_ERR_INVALID
    assert L.gq_sync(None, None, None) == _lib.GQ_ERR_INVALID
    assert L.gq_comm_connect(None, None) == _lib.GQ_ERR_INVALID
    assert L.gq_comm_destroy(None) == _lib.GQ_OK
    assert L.gq_comm_summed(None) is None


def test_comm_timeout_option_range():
    from paper_2305_18627_b200 import _lib
    L = _lib.lib()
    assert L.gq_set_option(_lib.GQ_OPT_COMM_TIMEOUT_S, 0) == _lib.GQ_ERR_INVALID
    assert L.gq_set_option(_lib.GQ_OPT_COMM_TIMEOUT_S, 86401) == _lib.GQ_ERR_INVALID
    assert L.gq_set_option(_lib.GQ_OPT_COMM_TIMEOUT_S, 600) == _lib.GQ_OK
    assert L.gq_set_option(_lib.GQ_OPT_COMM_TIMEOUT_S, 60) == _lib.GQ_OK
