"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

  Oracle     the plain-C restatement (oracle/gq_oracle.c -> _build/libgq_oracle.so)
  Reference  the unmodified reference compiled here (oracle/_ref/libgqsgd_ref.so),
             present when /root/reference was available at build time

Status codes: 0 ok, 1 invalid_argument, 2 overflow_error, 3 domain_error.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libgq_oracle.so"
REF_SO = HERE / "_ref" / "libgqsgd_ref.so"
NORM_INF = 0xFFFFFFFF

_u32, _u64, _i32, _i64, _vp, _d = C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_void_p, C.c_double


class OracleError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def build_oracle(force: bool = False) -> Path:
    if force or not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < (HERE / "gq_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    return ORACLE_SO


def build_reference() -> Path | None:
    """The unmodified reference (oracle/_ref/libgqsgd_ref.so) and the drop-in
    builds against it (integration/Makefile: dropin_check, acceptance_b200)."""
    if Path("/root/reference/proj/src").exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)
        subprocess.run(["make", "-s", "-j8", "-C", str(HERE.parent / "integration")], check=True)
    return REF_SO if REF_SO.exists() else None


def lane_payload_bytes(d: int, width: int) -> int:
    return (d * width + 7) // 8


class Oracle:
    """The C restatement."""

    def __init__(self, path: Path | None = None):
        path = path or build_oracle()
        L = C.CDLL(str(path))
        sig = {
            "gqo_mix64": (_u64, [_u64]),
            "gqo_rng_bits": (_u64, [_u64] * 5),
            "gqo_rng_u01": (_d, [_u64] * 5),
            "gqo_levels": (_i32, [_u32, _u32, _vp]),
            "gqo_bracket_index": (_u32, [_vp, _u32, _d]),
            "gqo_random_round": (_u32, [_vp, _u32, _d, _d]),
            "gqo_ceil_log2": (_u32, [_u64]),
            "gqo_prescale_shift": (_u32, [_u32]),
            "gqo_check_width": (_i32, [_u32, _u32, _u32, _u32]),
            "gqo_standard_lane_width": (_u32, [_u32, _u32, _u32]),
            "gqo_sample_k": (_u32, [_d, _u32]),
            "gqo_reduce_pair": (_i32, [_i32, _u32, _i32, _u32, _u32, _u32, _vp, _vp]),
            "gqo_local_norm_stat": (_i32, [_vp, _u64, _u32, _u32, _vp]),
            "gqo_norm_tree_combine": (_i32, [_vp, _u32, _u32, _u32, _vp]),
            "gqo_quantize": (_i32, [_vp, _u64, _d, _u32, _u32, _u64, _u32, _u64, _vp, _vp]),
            "gqo_encode": (_i32, [_u32, _u32, _u32, _u32, _vp, _vp, _u64, _vp]),
            "gqo_schedule": (_i64, [_u32, _u32, _vp, _u64]),
            "gqo_allreduce_inproc": (_i32, [_vp, _u32, _u64, _u32, _u32, _u32, _u32, _u64, _u64]),
            "gqo_decode": (_i32, [_u32, _vp, _u64, _d, _u32, _u32, _u32, _vp]),
            "gqo_mean": (_i32, [_vp, _u32, _u64, _u32, _u32, _u32, _u32, _u32, _u32, _u64, _u64,
                                _vp, _vp, _vp, _vp, _vp]),
            "gqo_gaussian_shards": (_i32, [_u32, _u64, _u64, _vp]),
            "gqo_gaussian_range": (_i32, [_u32, _u64, _u64, _u64, _vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        self.L = L

    @staticmethod
    def _ok(rc: int) -> None:
        if rc != 0:
            raise OracleError(rc)

    def rng_bits(self, seed, stream, a, b, c) -> int:
        return self.L.gqo_rng_bits(seed, stream, a, b, c)

    def u01(self, seed, stream, a, b, c) -> float:
        return self.L.gqo_rng_u01(seed, stream, a, b, c)

    def levels(self, kind: int, s: int) -> np.ndarray:
        out = np.zeros(s + 1)
        self._ok(self.L.gqo_levels(kind, s, _p(out)))
        return out

    def bracket_index(self, kind, s, y) -> int:
        lv = self.levels(kind, s)
        return self.L.gqo_bracket_index(_p(lv), s, y)

    def random_round(self, kind, s, y, u) -> int:
        lv = self.levels(kind, s)
        return self.L.gqo_random_round(_p(lv), s, y, u)

    def ceil_log2(self, v) -> int:
        return self.L.gqo_ceil_log2(v)

    def prescale_shift(self, n) -> int:
        return self.L.gqo_prescale_shift(n)

    def check_width(self, kind, s, n, w) -> bool:
        return bool(self.L.gqo_check_width(kind, s, n, w))

    def standard_lane_width(self, s, n, at_least) -> int | None:
        w = self.L.gqo_standard_lane_width(s, n, at_least)
        return w or None

    def sample_k(self, u, m) -> int:
        return self.L.gqo_sample_k(u, m)

    def reduce_pair(self, a, b, k, max_e):
        so, eo = C.c_int32(), C.c_uint32()
        self._ok(self.L.gqo_reduce_pair(a[0], a[1], b[0], b[1], k, max_e, C.byref(so), C.byref(eo)))
        return (so.value, eo.value)

    def gaussian_shards(self, n: int, d: int, seed: int) -> np.ndarray:
        out = np.zeros((n, d))
        self._ok(self.L.gqo_gaussian_shards(n, d, seed, _p(out)))
        return out

    def gaussian_range(self, n: int, j0: int, cnt: int, seed: int) -> np.ndarray:
        """Columns [j0, j0+cnt) of gaussian_shards(n, d, seed), any d >= j0+cnt."""
        out = np.zeros((n, cnt))
        self._ok(self.L.gqo_gaussian_range(n, j0, cnt, seed, _p(out)))
        return out

    def local_norm_stat(self, x: np.ndarray, q=NORM_INF, p=NORM_INF) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = C.c_double()
        self._ok(self.L.gqo_local_norm_stat(_p(x), x.size, q, p, C.byref(out)))
        return out.value

    def norm_tree_combine(self, stats, q=NORM_INF, p=NORM_INF) -> float:
        st = np.ascontiguousarray(stats, dtype=np.float64)
        out = C.c_double()
        self._ok(self.L.gqo_norm_tree_combine(_p(st), st.size, q, p, C.byref(out)))
        return out.value

    def quantize(self, x, norm, kind, s, seed, worker, round):
        x = np.ascontiguousarray(x, dtype=np.float64)
        sign = np.zeros(x.size, dtype=np.int8)
        idx = np.zeros(x.size, dtype=np.uint32)
        self._ok(self.L.gqo_quantize(_p(x), x.size, norm, kind, s, seed, worker, round, _p(sign), _p(idx)))
        return sign, idx

    def encode(self, kind, s, n, width, sign, idx) -> np.ndarray:
        out = np.zeros(lane_payload_bytes(sign.size, width), dtype=np.uint8)
        self._ok(self.L.gqo_encode(kind, s, n, width, _p(sign), _p(idx), sign.size, _p(out)))
        return out

    def schedule(self, topo, n) -> list[tuple]:
        cap = 4 * n * n + 16
        buf = np.zeros(5 * cap, dtype=np.uint32)
        cnt = self.L.gqo_schedule(topo, n, _p(buf), cap)
        return [tuple(int(v) for v in buf[5 * i:5 * i + 5]) for i in range(cnt)]

    def allreduce_inproc(self, lanes: np.ndarray, d, kind, width, s, topo, seed, round) -> np.ndarray:
        lanes = np.ascontiguousarray(lanes, dtype=np.uint8).copy()
        n = lanes.shape[0]
        self._ok(self.L.gqo_allreduce_inproc(_p(lanes), n, d, kind, width, s, topo, seed, round))
        return lanes

    def decode(self, kind, lanes, d, norm, s, n, width) -> np.ndarray:
        lanes = np.ascontiguousarray(lanes, dtype=np.uint8)
        out = np.zeros(d)
        self._ok(self.L.gqo_decode(kind, _p(lanes), d, norm, s, n, width, _p(out)))
        return out

    def mean(self, shards, kind, s, q=NORM_INF, p=NORM_INF, width=8, topo=0, seed=1, round=0,
             norm_override: float | None = None):
        sh = np.ascontiguousarray(shards, dtype=np.float64)
        n, d = sh.shape
        mean = np.zeros(d)
        norm = C.c_double()
        lw = C.c_uint32()
        nov = C.c_double(norm_override) if norm_override is not None else None
        # summed lanes sized for the widest lane the plan may pick
        summed = np.zeros(lane_payload_bytes(d, 64) + 8, dtype=np.uint8)
        self._ok(self.L.gqo_mean(_p(sh), n, d, kind, s, q, p, width, topo, seed, round,
                                 C.byref(nov) if nov is not None else None, _p(mean),
                                 C.byref(norm), C.byref(lw), _p(summed)))
        return mean, norm.value, lw.value, summed[:lane_payload_bytes(d, lw.value)]


class Reference:
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self, path: Path | None = None):
        path = path or REF_SO
        if not Path(path).exists():
            raise FileNotFoundError(path)
        L = C.CDLL(str(path))
        sig = {
            "gqr_last_error": (C.c_char_p, []),
            "gqr_rng_bits": (_u64, [_u64] * 5),
            "gqr_rng_u01": (_d, [_u64] * 5),
            "gqr_gaussian_shards": (_i32, [_u32, _u64, _u64, _vp]),
            "gqr_gaussian_range": (_i32, [_u32, _u64, _u64, _u64, _vp]),
            "gqr_levels": (_i32, [_u32, _u32, _vp]),
            "gqr_bracket_index": (_i32, [_u32, _u32, _d, _vp]),
            "gqr_random_round": (_i32, [_u32, _u32, _d, _d, _vp]),
            "gqr_local_norm_stat": (_i32, [_vp, _u64, _u32, _u32, _vp]),
            "gqr_combine_norm_stats": (_i32, [_vp, _u32, _u32, _u32, _vp]),
            "gqr_norm_allreduce_inproc": (_i32, [_vp, _u32, _u32, _u32, _u64, _vp]),
            "gqr_quantize_shard": (_i32, [_vp, _u64, _d, _u32, _u32, _u64, _u32, _u64, _vp, _vp]),
            "gqr_check_width": (_i32, [_u32, _u32, _u32, _u32]),
            "gqr_standard_lane_width": (_u32, [_u32, _u32, _u32]),
            "gqr_sample_k": (_i32, [_d, _u32, _vp]),
            "gqr_reduce_pair": (_i32, [_i32, _u32, _i32, _u32, _u32, _u32, _u32, _u32, _vp, _vp]),
            "gqr_encode": (_i32, [_u32, _u32, _u32, _u32, _vp, _vp, _u64, _vp]),
            "gqr_allreduce_inproc": (_i32, [_vp, _u32, _u64, _u32, _u32, _u32, _u32, _u64, _u64, _vp]),
            "gqr_gqsgd_mean": (_i32, [_vp, _u32, _u64, _u32, _u32, _u32, _u32, _u32, _u32, _u32, _u64,
                                      _u64, _vp, _vp, _vp, _vp]),
            "gqr_baseline_mean": (_i32, [_vp, _u32, _u64, _u32, _u32, _u64, _vp]),
            "gqr_schedule": (_i64, [_u32, _u32, _vp, _u64]),
            "gqr_sparse_payload": (_i32, [_vp, _u64, _d, _u32, _u32, _u64, _u32, _u64, _u32, _vp, _u64, _vp]),
            "gqr_gqsgd_mean_sparse": (_i32, [_vp, _u32, _u64, _u32, _u32, _u32, _u32, _u32, _u32, _u64, _u64,
                                             _vp, _vp, _vp]),
            "gqr_payload_combine": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _u32, _u64, _u64, _u32, _u32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        self.L = L

    def _ok(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(rc, self.L.gqr_last_error().decode())

    def rng_bits(self, seed, stream, a, b, c) -> int:
        return self.L.gqr_rng_bits(seed, stream, a, b, c)

    def u01(self, seed, stream, a, b, c) -> float:
        return self.L.gqr_rng_u01(seed, stream, a, b, c)

    def gaussian_shards(self, n: int, d: int, seed: int) -> np.ndarray:
        out = np.zeros((n, d))
        self._ok(self.L.gqr_gaussian_shards(n, d, seed, _p(out)))
        return out

    def gaussian_range(self, n: int, j0: int, cnt: int, seed: int) -> np.ndarray:
        out = np.zeros((n, cnt))
        self._ok(self.L.gqr_gaussian_range(n, j0, cnt, seed, _p(out)))
        return out

    def levels(self, kind, s) -> np.ndarray:
        out = np.zeros(s + 1)
        self._ok(self.L.gqr_levels(kind, s, _p(out)))
        return out

    def bracket_index(self, kind, s, y) -> int:
        out = C.c_uint32()
        self._ok(self.L.gqr_bracket_index(kind, s, y, C.byref(out)))
        return out.value

    def random_round(self, kind, s, y, u) -> int:
        out = C.c_uint32()
        self._ok(self.L.gqr_random_round(kind, s, y, u, C.byref(out)))
        return out.value

    def local_norm_stat(self, x, q=NORM_INF, p=NORM_INF) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = C.c_double()
        self._ok(self.L.gqr_local_norm_stat(_p(x), x.size, q, p, C.byref(out)))
        return out.value

    def norm_allreduce_inproc(self, stats, q=NORM_INF, p=NORM_INF, round=0) -> float:
        st = np.ascontiguousarray(stats, dtype=np.float64)
        out = C.c_double()
        self._ok(self.L.gqr_norm_allreduce_inproc(_p(st), st.size, q, p, round, C.byref(out)))
        return out.value

    def quantize(self, x, norm, kind, s, seed, worker, round):
        x = np.ascontiguousarray(x, dtype=np.float64)
        sign = np.zeros(x.size, dtype=np.int8)
        idx = np.zeros(x.size, dtype=np.uint32)
        self._ok(self.L.gqr_quantize_shard(_p(x), x.size, norm, kind, s, seed, worker, round,
                                           _p(sign), _p(idx)))
        return sign, idx

    def check_width(self, kind, s, n, w) -> bool:
        return bool(self.L.gqr_check_width(kind, s, n, w))

    def standard_lane_width(self, s, n, at_least) -> int | None:
        return self.L.gqr_standard_lane_width(s, n, at_least) or None

    def sample_k(self, u, m) -> int:
        out = C.c_uint32()
        self._ok(self.L.gqr_sample_k(u, m, C.byref(out)))
        return out.value

    def reduce_pair(self, a, b, k, s, n, width):
        so, eo = C.c_int32(), C.c_uint32()
        self._ok(self.L.gqr_reduce_pair(a[0], a[1], b[0], b[1], k, s, n, width, C.byref(so), C.byref(eo)))
        return (so.value, eo.value)

    def encode(self, kind, s, n, width, sign, idx) -> np.ndarray:
        out = np.zeros(sign.size * width // 8, dtype=np.uint8)
        self._ok(self.L.gqr_encode(kind, s, n, width, _p(sign), _p(idx), sign.size, _p(out)))
        return out

    def allreduce_inproc(self, lanes, d, kind, width, s, topo, seed, round) -> np.ndarray:
        lanes = np.ascontiguousarray(lanes, dtype=np.uint8).copy()
        n = lanes.shape[0]
        self._ok(self.L.gqr_allreduce_inproc(_p(lanes), n, d, kind, width, s, topo, seed, round, None))
        return lanes

    def payload_combine(self, acc, inp, elem_offset, kind, width, s, n, seed, round, step, dst):
        """IntSumOps / TokenReduceOps::combine on byte lanes (returns the new acc)."""
        a = np.ascontiguousarray(acc, dtype=np.uint8).copy()
        b = np.ascontiguousarray(inp, dtype=np.uint8)
        lanes = a.size // (width // 8)
        self._ok(self.L.gqr_payload_combine(_p(a), _p(b), lanes, elem_offset, kind, width, s, n, seed,
                                            round, step, dst))
        return a

    def schedule(self, topo, n) -> list[tuple]:
        cap = 4 * n * n + 16
        buf = np.zeros(5 * cap, dtype=np.uint32)
        cnt = self.L.gqr_schedule(topo, n, _p(buf), cap)
        return [tuple(int(v) for v in buf[5 * i:5 * i + 5]) for i in range(cnt)]

    def mean(self, shards, kind, s, q=NORM_INF, p=NORM_INF, width=8, topo=0, seed=1, round=0,
             transport=0):
        sh = np.ascontiguousarray(shards, dtype=np.float64)
        n, d = sh.shape
        mean = np.zeros(d)
        norm = C.c_double()
        lw = C.c_uint32()
        pb = C.c_uint64()
        self._ok(self.L.gqr_gqsgd_mean(_p(sh), n, d, kind, s, q, p, width, topo, transport, seed,
                                       round, _p(mean), C.byref(norm), C.byref(lw), C.byref(pb)))
        return mean, norm.value, lw.value

    def sparse_payload(self, x, norm, kind, s, seed, worker, round, width) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        cap = 16 + x.size * (4 + width // 8) + (x.size + 7) // 8
        out = np.zeros(cap, dtype=np.uint8)
        size = C.c_uint64()
        self._ok(self.L.gqr_sparse_payload(_p(x), x.size, norm, kind, s, seed, worker, round, width, _p(out),
                                           cap, C.byref(size)))
        return out[:size.value].copy()

    def mean_sparse(self, shards, kind, s, q=NORM_INF, p=NORM_INF, width=8, seed=1, round=0, transport=0):
        sh = np.ascontiguousarray(shards, dtype=np.float64)
        n, d = sh.shape
        mean = np.zeros(d)
        norm = C.c_double()
        pb = C.c_uint64()
        self._ok(self.L.gqr_gqsgd_mean_sparse(_p(sh), n, d, kind, s, q, p, width, transport, seed, round,
                                              _p(mean), C.byref(norm), C.byref(pb)))
        return mean, norm.value, pb.value

    def baseline_mean(self, shards, topo=0, transport=0, round=0) -> np.ndarray:
        sh = np.ascontiguousarray(shards, dtype=np.float64)
        n, d = sh.shape
        mean = np.zeros(d)
        self._ok(self.L.gqr_baseline_mean(_p(sh), n, d, topo, transport, round, _p(mean)))
        return mean


def reference_or_none() -> Reference | None:
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None
