"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

    make -C oracle ref && python tests/golden/make_golden.py [--only-large]

Writes tests/golden/golden.npz (small per-config vectors) and
tests/golden/fingerprints.json (sha256 of full-size outputs). Inputs are
gaussian_shards(n, d, 12345) (verify.cpp:118-128) cast to fp32, as SURVEY §8d
specifies. Run in the build container (the reference tree is not on the GPU
box); the outputs are committed.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.bind import NORM_INF, Reference  # noqa: E402

OUT = Path(__file__).resolve().parent
DATA_SEED = 12345

# name: (kind, s, n, d, width, topo, q, p, seed, round)
CONFIGS = {
    "c1_std_s31_n4": (0, 31, 4, 4096, 8, 0, NORM_INF, NORM_INF, 42, 0),
    "exp_s7_n4": (1, 7, 4, 4096, 8, 0, NORM_INF, NORM_INF, 42, 0),
    "c2_exp_s4_n8": (1, 4, 8, 4096, 8, 0, NORM_INF, NORM_INF, 42, 0),
    "std_s15_n8_ring": (0, 15, 8, 4096, 8, 1, NORM_INF, NORM_INF, 42, 3),
    "exp_s7_n5_ring_ragged": (1, 7, 5, 1001, 8, 1, NORM_INF, NORM_INF, 9, 1),
    "std_s63_n2_l2": (0, 63, 2, 777, 8, 0, 2, 2, 5, 0),
    "exp_s5_n3_w16_l2": (1, 5, 3, 333, 16, 0, 2, 2, 11, 7),
    "std_s7_n16": (0, 7, 16, 1000, 8, 0, NORM_INF, NORM_INF, 1, 2),
    "std_s1000_n4_w16": (0, 1000, 4, 512, 8, 0, NORM_INF, NORM_INF, 3, 0),
    "exp_s123_n16_w8": (1, 123, 16, 512, 8, 1, NORM_INF, NORM_INF, 4, 5),
    "exp_s7_n6_tree": (1, 7, 6, 700, 8, 0, NORM_INF, NORM_INF, 8, 0),
    "std_s31_n3_linf_l2": (0, 31, 3, 640, 8, 0, NORM_INF, 2, 6, 0),
}

# Full-size fingerprints: (kind, s, n, d, width, topo, seed, round)
FULL = {
    "C1_std_s31_n4_d2^20": (0, 31, 4, 1 << 20, 8, 0, 42, 0),
    "C2_exp_s4_n8_d2^24": (1, 4, 8, 1 << 24, 8, 0, 42, 0),
    "std_s15_n8_d2^20": (0, 15, 8, 1 << 20, 8, 0, 42, 0),
}


# North-star sizes, each one reference call on columns
# [j0, j0+d) of gaussian_shards(n, D, 12345): (kind, s, n, j0, d, width, topo,
# seed, round, sgd). C4 = the 340M-element BERT-large gradient in 25 MiB buckets
# of 6,553,600 elements (the last 5,766,400); bucket b of step t is its own call
# with round t*52 + b (t = 3 here) and its decode feeds the SGD line
# x[j] -= eta*est[j] (trainer.cpp:335) of a fixed fp32 parameter vector.
C4_BUCKET, C4_D, C4_NB, C4_T = 6_553_600, 340_000_000, 52, 3
LARGE = {
    "C3_std_s63_n2_d25.6M": (0, 63, 2, 0, 25_600_000, 8, 0, 42, 0, False),
    "C3_std_s31_n4_d25.6M": (0, 31, 4, 0, 25_600_000, 8, 0, 42, 0, False),
    "C3_std_s15_n8_d25.6M": (0, 15, 8, 0, 25_600_000, 8, 0, 42, 0, False),
}
for _b in (0, 1, 51):
    _db = min(C4_BUCKET, C4_D - _b * C4_BUCKET)
    LARGE[f"C4_std_s15_n8_bucket{_b}"] = (0, 15, 8, _b * C4_BUCKET, _db, 8, 0, 42, C4_T * C4_NB + _b, True)
LARGE["C4_exp_s7_n8_bucket51"] = (1, 7, 8, 51 * C4_BUCKET, C4_D - 51 * C4_BUCKET, 8, 0, 42,
                                  C4_T * C4_NB + 51, True)
SGD_LR = np.float32(1e-3)
SGD_PARAM_SEED = 777  # P0 = fp32(gaussian column range of worker 0 under this seed)


def sgd_f32(p0: np.ndarray, mean: np.ndarray) -> np.ndarray:
    """The device's fused update, p - fl32(lr * fl32(mean)) with separate
    fp32 roundings (trainer.cpp:335's mul then sub)."""
    return (p0 - SGD_LR * mean.astype(np.float32)).astype(np.float32)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_config(R: Reference, kind, s, n, d, width, topo, q, p, seed, rnd):
    x = R.gaussian_shards(n, d, DATA_SEED).astype(np.float32)
    xd = x.astype(np.float64)
    stats = np.array([R.local_norm_stat(xd[r], q, p) for r in range(n)])
    norm = R.norm_allreduce_inproc(stats, q, p, rnd)
    mean, norm2, lw = R.mean(xd, kind, s, q, p, width, topo, seed, rnd)
    assert norm2 == norm
    lanes = []
    for r in range(n):
        sign, idx = R.quantize(xd[r], norm, kind, s, seed, r, rnd)
        lanes.append(R.encode(kind, s, n, lw, sign, idx))
    lanes = np.stack(lanes)
    summed = R.allreduce_inproc(lanes, d, kind, lw, s, topo, seed, rnd)
    for r in range(1, n):
        assert np.array_equal(summed[r], summed[0])
    return x, stats, norm, lanes, summed[0], mean, lw


def main() -> None:
    R = Reference()
    arrays: dict[str, np.ndarray] = {}
    meta: dict[str, dict] = {}
    for name, cfg in CONFIGS.items():
        kind, s, n, d, width, topo, q, p, seed, rnd = cfg
        x, stats, norm, lanes, summed, mean, lw = run_config(R, *cfg)
        arrays[f"{name}/x"] = x
        arrays[f"{name}/stats"] = stats
        arrays[f"{name}/lanes"] = lanes
        arrays[f"{name}/summed"] = summed
        arrays[f"{name}/mean"] = mean
        meta[name] = dict(kind=kind, s=s, n=n, d=d, width=width, topo=topo, q=q, p=p, seed=seed,
                          round=rnd, lane_width=lw, norm=norm)
    # zero shards: norm 0 short-circuit (algorithm.cpp:175-178)
    z = np.zeros((3, 64), dtype=np.float32)
    mz, nz, lwz = R.mean(z.astype(np.float64), 1, 7, NORM_INF, NORM_INF, 8, 0, 1, 0)
    arrays["zero_n3/x"] = z
    arrays["zero_n3/mean"] = mz
    meta["zero_n3"] = dict(kind=1, s=7, n=3, d=64, width=8, topo=0, q=NORM_INF, p=NORM_INF,
                           seed=1, round=0, lane_width=lwz, norm=nz)

    # reduce_pair exhaustive table, ctx (s=7, n=16, w=16) as test_exp_arith.cpp:144-164
    rows = []
    for e1 in range(0, 13):
        for e2 in range(0, 13):
            for s1 in (1, -1):
                for s2 in (1, -1):
                    for k in range(1, 9):
                        try:
                            so, eo = R.reduce_pair((s1, e1), (s2, e2), k, 7, 16, 16)
                            rows.append((s1, e1, s2, e2, k, so, eo, 0))
                        except Exception as e:  # overflow_error cases
                            rows.append((s1, e1, s2, e2, k, 0, 0, getattr(e, "code", 9)))
    arrays["kat/reduce_pair"] = np.array(rows, dtype=np.int32)
    # RNG bits KAT
    keys = [(1, 1, 0, 0, 0), (42, 1, 3, 7, 123456), (99, 2, 5, (1 << 32) | 3, 77),
            (7, 5, 2, 9, 0x8000000000000000), (0xFFFFFFFFFFFFFFFF, 2, 1, 2, 3)]
    arrays["kat/rng_keys"] = np.array(keys, dtype=np.uint64)
    arrays["kat/rng_bits"] = np.array([R.rng_bits(*k) for k in keys], dtype=np.uint64)
    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))

    fps = {}
    for name, (kind, s, n, d, width, topo, seed, rnd) in FULL.items():
        x = R.gaussian_shards(n, d, DATA_SEED).astype(np.float32)
        xd = x.astype(np.float64)
        stats = np.array([R.local_norm_stat(xd[r]) for r in range(n)])
        norm = R.norm_allreduce_inproc(stats, NORM_INF, NORM_INF, rnd)
        lanes = []
        for r in range(n):
            sign, idx = R.quantize(xd[r], norm, kind, s, seed, r, rnd)
            lanes.append(R.encode(kind, s, n, width, sign, idx))
        lanes = np.stack(lanes)
        summed = R.allreduce_inproc(lanes, d, kind, width, s, topo, seed, rnd)[0]
        mean, norm2, lw = R.mean(xd, kind, s, NORM_INF, NORM_INF, width, topo, seed, rnd)
        assert norm2 == norm and lw == width
        fps[name] = dict(kind=kind, s=s, n=n, d=d, width=width, topo=topo, seed=seed, round=rnd,
                         data_seed=DATA_SEED, norm=norm, x_sha=sha(x),
                         lanes_sha=[sha(l) for l in lanes], summed_sha=sha(summed),
                         mean_f32_sha=sha(mean.astype(np.float32)),
                         mean_sum=float(mean.sum()))
        print(name, fps[name]["summed_sha"][:16], flush=True)
    (OUT / "fingerprints.json").write_text(json.dumps(fps, indent=1, sort_keys=True))


def main_large() -> None:
    """Fingerprints of the reference at the north-star sizes (C3, C4 buckets),
    merged into fingerprints.json."""
    R = Reference()
    path = OUT / "fingerprints.json"
    fps = json.loads(path.read_text()) if path.exists() else {}
    for name, (kind, s, n, j0, d, width, topo, seed, rnd, sgd) in LARGE.items():
        x = R.gaussian_range(n, j0, d, DATA_SEED).astype(np.float32)
        xd = x.astype(np.float64)
        mean, norm, lw = R.mean(xd, kind, s, NORM_INF, NORM_INF, width, topo, seed, rnd)
        assert lw == width
        lanes = []
        for r in range(n):
            sign, idx = R.quantize(xd[r], norm, kind, s, seed, r, rnd)
            lanes.append(R.encode(kind, s, n, width, sign, idx))
        lanes = np.stack(lanes)
        summed = R.allreduce_inproc(lanes, d, kind, width, s, topo, seed, rnd)[0]
        f = dict(kind=kind, s=s, n=n, j0=j0, d=d, width=width, topo=topo, seed=seed, round=rnd,
                 data_seed=DATA_SEED, norm=norm, x_sha=sha(x), lanes_sha=[sha(l) for l in lanes],
                 summed_sha=sha(summed), mean_f32_sha=sha(mean.astype(np.float32)), mean_f64_sha=sha(mean),
                 mean_sum=float(mean.sum()))
        if sgd:
            p0 = R.gaussian_range(1, j0, d, SGD_PARAM_SEED)[0].astype(np.float32)
            f.update(sgd_lr=float(SGD_LR), sgd_param_seed=SGD_PARAM_SEED, param0_sha=sha(p0),
                     param_f32_sha=sha(sgd_f32(p0, mean)))
        fps[name] = f
        print(name, f["summed_sha"][:16], flush=True)
    path.write_text(json.dumps(fps, indent=1, sort_keys=True))


if __name__ == "__main__":
    if "--only-large" in sys.argv:
        main_large()
    else:
        main()
        main_large()
