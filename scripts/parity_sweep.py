"""Randomised parity sweep: the device gqsgd_mean against the UNMODIFIED
reference (oracle/_ref, compiled from /root/reference here and shipped as a
.so) on random configurations - worker counts 1..16, ragged d, standard and
exponential grids, lane widths 8/16/32 (and 4 where admitted), tree and ring,
shard norms L-inf, L2 (parallel f64 sum) or L2 in element order
(GQ_NORM_L2_SEQUENTIAL), combined by max or by the tree L2 fold, seeds and
rounds. Every decoded mean must be the fp32 rounding of the reference's
doubles and the norm and lane width identical - except for the parallel L2
shard norm, whose summation order differs from the reference's sequential sum
(norms.cpp:41-43): there the norm must agree to 1e-12 relative and the mean
must equal the oracle's run with the device norm injected (level parity). Test infrastructure (evidence), not part of
the product path.

    python scripts/parity_sweep.py [--cases 300] [--seed 2024]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.bind import NORM_INF, Oracle, OracleError, Reference  # noqa: E402
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200._lib import GQ_NORM_L2_SEQUENTIAL  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=2024)
    args = ap.parse_args()
    ref, orc = Reference(), Oracle()
    rng = np.random.default_rng(args.seed)
    dev = torch.device("cuda:0")
    done = ok = skipped = l2_par = l2_seq = raised = 0
    first_bad = None
    while done < args.cases:
        kind = int(rng.integers(0, 2))
        n = int(rng.integers(1, 17))
        d = int(rng.choice([1, 7, 64, 1000, 4099, 65537, int(rng.integers(2, 200000))]))
        width = int(rng.choice([4, 8, 8, 16, 32]))
        s = int(rng.choice([1, 2, 3, 4, 5, 7, 15, 31, 63, 100])) if kind == 0 else int(rng.integers(1, 9))
        topo = int(rng.integers(0, 2))
        p = int(rng.choice([NORM_INF, 2]))
        q = int(rng.choice([NORM_INF, NORM_INF, 2, GQ_NORM_L2_SEQUENTIAL]))
        seed = int(rng.integers(0, 1 << 62))
        rnd = int(rng.integers(0, 1 << 40))
        # the reference's own admission (width 4 is a device extension for tokens)
        if kind == 1 and (width == 4 or not orc.check_width(kind, s, n, width)):
            skipped += 1
            continue
        if kind == 0 and (width == 4 or orc.standard_lane_width(s, n, width) is None):
            skipped += 1
            continue
        x = (orc.gaussian_shards(n, d, int(rng.integers(0, 1 << 30))) *
             float(rng.choice([1.0, 1e-30, 1e20]))).astype(np.float32).astype(np.float64)
        cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=width,
                            topo=G.TopologyKind(topo), norm=G.NormSpec(q, p), seed=seed)
        rq = NORM_INF if q == NORM_INF else 2
        conf = dict(kind=kind, n=n, d=d, width=width, s=s, topo=topo, q=q, p=p, seed=seed, round=rnd)
        dev_exc = ref_exc = None
        try:
            res = G.gqsgd_mean([torch.from_numpy(x[r].astype(np.float32)).to(dev) for r in range(n)], cfg, rnd)
        except Exception as e:  # noqa: BLE001 - compared with the reference's class below
            dev_exc = type(e).__name__
        try:
            want, wnorm, wlw = ref.mean(x, kind, s, q=rq, p=p, width=width, topo=topo, seed=seed, round=rnd)
        except OracleError as e:  # the reference throws: the device must raise the same exception class
            ref_exc = _lib._EXC.get(e.code, _lib.RuntimeFailure).__name__
        if dev_exc is not None or ref_exc is not None:
            same = dev_exc is not None and dev_exc == ref_exc
            raised += same
            done += 1
            ok += same
            if not same and first_bad is None:
                first_bad = dict(conf, device_exception=dev_exc, reference_exception=ref_exc)
            continue
        got = res.mean.cpu().numpy()
        if q == 2:  # parallel L2: norm to 1e-12, levels with the device norm injected
            inj, _, _, _ = orc.mean(x, kind, s, q=2, p=p, width=8 if width == 4 else width, topo=topo,
                                    seed=seed, round=rnd, norm_override=res.norm)
            same = (abs(res.norm - wnorm) <= 1e-12 * abs(wnorm) and res.lane_width_used == wlw and
                    np.array_equal(got, inj.astype(np.float32)))
            l2_par += 1
        else:
            same = (res.norm == wnorm and res.lane_width_used == wlw and np.array_equal(got, want.astype(np.float32)))
            l2_seq += q == GQ_NORM_L2_SEQUENTIAL
        done += 1
        ok += same
        if not same and first_bad is None:
            first_bad = conf
    print(json.dumps({"cases": done, "identical": ok, "of_which_l2_parallel_injected_norm": l2_par,
                      "of_which_l2_sequential_bit_exact": l2_seq, "of_which_both_raised": raised,
                      "skipped_refused": skipped,
                      "first_mismatch": first_bad}))
    return 0 if ok == done else 1


if __name__ == "__main__":
    sys.exit(main())
