"""Randomised parity sweep: the device gqsgd_mean against the UNMODIFIED
reference (oracle/_ref, compiled from /root/reference here and shipped as a
.so) on random configurations - worker counts 1..16, ragged d, standard and
exponential grids, lane widths 8/16/32 (and 4 where admitted), tree and ring,
L-inf shard norms combined by max or by the tree L2 fold, seeds and rounds.
Every decoded mean must be the fp32 rounding of the reference's doubles and
the norm and lane width identical. Test infrastructure (evidence), not part of
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

from oracle.bind import NORM_INF, Oracle, Reference  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=2024)
    args = ap.parse_args()
    ref, orc = Reference(), Oracle()
    rng = np.random.default_rng(args.seed)
    dev = torch.device("cuda:0")
    done = ok = skipped = 0
    first_bad = None
    while done < args.cases:
        kind = int(rng.integers(0, 2))
        n = int(rng.integers(1, 17))
        d = int(rng.choice([1, 7, 64, 1000, 4099, 65537, int(rng.integers(2, 200000))]))
        width = int(rng.choice([4, 8, 8, 16, 32]))
        s = int(rng.choice([1, 2, 3, 4, 5, 7, 15, 31, 63, 100])) if kind == 0 else int(rng.integers(1, 9))
        topo = int(rng.integers(0, 2))
        p = int(rng.choice([NORM_INF, 2]))
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
                            topo=G.TopologyKind(topo), norm=G.NormSpec(NORM_INF, p), seed=seed)
        res = G.gqsgd_mean([torch.from_numpy(x[r].astype(np.float32)).to(dev) for r in range(n)], cfg, rnd)
        want, wnorm, wlw = ref.mean(x, kind, s, q=NORM_INF, p=p, width=width, topo=topo, seed=seed, round=rnd)
        same = (res.norm == wnorm and res.lane_width_used == wlw and
                np.array_equal(res.mean.cpu().numpy(), want.astype(np.float32)))
        done += 1
        ok += same
        if not same and first_bad is None:
            first_bad = dict(kind=kind, n=n, d=d, width=width, s=s, topo=topo, p=p, seed=seed, round=rnd)
    print(json.dumps({"cases": done, "bit_identical": ok, "skipped_refused": skipped, "first_mismatch": first_bad}))
    return 0 if ok == done else 1


if __name__ == "__main__":
    sys.exit(main())
