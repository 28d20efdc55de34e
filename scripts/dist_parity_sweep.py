"""Randomised parity sweep of the multi-rank path: DistSync with the native
peer-memory communicator (exchange "p2p") for N virtual ranks as threads on one
GPU (tests/dist_fakes.ThreadComm: pointers shared directly, host waits), over
random configurations; every rank's decoded mean must be the fp32 rounding of
the unmodified reference's gqsgd_mean on all n shards. Test infrastructure.

    python scripts/dist_parity_sweep.py [--cases 60] [--seed 11]
"""
import argparse
import json
import sys
import threading
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from dist_fakes import ThreadComm  # noqa: E402
from oracle.bind import NORM_INF, Oracle, OracleError, Reference  # noqa: E402
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402
from paper_2305_18627_b200.dist import DeviceKernels, DistSync  # noqa: E402


def run_case(x, cfg, world, rnd, exchange):
    n, d = x.shape
    comms = ThreadComm.group(world)
    out, errs = [None] * world, []
    dev = torch.device("cuda:0")

    def body(r):
        try:
            torch.cuda.set_device(dev)
            eng = DistSync(cfg, d, comm=comms[r], kernels=DeviceKernels(dev), device=dev, exchange=exchange)
            eng.run([torch.from_numpy(x[w].astype(np.float32)).to(dev) for w in eng.worker_ids], rnd)
            eng.check()
            torch.cuda.synchronize()
            out[r] = (eng.exchange, eng.mean.cpu().numpy(), float(eng.norm.item()))
        except BaseException as e:  # noqa: BLE001 - reported by the caller
            errs.append(repr(e))
            comms[r].sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    return out, errs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=60)
    ap.add_argument("--seed", type=int, default=11)
    args = ap.parse_args()
    ref, orc = Reference(), Oracle()
    rng = np.random.default_rng(args.seed)
    done = ok = raised = 0
    first_bad = None
    while done < args.cases:
        world = int(rng.choice([2, 3, 4, 8]))
        n = world * int(rng.choice([1, 1, 2]))
        kind = int(rng.integers(0, 2))
        width = int(rng.choice([8, 16]))
        s = int(rng.choice([3, 7, 15])) if kind == 0 else int(rng.integers(2, 8))
        if kind == 1 and not orc.check_width(kind, s, n, width):
            continue
        if kind == 0 and orc.standard_lane_width(s, n, width) is None:
            continue
        d = int(rng.choice([1, 513, 4099, int(rng.integers(2, 100000))]))
        topo = int(rng.integers(0, 2))
        p = int(rng.choice([NORM_INF, 2]))
        seed, rnd = int(rng.integers(0, 1 << 62)), int(rng.integers(0, 1 << 40))
        x = orc.gaussian_shards(n, d, int(rng.integers(0, 1 << 30))).astype(np.float32).astype(np.float64)
        cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=width,
                            topo=G.TopologyKind(topo), norm=G.NormSpec(NORM_INF, p), seed=seed)
        out, errs = run_case(x, cfg, world, rnd, "p2p")
        try:
            want, wnorm, _ = ref.mean(x, kind, s, q=NORM_INF, p=p, width=width, topo=topo, seed=seed, round=rnd)
            same = not errs and all(o is not None and o[0] == "p2p" and o[2] == wnorm and
                                    np.array_equal(o[1], want.astype(np.float32)) for o in out)
        except OracleError as e:  # the reference throws: every rank must raise the same exception class
            cls = _lib._EXC.get(e.code, _lib.RuntimeFailure).__name__
            same = len(errs) == world and all(er.startswith(cls) for er in errs)
            raised += same
        done += 1
        ok += same
        if not same and first_bad is None:
            first_bad = dict(world=world, n=n, kind=kind, width=width, s=s, d=d, topo=topo, p=p, errs=errs[:1])
    print(json.dumps({"cases": done, "bit_identical_on_every_rank": ok,
                      "of_which_reference_raised_and_every_rank_raised_the_same_class": raised,
                      "first_mismatch": first_bad}))
    return 0 if ok == done else 1


if __name__ == "__main__":
    sys.exit(main())
