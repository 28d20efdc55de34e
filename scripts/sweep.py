"""C5 size sweep on one B200 (BASELINE.json configs[4]): d = 2^16..2^30 x
lane widths x schemes with n = 8 workers simulated on the device, device
time per sync (CUDA events, warm, inputs > L2 or re-used as stated) next to
the fp32 tree-sum of the same shards. Each sync is one CUDA graph launch
(InprocSync.graph), so small sizes measure the kernels, not launch latency.
Writes JSON lines to stdout.

    python scripts/sweep.py [--max-log2 30] [--n 8]

At n = 8 the admissible grids are (check_width / standard_lane_width):
standard 8-bit s <= 15, 4-bit refused (n (s+1) <= 8 needs s = 0), 2-bit
refused; exponential 8-bit s <= 124 (s = 7 used), 4-bit s <= 4, 2-bit refused.
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402

CONFIGS = [  # (label, kind, s, width)
    ("std-8bit-s15", 0, 15, 8),
    ("exp-8bit-s7", 1, 7, 8),
    ("exp-4bit-s4", 1, 4, 4),
]


def time_it(fn, reps):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=16)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--n", type=int, default=8)
    args = ap.parse_args()
    L = _lib.lib()
    dev = torch.device("cuda:0")
    n = args.n
    for lg in range(args.min_log2, args.max_log2 + 1):
        d = 1 << lg
        per_worker = d * 4
        if n * per_worker * 2.2 > 150e9:  # shards + lanes + mean must fit with margin
            break
        gen = torch.Generator(device=dev).manual_seed(lg)
        shards = [torch.randn(d, device=dev, generator=gen) for _ in range(n)]
        reps = max(3, min(200, (1 << 28) // (n * d)))
        acc = torch.empty(d, device=dev)
        ptrs = _lib.ptr_array([x.data_ptr() for x in shards])
        sp = torch.cuda.current_stream().cuda_stream
        fp32_ms = time_it(lambda: L.gq_baseline_mean_inproc(ptrs, n, d, 0, acc.data_ptr(), sp), reps)
        for label, kind, s, width in CONFIGS:
            cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=width, seed=7)
            try:
                eng = G.InprocSync(cfg, d, dev)
            except G.InvalidArgument as e:
                print(json.dumps({"d": d, "config": label, "refused": str(e)}), flush=True)
                continue
            g = eng.graph(shards, 0, write_lanes=False)  # one launch per sync (round on the device)
            ms = time_it(g.launch, reps)
            eng.check()
            print(json.dumps({"d": d, "log2d": lg, "n": n, "config": label, "lane_width": eng.plan.lane_width,
                              "ms": ms, "elem_per_s": n * d / (ms * 1e-3),
                              "fp32_tree_sum_ms": fp32_ms, "speedup_vs_fp32_sum": fp32_ms / ms,
                              "reps": reps, "l2": "inputs > 126 MB L2" if n * d * 4 > 126e6 else "inputs fit L2"}),
                  flush=True)
            del eng
        del shards
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
