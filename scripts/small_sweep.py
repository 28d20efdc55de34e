"""Per-call time of gq_mean_inproc (eager, stream-ordered) with the fused
small-d kernel on and off, over n*d: python scripts/small_sweep.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402

dev = torch.device("cuda:0")
rows = []
for kind, s, w in [(0, 31, 8), (1, 4, 4)]:
    n = 4 if kind == 0 else 8
    for lg in range(8, 22):
        d = 1 << lg
        cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=w, seed=42)
        shards = [torch.randn(d, device=dev) for _ in range(n)]
        res = {}
        for small in (2, 0):  # 2: the fused kernel forced (up to n * d = 2^23)
            _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_SMALL_PATH, small))
            eng = G.InprocSync(cfg, d, dev, torch.float32, kdraws=False)
            for r in range(5):
                eng.run(shards, r)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for r in range(200):
                eng.run(shards, 10 + r)
            b.record()
            torch.cuda.synchronize()
            eng.check()
            res[small] = a.elapsed_time(b) / 200 * 1e3
        rows.append({"kind": kind, "n": n, "d": d, "fused_us": round(res[2], 2), "three_kernel_us": round(res[0], 2)})
        print(json.dumps(rows[-1]), flush=True)
_lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_SMALL_PATH, 1))
