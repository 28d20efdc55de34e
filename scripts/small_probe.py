"""Run the in-process sync through gq_mean_inproc (the fused small-d kernel
when it applies) for profiling: python scripts/small_probe.py [c1|c2] [small] [cold]
(cold = 1: a 256 MiB read before every run evicts the shards from L2)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
small = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # 2: force the fused kernel
_lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_SMALL_PATH, small))
n, d, kind, s, w = (4, 1 << 20, 0, 31, 8) if wl == "c1" else (8, 1 << 20, 1, 4, 4)
dev = torch.device("cuda:0")
cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=w, seed=42)
shards = [torch.randn(d, device=dev) for _ in range(n)]
eng = G.InprocSync(cfg, d, dev, torch.float32, kdraws=False)
cold = int(sys.argv[3]) if len(sys.argv) > 3 else 0
flush = torch.ones(64 << 20, device=dev) if cold else None
for r in range(6):
    if flush is not None:
        flush.sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run(shards, r)
    b.record()
    torch.cuda.synchronize()
    print("step %d: %.2f us (events)" % (r, a.elapsed_time(b) * 1e3), flush=True)
eng.check()
torch.cuda.synchronize()
print("ok", eng.norm.item())
