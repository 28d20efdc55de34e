"""Small runs of every round-2 kernel path for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_probe.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)


def shards(n, d):
    return [torch.from_numpy(rng.standard_normal(d).astype(np.float32)).to(dev) for _ in range(n)]


for small in (1, 0):
    _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_SMALL_PATH, small))
    for kind, s, w, n, d in [(0, 31, 8, 4, 70001), (1, 4, 4, 8, 65536 + 12), (0, 3, 4, 2, 999), (1, 7, 8, 4, 4099)]:
        cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=w, seed=3)
        sh = shards(n, d)
        eng = G.InprocSync(cfg, d, dev, torch.float32, kdraws=False)
        p = torch.zeros(d, device=dev)
        eng.run(sh, 1, param=p, lr=0.1)
        eng.check()
        g = eng.graph(sh, 5)
        g.launch()
        g.launch()
        eng.check()
        res = G.gqsgd_mean(sh, cfg, 2)  # the kdraws path for the exponential kind
_lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_SMALL_PATH, 1))
# the big-chunk quantize geometry (>= 2^25 quads) and the vector-group reduce
n, d = 8, 1 << 22
cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind.Exponential, s=4, width_bits=4, seed=9)
res = G.gqsgd_mean(shards(n, d), cfg, 1)
cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind.Standard, s=15, width_bits=8, seed=9)
res = G.gqsgd_mean(shards(n, 6553600 // 8), cfg, 1, param=torch.zeros(6553600 // 8, device=dev), lr=0.5)
# 64-bit lanes
x = shards(3, 1001)
lanes = [G.quantize_shard(t, float(max(abs(v).max().item() for v in x)), G.LevelKind.Standard, 15, 1, r, 0, 64, 3)
         for r, t in enumerate(x)]
G.allreduce_inproc(lanes, 1001, G.LevelKind.Standard, 64, 15, G.TopologyKind.Ring, 1, 0)
# the comm path at world 1 (folded graph and eager)
from dist_fakes import ThreadComm  # noqa: E402
from paper_2305_18627_b200.dist import DeviceKernels, DistSync  # noqa: E402
cfg = G.GqsgdConfig(workers=2, scheme=G.LevelKind.Exponential, s=4, width_bits=4, seed=5)
eng = DistSync(cfg, 30001, comm=ThreadComm.group(1)[0], kernels=DeviceKernels(dev), device=dev, exchange="p2p")
sh = shards(2, 30001)
eng.run(sh, 3)
eng.check()
gg = eng.make_graph(sh, 7)
gg.launch()
gg.launch()
eng.check()
# general norm orders (device sums of |x|^q + host root), the warp-layout decode with an offset param
cfg = G.GqsgdConfig(workers=4, scheme=G.LevelKind.Standard, s=15, width_bits=8, seed=2, norm=G.NormSpec(3, 5))
res = G.gqsgd_mean(shards(4, 20011), cfg, 1)
store = torch.zeros(20011 + 4, device=dev)
G.decode(res.summed_lanes, 20011, res.norm, G.LevelKind.Standard, 15, 4, 8, param=store[1:20012], lr=0.25)
torch.cuda.synchronize()
print("sanitize probe ok")
