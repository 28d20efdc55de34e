"""Where the e2e step's time goes: the H2D of the 8 C2 shards, the step, the
D2H, alone and in the pipelined loop bench.py times."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_18627_b200 import gqsgd as G  # noqa: E402

dev = torch.device("cuda:0")
n, d = 8, 1 << 24
cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind.Exponential, s=4, width_bits=4, seed=42)
host = [torch.randn(d).pin_memory() for _ in range(n)]
out_host = torch.empty(d, pin_memory=True)
bufs = [[torch.empty(d, device=dev) for _ in range(n)] for _ in range(2)]
engs = [G.InprocSync(cfg, d, dev, torch.float32) for _ in range(2)]
s_h2d, s_d2h, comp = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)


def timed(fn, k=5):
    a, b = ev(), ev()
    torch.cuda.synchronize()
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


print("h2d alone ms", timed(lambda: [x.copy_(h, non_blocking=True) for x, h in zip(bufs[0], host)]))
print("step alone ms", timed(lambda: engs[0].run(bufs[0], 1)))
print("d2h alone ms", timed(lambda: out_host.copy_(engs[0].mean, non_blocking=True)))
ev_h = [torch.cuda.Event() for _ in range(2)]
ev_c = [torch.cuda.Event() for _ in range(2)]
ev_d = torch.cuda.Event()


def step(t):
    i = t % 2
    s_h2d.wait_event(ev_c[i])
    with torch.cuda.stream(s_h2d):
        for x, h in zip(bufs[i], host):
            x.copy_(h, non_blocking=True)
    ev_h[i].record(s_h2d)
    comp.wait_event(ev_h[i])
    comp.wait_event(ev_d)
    with torch.cuda.stream(comp):
        engs[i].run(bufs[i], t, stream=comp.cuda_stream)
    ev_c[i].record(comp)
    s_d2h.wait_event(ev_c[i])
    with torch.cuda.stream(s_d2h):
        out_host.copy_(engs[i].mean, non_blocking=True)
    ev_d.record(s_d2h)


for t in range(2):
    step(t)
torch.cuda.synchronize()
a, b = ev(), ev()
a.record(s_h2d)
for t in range(10):
    step(100 + t)
b.record(s_d2h)
torch.cuda.synchronize()
print("pipelined ms/step", a.elapsed_time(b) / 10, "h2d GB/s", n * d * 4 / (a.elapsed_time(b) / 10 * 1e-3) / 1e9)
