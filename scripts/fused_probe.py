import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2305_18627_b200 import _lib, gqsgd as G
dev = torch.device('cuda:0')
def t_of(eng, x, p, reps=30):
    for _ in range(3): eng.run(x, 1, param=p, lr=0.1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for r in range(reps): eng.run(x, r, param=p, lr=0.1)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
for name, kind, s, w, n, d, sgd in [('c4bucket', 0, 15, 8, 8, 6553600, True), ('c2', 1, 4, 4, 8, 1 << 24, False), ('c3n4', 0, 31, 8, 4, 25600000, False)]:
    cfg = G.GqsgdConfig(workers=n, scheme=G.LevelKind(kind), s=s, width_bits=w, seed=3)
    x = [torch.randn(d, device=dev) for _ in range(n)]
    p = torch.zeros(d, device=dev) if sgd else None
    res = []
    for fused in (1, 0):
        _lib.check(_lib.lib().gq_set_option(_lib.GQ_OPT_FUSED_PATH, fused))
        eng = G.InprocSync(cfg, d, dev, kdraws=(kind == 1))
        # graph path (exp uses the k-draw buffer there)
        g = eng.graph(x, 0, param=p, lr=0.1)
        for _ in range(3): g.launch()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30): g.launch()
        b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 30 * 1e3)
    print(name, 'graph us fused %.1f unfused %.1f' % tuple(res))
