"""Cold- vs warm-L2 time of small streaming reads on one B200: torch sum and
gq_norm over 4 workers, after a 256 MiB read (cold) or back to back (warm).
    python scripts/cold_probe.py -> lines on stdout"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200._lib import check, lib, ptr_array  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.ones(64 << 20, device=dev)
L = lib()
sp = torch.cuda.current_stream().cuda_stream


def t_of(fn, cold, reps=20):
    tot = 0.0
    for _ in range(reps + 2):
        if cold:
            flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / (reps + 2) * 1e3


for mb in (4, 16, 64, 256):
    d = (mb << 20) // 16
    xs = [torch.randn(d, device=dev) for _ in range(4)]
    big = torch.cat(xs)
    st = torch.zeros(4, dtype=torch.float64, device=dev)
    nm = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = torch.zeros(int(L.gq_norm_workspace_bytes(4, d)), dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    arr = ptr_array([x.data_ptr() for x in xs])
    norm = lambda: check(L.gq_norm(arr, 0, 4, d, 0xFFFFFFFF, 0xFFFFFFFF, st.data_ptr(), nm.data_ptr(),
                                   ws.data_ptr(), err.data_ptr(), sp))
    amax = lambda: big.abs().amax()
    cp = torch.empty_like(big)
    copy = lambda: cp.copy_(big)
    for name, fn in (("gq_norm", norm), ("torch_sum", lambda: big.sum()), ("copy", copy)):
        w, c = t_of(fn, False), t_of(fn, True)
        print(f"{mb:4d} MiB {name:10s} warm {w:8.2f} us  cold {c:8.2f} us  cold GB/s {mb * 2**20 / c / 1e3:8.1f}")
