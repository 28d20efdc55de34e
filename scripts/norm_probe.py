"""Norm pass at C2 (8 x 2^24 fp32) with and without the k draws riding along,
and the k draws alone (scripts/norm_probe.py -> lines on stdout)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_18627_b200 import _lib  # noqa: E402
from paper_2305_18627_b200._lib import check, lib, ptr_array  # noqa: E402

dev = torch.device("cuda:0")
L = lib()
sp = torch.cuda.current_stream().cuda_stream
n, d = 8, 1 << 24
xs = [torch.randn(d, device=dev) for _ in range(n)]
st = torch.zeros(n, dtype=torch.float64, device=dev)
nm = torch.zeros(1, dtype=torch.float64, device=dev)
ws = torch.zeros(int(L.gq_norm_workspace_bytes(n, d)), dtype=torch.uint8, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
arr = ptr_array([x.data_ptr() for x in xs])
INF = 0xFFFFFFFF
spec = _lib.GqKdraws(None, n, 1, 4, 4, 0, 0, 0, d, 42, 0)
kb = int(L.gq_kdraws_bytes(C.byref(spec)))
kbuf = torch.empty(kb // 4, dtype=torch.int32, device=dev)
spec.buf = kbuf.data_ptr()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


print("norm plain      %.1f us" % timed(lambda: check(L.gq_norm(arr, 0, n, d, INF, INF, st.data_ptr(), nm.data_ptr(),
                                                                  ws.data_ptr(), err.data_ptr(), sp))))
print("norm + kdraws   %.1f us" % timed(lambda: check(L.gq_norm_kdraws(arr, 0, n, d, INF, INF, st.data_ptr(),
                                                                         nm.data_ptr(), ws.data_ptr(), err.data_ptr(),
                                                                         C.byref(spec), sp))))
one = ptr_array([xs[0].data_ptr()])
d1 = 4096
# the k draws alone: the element-order L2 pass over 4096 elements runs them in a separate full-grid kernel
print("kdraws alone    %.1f us  [element-order L2 of 4096 elements + kdraw_kernel over all k words]" % timed(
    lambda: check(L.gq_norm_kdraws(one, 0, 1, d1, _lib.GQ_NORM_L2_SEQUENTIAL, INF, st.data_ptr(), nm.data_ptr(),
                                   ws.data_ptr(), err.data_ptr(), C.byref(spec), sp))))
print("k words bytes", kb)
