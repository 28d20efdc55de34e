"""Per-rank quantize (one worker, d = 2^24, 4-bit tokens) at several CTAs per SM."""
import sys, ctypes as C, torch
sys.path.insert(0, '/root/repo')
from paper_2305_18627_b200 import _lib
from paper_2305_18627_b200 import gqsgd as G
from paper_2305_18627_b200._lib import check, lib, ptr_array
L = lib(); dev = torch.device('cuda:0'); sp = torch.cuda.current_stream().cuda_stream
d = 1 << 24
x = torch.randn(d, device=dev); norm = torch.tensor([float(x.abs().max())], dtype=torch.float64, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
lanes = torch.zeros(G.lane_bytes(d, 4), dtype=torch.uint8, device=dev)
ids = (C.c_uint32 * 1)(0); sh = ptr_array([x.data_ptr()]); la = ptr_array([lanes.data_ptr()])
for ctas in (0, 2, 1, 4):
    check(L.gq_set_option(_lib.GQ_OPT_QUANT_CTAS_PER_SM, ctas))
    f = lambda: check(L.gq_quantize(sh, 0, 1, ids, d, norm.data_ptr(), 1, 4, 8, 4, 42, 0, la, err.data_ptr(), sp))
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30): f()
    b.record(); torch.cuda.synchronize()
    print('ctas/sm', ctas, '%.2f us' % (a.elapsed_time(b) / 30 * 1e3))
