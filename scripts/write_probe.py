import torch
x=torch.empty(1<<24, device='cuda'); y=torch.empty(1<<24, device='cuda'); z=torch.empty(1<<21, dtype=torch.int32, device='cuda')
def t(fn, k=50):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/k*1e3
us=t(lambda: x.fill_(1.0)); print('fill 64MB us', us, 'GB/s', 64*2**20/us/1e3)
us=t(lambda: y.copy_(x)); print('copy 64MB us', us, 'GB/s', 128*2**20/us/1e3)
big=torch.empty(1<<28, device='cuda'); us=t(lambda: big.fill_(2.0), 10); print('fill 1GB GB/s', 2**30/us/1e3)
