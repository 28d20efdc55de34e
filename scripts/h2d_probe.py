import torch, time
N=512<<20
h=torch.empty(N, dtype=torch.uint8, pin_memory=True); d=torch.empty(N, dtype=torch.uint8, device='cuda')
h2=torch.empty(64<<20, dtype=torch.uint8, pin_memory=True); d2=torch.empty(64<<20, dtype=torch.uint8, device='cuda')
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record(); 
for _ in range(5): d.copy_(h, non_blocking=True)
b.record(); torch.cuda.synchronize(); print('H2D GB/s', 5*N/(a.elapsed_time(b)*1e-3)/1e9)
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
a.record()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); b.record(); torch.cuda.synchronize()
print('H2D with concurrent D2H GB/s', 5*N/(a.elapsed_time(b)*1e-3)/1e9)
# 8 chunks of 64 MiB
hs=[torch.empty(64<<20, dtype=torch.uint8, pin_memory=True) for _ in range(8)]; ds=[torch.empty(64<<20, dtype=torch.uint8, device='cuda') for _ in range(8)]
torch.cuda.synchronize(); a.record()
for _ in range(5):
    for x,y in zip(ds,hs): x.copy_(y, non_blocking=True)
b.record(); torch.cuda.synchronize(); print('8x64MiB H2D GB/s', 5*N/(a.elapsed_time(b)*1e-3)/1e9)
