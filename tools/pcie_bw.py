import torch, time
dev=torch.device('cuda:0')
n=28_320_000//4
h=torch.empty(n,dtype=torch.float32).pin_memory(); d=torch.empty(n,device=dev)
h2=torch.empty(n,dtype=torch.float32).pin_memory(); d2=torch.empty(n,device=dev)
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
for _ in range(3): d.copy_(h,non_blocking=True); h2.copy_(d2,non_blocking=True)
torch.cuda.synchronize()
def t(f,k=20):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/k
h2d=t(lambda: d.copy_(h,non_blocking=True)); d2h=t(lambda: h2.copy_(d2,non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h,non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2,non_blocking=True)
bb=t(both)
print(f"H2D {28.32/h2d/1e3:.1f} GB/s  D2H {28.32/d2h/1e3:.1f} GB/s  both-concurrent {bb*1e3:.3f} ms/step -> {1/bb:.0f}/s")
