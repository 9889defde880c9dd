import torch, time, numpy as np
n = 640*480
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
def med(f, k=300):
    for _ in range(20): f()
    ts=[]
    for _ in range(k):
        t=time.perf_counter(); f(); ts.append(time.perf_counter()-t)
    return np.median(ts)*1e6
def one():
    d.copy_(h, non_blocking=True); torch.cuda.current_stream().synchronize()
def split(m):
    c = n // m
    for i in range(m):
        with torch.cuda.stream(streams[i % 4]):
            d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
    for s in streams[:m]: s.synchronize()
print("one copy us", med(one))
for m in (2, 4):
    print(f"{m} copies us", med(lambda: split(m)))
def sync_only():
    torch.cuda.current_stream().synchronize()
print("sync only us", med(sync_only))
