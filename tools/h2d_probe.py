"""Scratch: raw pinned H2D bandwidth, one vs several rotating host buffers."""
import torch, time
N = 78653440 // 4
d = torch.empty(N, dtype=torch.float32, device="cuda")
for nbuf in (1, 2, 4, 16):
    hs = [torch.empty(N, dtype=torch.float32).pin_memory() for _ in range(nbuf)]
    s = torch.cuda.Stream()
    for it in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for rep in range(16):
            with torch.cuda.stream(s):
                d.copy_(hs[rep % nbuf], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(nbuf, "host buffers: H2D GB/s %.1f" % (16 * N * 4 / dt / 1e9))
    del hs
