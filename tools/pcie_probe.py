import torch, time
dev = torch.device("cuda", 0)
n = 1 << 28  # 1 GiB of f32
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device=dev); d2 = torch.empty(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - t0
th = t(lambda: d.copy_(h, non_blocking=True))
tdh = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tb = t(both)
print(f"H2D {4*n/th/1e9:.1f} GB/s  D2H {4*n/tdh/1e9:.1f} GB/s  both: {tb*1e3:.1f} ms vs serial {1e3*(th+tdh):.1f} ms")
