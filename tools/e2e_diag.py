import sys, time, torch
sys.path.insert(0, '.')
from paper_2103_11991_b200 import SpGEMM, CsrMatrix
from workloads import generators as g
A, B = g.config("C2", device="cuda")
def host(M):
    return CsrMatrix(M.nrows, M.ncols, M.row_map.to(torch.int32).cpu().pin_memory(), M.entries.cpu().pin_memory(), M.values.cpu().pin_memory())
hA, hB = host(A), host(B)
h = SpGEMM()
for nb in (1, 8):
    for _ in range(2): h.multiply_host(hA, hB, blocks=nb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3): C = h.multiply_host(hA, hB, blocks=nb)
    torch.cuda.synchronize()
    print(nb, "wall ms/call", (time.perf_counter() - t0) / 3 * 1e3)
# pure copies of the same bytes, duplex
d = [torch.empty_like(x, device="cuda") for x in (hA.row_map, hA.entries, hA.values, hB.row_map, hB.entries, hB.values)]
hc = [torch.empty(C.entries.numel(), dtype=torch.int32, pin_memory=True), torch.empty(C.values.numel(), dtype=torch.float64, pin_memory=True)]
dc = [torch.empty(C.entries.numel(), dtype=torch.int32, device="cuda"), torch.empty(C.values.numel(), dtype=torch.float64, device="cuda")]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1):
    for x, y in zip(d, (hA.row_map, hA.entries, hA.values, hB.row_map, hB.entries, hB.values)): x.copy_(y, non_blocking=True)
with torch.cuda.stream(s2):
    for x, y in zip(hc, dc): x.copy_(y, non_blocking=True)
torch.cuda.synchronize(); print("duplex copies ms", (time.perf_counter() - t0) * 1e3)
torch.cuda.synchronize(); t0 = time.perf_counter()
for x, y in zip(hc, dc): x.copy_(y, non_blocking=True)
torch.cuda.synchronize(); print("D2H only ms", (time.perf_counter() - t0) * 1e3)
