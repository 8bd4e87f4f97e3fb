import time, torch
n = 10077696
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    V = torch.empty((251, n), dtype=torch.float64, device="cuda")
    Z = torch.empty((250, n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    V[100].fill_(1.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(rep, "alloc", t1 - t0, "first touch row", t2 - t1)
    del V, Z
    t3 = time.perf_counter(); torch.cuda.empty_cache(); torch.cuda.synchronize(); print("free", time.perf_counter() - t3)
