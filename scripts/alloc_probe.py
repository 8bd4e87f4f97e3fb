import time, torch
torch.cuda.init(); torch.empty(1, device="cuda"); torch.cuda.synchronize()
for gb in (5, 20, 40):
    n = gb * (1 << 30) // 8
    t0 = time.perf_counter(); a = torch.empty(n, dtype=torch.float64, device="cuda"); torch.cuda.synchronize()
    t1 = time.perf_counter(); a.fill_(0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    a.fill_(1.0); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"{gb} GB: empty {1e3*(t1-t0):.1f} ms, first fill {1e3*(t2-t1):.1f} ms, second fill {1e3*(t3-t2):.1f} ms")
    del a; torch.cuda.empty_cache()
