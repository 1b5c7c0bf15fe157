import os, time, subprocess, torch
print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
subprocess.run("lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv", shell=True)
d = torch.device("cuda")
for n in (4096, 8192):
    a = torch.rand(n, n, dtype=torch.float64, device=d); b = torch.rand(n, n, dtype=torch.float64, device=d)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS DGEMM {n}: {best:.3f} ms {2*n**3/best/1e9:.2f} TFLOP/s")
nb = 1 << 30
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True); g = torch.empty(nb, dtype=torch.uint8, device=d)
for name, fn in (("H2D", lambda: g.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(g, non_blocking=True))):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
    print(f"{name} pinned 1GiB: {nb/dt/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True); g2 = torch.empty(nb, dtype=torch.uint8, device=d)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): g.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
print(f"duplex H2D+D2H concurrently: {2*nb/dt/1e9:.1f} GB/s total")
