import torch, time
n = 1 << 29  # 4 GiB of doubles
d = torch.empty(n, dtype=torch.float64, device="cuda")
d.fill_(1.0)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for chunk in [1 << 22, 1 << 25, n]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(0, n, chunk):
        h[i:i + chunk].copy_(d[i:i + chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"D2H chunk {chunk*8>>20} MiB: {n*8/dt/1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
half = n // 2
h[:half].copy_(d[:half], non_blocking=True)
with torch.cuda.stream(s2):
    h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"D2H two streams: {n*8/dt/1e9:.1f} GB/s")
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"H2D: {n*8/dt/1e9:.1f} GB/s")
