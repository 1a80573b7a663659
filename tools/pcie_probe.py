"""PCIe H2D throughput from pinned host memory with 1-4 streams and 1-4 pieces,
and H2D beside D2H (development probe for the e2e pipeline bound)."""
import torch, time
n = 64 << 20  # 256 MB of fp32
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(4)]
s = [torch.cuda.Stream() for _ in range(4)]
def run(k, parts):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(k):
        with torch.cuda.stream(s[i]):
            for p in range(parts):
                lo, hi = n * p // parts, n * (p + 1) // parts
                d[i][lo:hi].copy_(h[i][lo:hi], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return k * n * 4 / dt / 1e9
for k in (1, 2, 4):
    for parts in (1, 4):
        r = max(run(k, parts) for _ in range(3))
        print("streams %d pieces %d: %.1f GB/s H2D" % (k, parts, r))
# D2H concurrently with H2D
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s[0]): d[0].copy_(h[0], non_blocking=True)
with torch.cuda.stream(s[1]): h[1].copy_(d[1], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("H2D + D2H concurrent 256 MB each: %.2f ms" % (dt * 1e3))
