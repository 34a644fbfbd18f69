"""D2H bandwidth probe: one copy vs several concurrent copy streams (pinned host)."""
import time, torch
n = 1 << 30
d = torch.empty(n, dtype=torch.complex128, device="cuda")
h = torch.empty(n, dtype=torch.complex128, pin_memory=True)
def run(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    chunk = n // k
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            h[i * chunk:(i + 1) * chunk].copy_(d[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return 16 * n / dt / 1e9
for k in (1, 1, 2, 4, 8):
    print(f"D2H streams={k}: {run(k):.1f} GB/s", flush=True)
# chunked sequential on one stream (64 MiB pieces)
torch.cuda.synchronize(); t = time.perf_counter()
c = 1 << 22
for i in range(0, n, c):
    h[i:i + c].copy_(d[i:i + c], non_blocking=True)
torch.cuda.synchronize(); print(f"D2H 64MiB chunks one stream: {16*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
d.copy_(h, non_blocking=True); torch.cuda.synchronize()
print(f"H2D: {16*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
