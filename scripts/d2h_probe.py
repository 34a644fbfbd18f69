"""Raw pinned device->host / host->device copy rates of the box (one copy, two streams, 256 MiB pieces):
the bound of the end-to-end C2 number, which downloads 16 GiB per step."""
import torch, time
n = 1 << 32  # 4 GiB
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
one = t(lambda: h.copy_(d, non_blocking=True))
print("one stream  D2H %.1f GB/s" % (n / one / 1e9))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def two():
    with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h[n // 2 :].copy_(d[n // 2 :], non_blocking=True)
print("two streams D2H %.1f GB/s" % (n / t(two) / 1e9))
def chunks():
    c = 1 << 28
    for i in range(0, n, c): h[i:i+c].copy_(d[i:i+c], non_blocking=True)
print("256MiB chunks   %.1f GB/s" % (n / t(chunks) / 1e9))
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
print("H2D             %.1f GB/s" % (n / t(lambda: d.copy_(h2, non_blocking=True)) / 1e9))
