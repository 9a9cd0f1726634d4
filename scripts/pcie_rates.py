"""PCIe copy rates of an 80 MB float64 array between pinned host memory and the
device: one copy vs chunks spread over several streams."""
import torch

n = 10_000_000
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(16)]


def chunked(dst, src, k, ns):
    m = (n + k - 1) // k
    cur = torch.cuda.current_stream()
    for s in streams[:ns]:
        s.wait_stream(cur)
    for i in range(k):
        with torch.cuda.stream(streams[i % ns]):
            dst[i * m:(i + 1) * m].copy_(src[i * m:(i + 1) * m], non_blocking=True)
    for s in streams[:ns]:
        cur.wait_stream(s)


def rate(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[5], 8 * n / (ts[5] * 1e-3) / 1e9


for name, f in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    print("%-16s %.3f ms %.1f GB/s" % ((name,) + rate(f)))
for k, ns in [(2, 2), (4, 2), (4, 4), (8, 4), (8, 8), (16, 8), (16, 16)]:
    print("%-16s %.3f ms %.1f GB/s" % (("h2d %dx%d" % (k, ns),) + rate(lambda: chunked(d, h, k, ns))))
    print("%-16s %.3f ms %.1f GB/s" % (("d2h %dx%d" % (k, ns),) + rate(lambda: chunked(h, d, k, ns))))
