"""Pinned H2D bandwidth: one copy stream vs the same bytes split over 2 / 4 streams,
and chunk-size sensitivity (the e2e floor)."""
import torch

n = 1 << 28  # 2 GiB of f64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]


def run(k, pieces):
    step = n // pieces
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(pieces):
        s = ss[i % k]
        s.wait_event(a)
        with torch.cuda.stream(s):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    for s in ss[:k]:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return n * 8 / a.elapsed_time(b) / 1e6


for k, pieces in [(1, 1), (1, 8), (2, 2), (2, 8), (4, 4), (4, 16), (1, 64)]:
    run(k, pieces)
    print("streams %d pieces %2d: %.1f GB/s" % (k, pieces, max(run(k, pieces) for _ in range(3))), flush=True)
