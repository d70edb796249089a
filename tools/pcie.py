"""Pinned host <-> device copy bandwidth, one direction and both at once (development tool)."""
import torch

n = 64 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    s1.wait_stream(torch.cuda.current_stream())
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
torch.cuda.synchronize()
st = torch.cuda.current_stream()
s1.wait_stream(st)
s2.wait_stream(st)
bo = t(both)
print(f"H2D {n / h2d / 1e6:.1f} GB/s ({h2d:.3f} ms), D2H {n / d2h / 1e6:.1f} GB/s ({d2h:.3f} ms), "
      f"both at once {bo:.3f} ms per 64 MiB pair")
