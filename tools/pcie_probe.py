"""Host<->device copy bandwidth on the box: pinned 1 GiB H2D, D2H, and both
concurrently on two streams (bounds the e2e number)."""
import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for _ in range(2):
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    tb = t(both)
print(f"H2D {n / th / 1e6:.1f} GB/s  D2H {n / td / 1e6:.1f} GB/s  both {2 * n / tb / 1e6:.1f} GB/s combined")
