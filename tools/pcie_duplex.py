"""Is PCIe full duplex here?  H2D and D2H copy-engine copies alone and concurrently, and
the zero-copy kernels (host reads / host writes) alone and concurrently."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

dev = torch.device("cuda", 0)
nb = 32 << 20
h1 = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d1 = torch.empty(nb, dtype=torch.uint8, device=dev)
d2 = torch.empty(nb, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    s1.synchronize()
    s2.synchronize()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t1 = timed(h2d)
t2 = timed(d2h)
t3 = timed(lambda: (h2d(), d2h()))
print(f"CE H2D {nb / t1 / 1e6:.1f} GB/s, D2H {nb / t2 / 1e6:.1f} GB/s, both {2 * nb / t3 / 1e6:.1f} GB/s combined")
# zero-copy: a kernel reading host memory (sum) and one writing host memory (fill)
hv1 = h1.view(torch.int32)
hv2 = h2.view(torch.int32)
x1 = torch.empty_like(d1).view(torch.int32)
t4 = timed(lambda: x1.copy_(hv1.to(dev, non_blocking=True)))
print(f"(reference) to(dev) {nb / t4 / 1e6:.1f} GB/s")
