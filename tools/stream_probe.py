"""Reference HBM rates for the volume kernel's traffic mix on this GPU:
torch elementwise kernels over config-5-sized float64 arrays (2.2 GB each):
copy (1 read : 1 write) and add (2 reads : 1 write, the apply's 16 B read
+ 8 B written per row).  CUDA events, best of 10."""
import torch

n = 270_000_000
a = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.rand(n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)


def best(f, nbytes):
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{f.__name__:6s} {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s", flush=True)


def copy():
    c.copy_(a)


def add():
    torch.add(a, b, out=c)


def read2():
    torch.dot(a, b)


best(copy, 16 * n)
best(add, 24 * n)
best(read2, 16 * n)
