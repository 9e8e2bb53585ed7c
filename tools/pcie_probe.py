"""Host<->device copy bandwidth on the GPU box (pinned memory), alone and
bidirectional: the ceiling of bench.py's e2e leg."""
import time
import torch

n = 2160085000 // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


gb = n * 8 / 1e9
t = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
print(f"H2D alone   {gb / t:6.1f} GB/s  {t * 1e3:6.1f} ms")
t = timeit(lambda: h_out.copy_(d_out, non_blocking=True))
print(f"D2H alone   {gb / t:6.1f} GB/s  {t * 1e3:6.1f} ms")


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


t = timeit(both)
print(f"H2D+D2H     {2 * gb / t:6.1f} GB/s total  {t * 1e3:6.1f} ms (2 x {gb:.2f} GB)")


# several concurrent D2H / H2D copies (separate copy engines?)
for ns in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns

    def multi_d2h():
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                h_out[i * chunk:(i + 1) * chunk].copy_(d_out[i * chunk:(i + 1) * chunk],
                                                       non_blocking=True)

    def multi_h2d():
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                d_in[i * chunk:(i + 1) * chunk].copy_(h_in[i * chunk:(i + 1) * chunk],
                                                      non_blocking=True)
    t = timeit(multi_d2h)
    print(f"D2H {ns} streams {gb / t:6.1f} GB/s  {t * 1e3:6.1f} ms")
    t = timeit(multi_h2d)
    print(f"H2D {ns} streams {gb / t:6.1f} GB/s  {t * 1e3:6.1f} ms")
