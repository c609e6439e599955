"""Streaming bandwidth of plain read/write mixes on this GPU (torch elementwise
kernels, 128 MB fp64 vectors): what a 1R1W / 2R1W / 3R1W stream reaches, to
put the sweep kernels' fractions in context."""
import torch

n = 256 ** 3
dev = "cuda"
a, b, c, d = (torch.rand(n, dtype=torch.float64, device=dev) for _ in range(4))
out = torch.empty_like(a)


def timeit(fn, nbytes, reps=50):
    for _ in range(5):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / reps * 1e-3
    return nbytes / t / 1e9, t * 1e6


print("1R1W copy   %.0f GB/s %.1f us" % timeit(lambda: out.copy_(a), 16 * n))
print("2R1W add    %.0f GB/s %.1f us" % timeit(lambda: torch.add(a, b, out=out), 24 * n))
print("3R1W addcmul %.0f GB/s %.1f us" % timeit(lambda: torch.addcmul(a, b, c, out=out), 32 * n))
print("1R0W sum    %.0f GB/s %.1f us" % timeit(lambda: a.sum(), 8 * n))
print("2R1W inplace a+=b %.0f GB/s %.1f us" % timeit(lambda: a.add_(b), 24 * n))
