"""Host<->device copy bandwidth of 1 GiB pinned buffers: H2D alone, D2H
alone, both at once on two streams (is the link full duplex here?)."""
import torch

n = 1 << 28  # floats = 1 GiB
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d0 = torch.empty(n, dtype=torch.float32, device="cuda")
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        s0.synchronize(); s1.synchronize()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def h2d():
    with torch.cuda.stream(s0):
        d0.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s1):
        h_out.copy_(d1, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timeit(fn)
    gb = (2 if name == "both" else 1) * 4 * n / 1e9
    print(f"{name}: {ms:.2f} ms  {gb / ms * 1e3:.1f} GB/s")
