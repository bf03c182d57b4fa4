"""Time the e2e pieces through the C-ABI: sk_upload_native, the QFT program,
sk_download_native(_async), each alone and pipelined over two streams."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2304_14969_b200 import _lib  # noqa: E402
from paper_2304_14969_b200.distributed import ShardedQFT  # noqa: E402

n = 27
sq = ShardedQFT(n, "c64")
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
hin = [torch.empty(2 << n, dtype=torch.float32, pin_memory=True) for _ in range(2)]
hout = [torch.empty(2 << n, dtype=torch.float32, pin_memory=True) for _ in range(2)]
slabs = [sq.state, torch.empty_like(sq.state)]


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s0)
        fn()
        _lib.call("sk_set_stream", 0, s0.cuda_stream)
        s0.wait_stream(s1)
        b.record(s0)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def use(i):
    _lib.call("sk_set_stream", 0, (s0, s1)[i].cuda_stream)
    _lib.call("sk_rebind", sq._h, slabs[i].data_ptr())


def up():
    use(0)
    _lib.call("sk_upload_native", sq._h, hin[0].data_ptr(), 1 << n)


def down():
    use(0)
    _lib.call("sk_download_native_async", sq._h, hout[0].data_ptr(), 1 << n)


def qft():
    use(0)
    _lib.call("sk_program_run", sq._h, sq.body._h, 0, -1)


def torch_up():
    with torch.cuda.stream(s0):
        slabs[0].copy_(hin[0], non_blocking=True)


def pipe(k=6):
    def f():
        s1.wait_stream(s0)
        for j in range(k):
            use(j % 2)
            _lib.call("sk_upload_native", sq._h, hin[j % 2].data_ptr(), 1 << n)
            _lib.call("sk_program_run", sq._h, sq.body._h, 0, -1)
            _lib.call("sk_download_native_async", sq._h, hout[j % 2].data_ptr(), 1 << n)
    return f


for name, fn in (("sk_upload", up), ("torch_upload", torch_up), ("sk_download_async", down), ("qft", qft)):
    print(f"{name}: {timed(fn):.2f} ms", flush=True)
print(f"pipelined per step (6 steps): {timed(pipe(6)) / 6:.2f} ms", flush=True)
