"""Time the fused random 30x20 program at the default geometry (CUDA events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2304_14969_b200 import _lib  # noqa: E402
from paper_2304_14969_b200.circuit import build_random_circuit  # noqa: E402
from paper_2304_14969_b200.executor import compile_circuit  # noqa: E402
from paper_2304_14969_b200.ket import DenseKet  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
_lib.call("sk_set_stream", 0, s.cuda_stream)
for dtype in sys.argv[2:] or ["c64"]:
    prog = compile_circuit(build_random_circuit(n, 20, 1), dtype=dtype)
    st = DenseKet(n, dtype=dtype)
    prog.run(st)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        prog.run(st)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(dtype, "sweeps", prog.n_sweeps, "ms", min(ts), flush=True)
    del st
