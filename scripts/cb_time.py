"""Time k_ctrl_bloch (apply_controlled_bloch_sums) at width w (CUDA events,
warm): python scripts/cb_time.py [w] [dtype]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2304_14969_b200 import _lib  # noqa: E402
from paper_2304_14969_b200.circuit import gate_matrix, u3_matrix  # noqa: E402
from paper_2304_14969_b200.ket import DenseKet  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dtype = sys.argv[2] if len(sys.argv) > 2 else "c128"
s_ = torch.cuda.Stream()
torch.cuda.set_stream(s_)
_lib.call("sk_set_stream", 0, s_.cuda_stream)
s = DenseKet(w, dtype=dtype)
s.apply_1q(w - 1, gate_matrix("h"))
U = u3_matrix(0.3, 0.7, 1.1)
for c, t in ((4, 17), (0, 1), (w - 1, 3)):
    s.apply_controlled_bloch_sums(c, 1, t, U)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_)
    for _ in range(10):
        s.apply_controlled_bloch_sums(c, 1, t, U)
    b.record(s_)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    nb = (1 << w) * (8 if dtype == "c64" else 16) * 1.5
    print(f"c={c} t={t}: {ms * 1e3:.1f} us  {nb / ms / 1e6:.0f} GB/s (algorithmic 1.5x state)", flush=True)
