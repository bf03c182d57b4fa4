"""HBM bandwidth of the per-gate DenseKet kernels at width w (default 28):
CUDA-event time per call, algorithmic bytes per call, and
the fraction of MEASURED_PEAKS.json hbm_gbs.  One JSON line per kernel.

    python scripts/pergate_bw.py [w] [dtype]
"""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_14969_b200 import _lib  # noqa: E402
from paper_2304_14969_b200.circuit import gate_matrix, u3_matrix  # noqa: E402
from paper_2304_14969_b200.ket import DenseKet, permute_qubits  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 28
dtype = sys.argv[2] if len(sys.argv) > 2 else "c64"
B = 8 if dtype == "c64" else 16
N = 1 << w
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
    else 6650.0
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
_lib.call("sk_set_stream", 0, stream.cuda_stream)
s = DenseKet(w, dtype=dtype)
s.apply_1q(w - 1, gate_matrix("h"))
U = u3_matrix(0.3, 0.7, 1.1)
P = gate_matrix("p", (0.4,))
keep = []


def timed(name, fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        r = fn()
        if r is not None:
            keep.append(r)
            if len(keep) > 2:
                keep.pop(0)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = nbytes / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": name, "width": w, "dtype": dtype, "ms": round(ms, 4), "bytes": nbytes,
                      "gbs": round(gbs, 1), "frac": round(gbs / peak, 3)}), flush=True)


for q in (0, 1, 5, w // 2, w - 1):
    timed(f"k_apply_1q q={q}", lambda q=q: s._apply_1q_unchecked(q, U), 2 * N * B)
timed("k_apply_1q diag q=3", lambda: s._apply_1q_unchecked(3, P), 2 * N * B)
timed("k_apply_ctrl cx c=2 t=9", lambda: s.apply_controlled((2,), (1,), 9, gate_matrix("x")), 2 * (N // 2) * B)
timed("k_apply_ctrl cp c=2 t=9 (|11> quarter)", lambda: s.apply_controlled((2,), (1,), 9, P), 2 * (N // 4) * B)
timed("k_ctrl_bloch c=4 t=17", lambda: s.apply_controlled_bloch_sums(4, 1, 17, U), N * B + (N // 2) * B)
timed("k_bloch q=0", lambda: s._bloch_sums(0), N * B)
timed("k_bloch q=13", lambda: s._bloch_sums(13), N * B)
timed("k_norm2", lambda: s.norm(), N * B)
timed("k_round (rotate-project-compact) q=7", lambda: s.round_qubit(7, U, 1.0), N * B + (N // 2) * B, reps=5)
timed("k_compact q=7", lambda: s._compact(7, 0, 1.0), (N // 2) * B * 2, reps=5)
half = DenseKet(w - 1, dtype=dtype)
one = DenseKet(1, np.array([0.6, 0.8], dtype=complex), dtype=dtype)
timed("k_kron (w-1) x 1", lambda: half.kron_compose(one), N * B + (N // 2) * B, reps=5)
del half
timed("k_scale", lambda: s.scale(1j), 2 * N * B)
timed("k_pauli x0 z5", lambda: s.apply_pauli_layer([(0, "x"), (5, "z")]), 2 * N * B)
rev = list(reversed(range(w)))
timed("k_permute bit-reversal", lambda: permute_qubits(s, rev), 2 * N * B, reps=3)
rot = list(range(1, w)) + [0]
timed("k_permute rotate-by-1", lambda: permute_qubits(s, rot), 2 * N * B, reps=3)
