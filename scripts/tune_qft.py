"""Time QFT-n fused programs across tile geometries (per-sweep CUDA-event
timings, warm, state >> L2).  Usage: python scripts/tune_qft.py [n] [dtype]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2304_14969_b200 import _lib  # noqa: E402
from paper_2304_14969_b200.circuit import build_qft, build_random_circuit  # noqa: E402
from paper_2304_14969_b200.executor import compile_circuit  # noqa: E402
from paper_2304_14969_b200.ket import DenseKet  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dtype = sys.argv[2] if len(sys.argv) > 2 else "c64"
circ = sys.argv[3] if len(sys.argv) > 3 else "qft"
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
_lib.call("sk_set_stream", 0, stream.cuda_stream)
st = DenseKet(n, dtype=dtype)
c = build_qft(n) if circ == "qft" else build_random_circuit(n, 20, 1)
esz = 8 if dtype == "c64" else 16
tiles = [int(t) for t in os.environ["TILES"].split(",")] if "TILES" in os.environ else (
    [11, 12, 13] if dtype == "c64" else [10, 11, 12])
for T in tiles:
    for low in ([int(x) for x in os.environ["LOWS"].split(",")] if "LOWS" in os.environ else (3, 4, 5)):
        try:
            kw = {"qft_nreg": int(os.environ["QFT_NREG"])} if "QFT_NREG" in os.environ else {}
            prog = compile_circuit(c, dtype=dtype, tile_bits=T, low_bits=low, **kw)
        except Exception as exc:  # noqa: BLE001
            print(T, low, "plan failed", exc)
            continue
        ns = prog.n_sweeps
        for _ in range(3):
            prog.run(st)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(ns + 1)]
        reps = 5
        per = [0.0] * ns
        for _ in range(reps):
            ev[0].record(stream)
            for i in range(ns):
                prog.run(st, i, 1)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            for i in range(ns):
                per[i] += ev[i].elapsed_time(ev[i + 1]) / reps
        tot = sum(per)
        gbs = ns * 2 * esz * (1 << n) / (tot / 1e3) / 1e9
        print(f"T={T} low={low} sweeps={ns} total={tot:.3f} ms  {gbs:7.1f} GB/s  per-sweep=" +
              " ".join(f"{x:.3f}" for x in per), flush=True)
