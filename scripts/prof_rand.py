"""Run the fused random 30x20 program a couple of times (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200.circuit import build_random_circuit  # noqa: E402
from paper_2304_14969_b200.executor import compile_circuit  # noqa: E402
from paper_2304_14969_b200.ket import DenseKet  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dtype = sys.argv[2] if len(sys.argv) > 2 else "c64"
prog = compile_circuit(build_random_circuit(n, 20, 1), dtype=dtype)
st = DenseKet(n, dtype=dtype)
print("sweeps", prog.n_sweeps, [len(s.stages) for s in prog.plan.sweeps],
      [sum(len(st_.ops) for st_ in s.stages) for s in prog.plan.sweeps], flush=True)
prog.run(st)
