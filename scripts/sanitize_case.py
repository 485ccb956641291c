"""One first Newton corrector pass on a small seeded cube (compute-sanitizer target):
every kernel family of the path runs -- element kernels, K4 split, coupled SpMV,
tagged dataflow / group / chain sweeps, dense tail, Krylov vector kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cp = CubeProblem(n=n, nu=0.5)
ctx = cp.context(0)
ctx.set_state(cp.seeded_state())
out = ctx.newton_first_pass(cp.ts, cp.solver_options())
print("n", n, "norm", out["norm"], "stats", out["stats"], "launches", out["times"]["kernel_launches"])
