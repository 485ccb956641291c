"""AMG setup breakdown of the 3rd Newton first pass at n^3 (ED_AMG_VERBOSE=1 output of the last pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cp = CubeProblem(n=n, nu=0.5)
ctx = cp.context(0)
st = cp.seeded_state()
for rep in range(3):
    ctx.set_state(st)
    if rep == 2:
        print("=== pass 3 ===", file=sys.stderr, flush=True)
    out = ctx.newton_first_pass(cp.ts, cp.solver_options())
    print(rep, out["times"], flush=True)
