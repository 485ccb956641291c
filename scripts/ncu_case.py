"""One Newton first pass on an n^3 cube (for ncu captures): python scripts/ncu_case.py N [NU] [DT]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
nu = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
dt = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
cp = CubeProblem(n=n, nu=nu, dt=dt)
ctx = cp.context(0)
ctx.set_state(cp.seeded_state())
out = ctx.newton_first_pass(cp.ts, cp.solver_options())
print("ok", out["stats"], out["times"]["total_ms"])
