"""amg_setup_ms of 6 consecutive first passes at n^3 (variance probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cp = CubeProblem(n=n, nu=0.5)
ctx = cp.context(0)
st = cp.seeded_state()
res = []
for rep in range(6):
    ctx.set_state(st)
    out = ctx.newton_first_pass(cp.ts, cp.solver_options())
    res.append((round(out["times"]["amg_setup_ms"], 1), round(out["times"]["total_ms"], 1)))
print(os.cpu_count(), os.environ.get("OMP_WAIT_POLICY"), res, flush=True)
