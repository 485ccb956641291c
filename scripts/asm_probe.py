"""Residual + tangent assembly once at the n^3 cube (ncu target for the
assembly FP64 / DRAM counters), then the device-timed assembly row.

    python scripts/asm_probe.py [N]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cp = CubeProblem(n=n, nu=0.5)
ctx = cp.context(0)
ctx.set_state(cp.seeded_state())
ctx.assemble_residuals()
ctx.assemble_tangent(cp.ts)
if os.environ.get("ASM_BENCH", "1") == "1":
    r = ctx.bench_assembly(cp.ts, n_rep=3)
    print(json.dumps(dict(n=n, tets=cp.mesh.n_tets, **r)), flush=True)
