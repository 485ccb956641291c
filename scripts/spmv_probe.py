"""SpMV / sweep kernels standalone at a BASELINE cube size (default configs[4], 160^3):
mesh + tangent assembly on the device, then ed_bench_kernels.  The matrices are far
larger than the 126 MB L2, so the SpMV rows measure HBM streaming.

    python scripts/spmv_probe.py [N]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CubeProblem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
t = time.time()
cp = CubeProblem(n=n, nu=0.5, dt=0.1)
t_mesh = time.time() - t
t = time.time()
ctx = cp.context(0)
t_ctx = time.time() - t
ctx.set_state(cp.seeded_state())
t = time.time()
ctx.assemble_residuals()
ctx.assemble_tangent(cp.ts)
t_asm = time.time() - t
k = ctx.bench_kernels(cp.solver_options(), n_rep=5)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6450.0
res = {name: dict(ms=round(ms, 4), GB=round(by / 1e9, 4), gbs=round(by / ms / 1e6, 1), frac=round(by / ms / 1e6 / peak, 3))
       for name, (ms, by) in k.items()}
print(json.dumps(dict(n=n, nodes=cp.mesh.n_nodes, tets=cp.mesh.n_tets, mesh_s=round(t_mesh, 1), ctx_s=round(t_ctx, 1),
                      assemble_s=round(t_asm, 2), kernels=res)), flush=True)
