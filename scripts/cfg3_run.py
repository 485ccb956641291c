"""BASELINE configs[3] on the GPU path: tensile test of the anisotropic arterial wall
(CylinderProblem: 8 x 128 x 64 hexes, HGO fibres in local circumferential frames, 10 % axial
stretch prescribed on the top end, ramped over 10 generalized-alpha steps).

    python scripts/cfg3_run.py [n_r n_theta n_z] [steps]

Prints one JSON line per step (Newton and linear counts, residual history, wall time) and a
summary line.  The reference cannot run this configuration; parity of the pieces
is pinned by tests/test_gpu_parity.py against oracle/restate.py on a small cylinder."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1809_06350_b200 import CylinderProblem, api  # noqa: E402

dims = [int(v) for v in sys.argv[1:4]] if len(sys.argv) >= 4 else [8, 128, 64]
steps = int(sys.argv[4]) if len(sys.argv) >= 5 else 10
t0 = time.perf_counter()
cy = CylinderProblem(n_r=dims[0], n_theta=dims[1], n_z=dims[2])
ctx = cy.context(0)
ctx.set_state(api.State.zeros(cy.mesh.n_nodes))
opts = cy.solver_options()
print(json.dumps(dict(nodes=cy.mesh.n_nodes, tets=cy.mesh.n_tets, unknowns=cy.nv + cy.np,
                      setup_s=round(time.perf_counter() - t0, 2))), flush=True)
tot = 0.0
for k in range(1, steps + 1):
    ctx.set_prescribed_displacement(cy.top_nodes, cy.top_displacement(k))
    t = time.perf_counter()
    g = ctx.step(cy.ts, opts, tol_r=1e-8, tol_a=1e-6, l_max=20)
    dt = time.perf_counter() - t
    tot += dt
    s = ctx.get_state()
    u = s.u.reshape(-1, 3)
    r = np.hypot(cy.mesh.nodes[:, 0] + u[:, 0], cy.mesh.nodes[:, 1] + u[:, 1])
    mid = np.abs(cy.mesh.nodes[:, 2] - 0.5 * cy.length) < 1e-9 * cy.length
    print(json.dumps(dict(step=k, stretch=round(cy.stretch * k / cy.n_steps, 4), converged=int(g["converged"]),
                          newton_iters=g["newton_iters"], res_history=[float(v) for v in g["res_history"]],
                          linear={a: int(b) for a, b in g["linear"].items() if a != "t_solve"},
                          wall_s=round(dt, 3), p_max=float(np.abs(s.p).max()),
                          mid_plane_outer_radius=float(r[mid].max()) if mid.any() else None)), flush=True)
    if not g["converged"]:
        break
print(json.dumps(dict(steps=k, total_s=round(tot, 2), s_per_step=round(tot / k, 3))), flush=True)
