"""Generates the golden vectors in tests/golden/ from the compiled reference
(oracle/_ref, built from /root/reference/proj/src by oracle/Makefile).

  python tests/golden/make_golden.py

cube_n3.npz   : seeded 3^3 cube (nu 0.4): residuals, tangent planes, first
                corrector pass (x, rhs, |R|, stats, history)
cfg0.json     : configs[0] (10^3, nu 0.4) first corrector pass from the seeded
                state: |R|, stats, outer history, checksums of x
cfg0_zero.json: configs[0] first corrector pass from rest (the loaded first step)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1809_06350_b200 import CubeProblem  # noqa: E402


def first_pass(n, nu, seeded=True):
    cp = CubeProblem(n=n, nu=nu)
    P = ref.RefProblem(ref.cube_params(n, nu=nu))
    st = cp.seeded_state() if seeded else None
    if st is not None:
        P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    opts = ref.SolverOptions.from_buffer_copy(bytes(cp.solver_options()))
    return cp, P, P.newton_first_pass(opts)


def main():
    cp, P, out = first_pass(3, 0.4)
    P2 = ref.RefProblem(ref.cube_params(3, nu=0.4))
    st = cp.seeded_state()
    P2.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    rm, rp, _ = P2.assemble_residuals()
    P2.assemble_tangent()
    arrs = dict(rm=rm, rp=rp, x=out["x"], rhs=out["rhs"], history=out["history"], norm=np.array([out["norm"]]))
    for k, name in enumerate(("A", "B", "C", "D", "A_rate", "C_rate")):
        m = P2.tangent_plane(k)
        arrs[f"{name}_rowptr"], arrs[f"{name}_col"], arrs[f"{name}_val"] = m.rowptr, m.col, m.val
    np.savez_compressed(os.path.join(HERE, "cube_n3.npz"), **arrs)
    for name, seeded in (("cfg0.json", True), ("cfg0_zero.json", False)):
        cp, P, out = first_pass(10, 0.4, seeded)
        x = out["x"]
        rec = dict(n=10, nu=0.4, seeded=seeded, norm=out["norm"], stats={k: v for k, v in out["stats"].items()
                                                                         if k != "t_solve"},
                   history=[float(h) for h in out["history"]], x_norm=float(np.linalg.norm(x)),
                   x_sum=float(x.sum()), x_first=[float(v) for v in x[:8]], x_last=[float(v) for v in x[-8:]])
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(rec, f, indent=1)
    print("golden vectors written")


if __name__ == "__main__":
    main()
