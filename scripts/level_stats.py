"""Level-schedule statistics of the reference's SA-AMG hierarchies (CPU, via
the oracle): rows, blocks/row, Gauss-Seidel dependency levels, and the
number of <=32-scalar-row groups a blocked sweep needs.

    python scripts/level_stats.py N [NU] [DT]
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref, restate  # noqa: E402
from paper_1809_06350_b200 import CubeProblem  # noqa: E402


def levels_of(M, B):
    """Forward level schedule of the block-row graph."""
    nb = M.shape[0] // B
    Mb = sp.csr_matrix((np.ones(M.nnz), M.indices // B, M.indptr[::B][: nb + 1] if B > 1 else M.indptr),
                       shape=(nb, nb)) if B == 1 else None
    if B > 1:
        coo = M.tocoo()
        Mb = sp.csr_matrix((np.ones(coo.nnz), (coo.row // B, coo.col // B)), shape=(nb, nb))
    Mb.sum_duplicates()
    lev = np.zeros(nb, np.int64)
    ip, ix = Mb.indptr, Mb.indices
    for i in range(nb):
        c = ix[ip[i]:ip[i + 1]]
        c = c[c < i]
        lev[i] = lev[c].max() + 1 if c.size else 0
    return Mb, lev


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    nu = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    dt = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
    cp = CubeProblem(n=n, nu=nu, dt=dt)
    P = ref.RefProblem(ref.cube_params(n, nu=nu, dt=dt))
    st = cp.seeded_state()
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    P.assemble_tangent()
    A, B, C, D = (P.tangent_plane(k).to_scipy() for k in range(4))
    wv, wp = restate.block_scaling(A, D)
    A = (sp.diags(wv) @ A @ sp.diags(wv)).tocsr()
    B = (sp.diags(wv) @ B @ sp.diags(wp)).tocsr()
    C = (sp.diags(wp) @ C @ sp.diags(wv)).tocsr()
    D = (sp.diags(wp) @ D @ sp.diags(wp)).tocsr()
    S = restate.build_shat(A, B, C, D)
    for name, M, bs in (("A", A, 3), ("S", S, 1)):
        h = restate.Amg(M, block_size=bs)
        for li, L in enumerate(h.levels):
            Ml = L["A"]
            Mb, lev = levels_of(Ml, bs)
            nl = int(lev.max()) + 1
            order = np.argsort(lev, kind="stable")
            gr = 32 // bs
            groups = 0
            cnt = np.bincount(lev)
            for c in cnt:
                groups += -(-int(c) // gr)
            print(f"{name}{li}: rows {Ml.shape[0]:8d} block_rows {Mb.shape[0]:7d} nnz/row {Ml.nnz / Ml.shape[0]:8.1f} "
                  f"levels {nl:6d} rows/level {Mb.shape[0] / nl:8.1f} groups(level-split,{gr}) {groups:6d}", flush=True)


if __name__ == "__main__":
    main()
