"""Offline analysis of the Gauss-Seidel dependency structure of the 40^3
hierarchies (CPU, via the oracle restatement): per level operator, the
level schedule and, for groups of g consecutive dependency levels, the size
of the dense in-group triangular inverse and of the external lower coupling.

    python scripts/sweep_analysis.py [N] [NU] [DT]
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref, restate  # noqa: E402
from paper_1809_06350_b200 import CubeProblem  # noqa: E402


def block_levels(M, B):
    coo = M.tocoo()
    nb = M.shape[0] // B
    Mb = sp.csr_matrix((np.ones(coo.nnz), (coo.row // B, coo.col // B)), shape=(nb, nb))
    Mb.sum_duplicates()
    lev = np.zeros(nb, np.int64)
    ip, ix = Mb.indptr, Mb.indices
    for i in range(nb):
        c = ix[ip[i]:ip[i + 1]]
        c = c[c < i]
        lev[i] = lev[c].max() + 1 if c.size else 0
    return Mb, lev


def analyse(name, M, B):
    Mb, lev = block_levels(M, B)
    nl = int(lev.max()) + 1
    nb = Mb.shape[0]
    print(f"{name}: block rows {nb} blocks {Mb.nnz} levels {nl} rows/level {nb / nl:.1f} blocks/row {Mb.nnz / nb:.1f}")
    # how far back (in levels) do lower neighbours reach?
    coo = Mb.tocoo()
    low = coo.col < coo.row
    back = lev[coo.row[low]] - lev[coo.col[low]]
    print(f"   lower-neighbour level distance: mean {back.mean():.2f} p50 {np.median(back):.0f} p90 "
          f"{np.percentile(back, 90):.0f} max {back.max()}")
    for g in (2, 4, 8, 16):
        grp = lev // g
        ng = int(grp.max()) + 1
        cnt = np.bincount(grp, minlength=ng) * B
        tinv = float(np.sum(cnt.astype(np.float64) * (cnt + 1) / 2) * 8)
        ext = np.zeros(ng)
        r, c = coo.row[low], coo.col[low]
        x = grp[r] != grp[c]
        # distinct external columns per group
        key = np.unique(grp[r[x]].astype(np.int64) * nb + c[x])
        ext = np.bincount(key // nb, minlength=ng) * B
        w = float(np.sum(cnt.astype(np.float64) * ext) * 8)
        print(f"   g={g:2d}: steps {ng:4d} max rows {cnt.max():6d} Tinv {tinv / 1e6:8.1f} MB  ext cols mean {ext.mean():7.0f}"
              f" max {ext.max():6d}  W {w / 1e6:8.1f} MB")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    nu = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    dt = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
    cp = CubeProblem(n=n, nu=nu, dt=dt)
    P = ref.RefProblem(ref.cube_params(n, nu=nu, dt=dt))
    st = cp.seeded_state()
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    P.assemble_tangent()
    A, Bm, Cm, D = (P.tangent_plane(k).to_scipy() for k in range(4))
    wv, wp = restate.block_scaling(A, D)
    A = (sp.diags(wv) @ A @ sp.diags(wv)).tocsr()
    Bm = (sp.diags(wv) @ Bm @ sp.diags(wp)).tocsr()
    Cm = (sp.diags(wp) @ Cm @ sp.diags(wv)).tocsr()
    D = (sp.diags(wp) @ D @ sp.diags(wp)).tocsr()
    S = restate.build_shat(A, Bm, Cm, D)
    out = {}
    for nm, M, bs in (("A", A, 3), ("S", S, 1)):
        h = restate.Amg(M, block_size=bs)
        for li, L in enumerate(h.levels[:-1]):
            analyse(f"{nm}{li}", L["A"], bs)
            out[f"{nm}{li}"] = L["A"]
    np.savez_compressed(f"/tmp/levels_{n}.npz", **{k: v.data for k, v in out.items()},
                        **{k + "_ip": v.indptr for k, v in out.items()}, **{k + "_ix": v.indices for k, v in out.items()})


if __name__ == "__main__":
    main()
