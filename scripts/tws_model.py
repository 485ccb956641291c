"""Critical-path model of a tiled wavefront Gauss-Seidel sweep (offline, CPU):
rows owned by spatial tiles (one CTA each) processed in level order; an item
(tile, level) starts when the tile's previous item is done and every
cross-tile lower neighbour's item is done + lam (flag latency).

    python scripts/tws_model.py [N]
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref, restate  # noqa: E402
from paper_1809_06350_b200 import CubeProblem  # noqa: E402


def block_graph(M, B):
    coo = M.tocoo()
    nb = M.shape[0] // B
    Mb = sp.csr_matrix((np.ones(coo.nnz), (coo.row // B, coo.col // B)), shape=(nb, nb))
    Mb.sum_duplicates()
    Mb.sort_indices()
    return Mb


def levels(Mb):
    nb = Mb.shape[0]
    lev = np.zeros(nb, np.int64)
    ip, ix = Mb.indptr, Mb.indices
    for i in range(nb):
        c = ix[ip[i]:ip[i + 1]]
        c = c[c < i]
        lev[i] = lev[c].max() + 1 if c.size else 0
    return lev


def model(Mb, lev, xy, T, tau0=0.25, tau_row=0.004, lam=1.0):
    nb = Mb.shape[0]
    lo, hi = xy.min(0), xy.max(0) + 1e-12
    tx = np.minimum(((xy[:, 0] - lo[0]) / (hi[0] - lo[0]) * T).astype(int), T - 1)
    ty = np.minimum(((xy[:, 1] - lo[1]) / (hi[1] - lo[1]) * T).astype(int), T - 1)
    tile = tx * T + ty
    ip, ix = Mb.indptr, Mb.indices
    order = np.lexsort((np.arange(nb), lev))
    item_fin = {}
    tile_last = np.zeros(T * T)
    row_fin = np.zeros(nb)
    # group rows into items (tile, level) in level order
    cur = None
    for lv in range(lev.max() + 1):
        pass
    by_item = {}
    for i in order:
        by_item.setdefault((lev[i], tile[i]), []).append(i)
    n_cross = 0
    for (lv, t), rows in sorted(by_item.items()):
        start = tile_last[t]
        for i in rows:
            c = ix[ip[i]:ip[i + 1]]
            c = c[c < i]
            for j in c:
                if tile[j] != t:
                    start = max(start, row_fin[j] + lam)
                    n_cross += 1
        fin = start + tau0 + tau_row * len(rows)
        for i in rows:
            row_fin[i] = fin
        tile_last[t] = fin
    return row_fin.max(), len(by_item), n_cross


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    nu, dt = 0.5, 1e-3
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
    xyz = cp.mesh.nodes
    free = ~cp.fixed[:, 0]
    hA = restate.Amg(A, block_size=3)
    hS = restate.Amg(S, block_size=1)
    cases = [("A0", hA.levels[0]["A"], 3, xyz[free][:, :2]), ("S0", hS.levels[0]["A"], 1, xyz[:, :2])]
    # A1 aggregate centroids from the smoothed prolongator weights
    P0 = abs(hA.levels[0]["P"]).tocsc()
    fx = np.repeat(xyz[free][:, :2], 3, axis=0)
    ncol = P0.shape[1]
    w = np.asarray(P0.sum(0)).ravel()
    cen = (P0.T @ fx) / w[:, None]
    cases.append(("A1", hA.levels[1]["A"], 3, cen[::3]))
    for name, M, B, xy in cases:
        Mb = block_graph(M, B)
        lev = levels(Mb)
        print(f"{name}: rows {Mb.shape[0]} levels {lev.max() + 1}", flush=True)
        for T in (1, 2, 4, 6, 8, 12):
            for lam in (0.7, 1.5):
                cp_us, nit, ncr = model(Mb, lev, xy, T, lam=lam)
                print(f"   tiles {T}x{T} lam {lam}: critical path {cp_us:8.1f} us  items {nit}  cross edges {ncr}", flush=True)


if __name__ == "__main__":
    main()
