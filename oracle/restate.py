"""ORACLE TEST INFRASTRUCTURE -- a numpy restatement of the reference's
Newton-step hot path, for small cases only.  Never imported by the product.

Each function cites the reference routine it restates (paths relative to
/root/reference/proj).  Element kernels are vectorised over elements with
the reference's expression order; the solver layer restates the control
flow of krylov.cpp / amg.cpp / precond.cpp literally.  The restatement is
pinned against the compiled reference (oracle/_ref) by
tests/test_oracle_cpu.py and against the committed golden vectors in
tests/golden/.  Tolerances are roundoff-level (summation order differs in
the scatter and in the Gauss-Seidel sweeps, which use triangular solves).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

QA, QB = 0.5854101966249685, 0.1381966011250105  # quadrature.hpp:20-21
BARY = np.array([[QA, QB, QB, QB], [QB, QA, QB, QB], [QB, QB, QA, QB], [QB, QB, QB, QA]])
W4 = 0.25


# ---------------------------------------------------------------------------
# materials.hpp / materials.cpp

def volumetric(mat, p):
    """CompressibleVolumetric (materials.hpp:41-71) / IncompressibleVolumetric (:74-85)."""
    if mat["incompressible"]:
        z = np.zeros_like(p)
        return mat["rho0"] + z, z, z, z
    k = mat["kappa"]
    s = np.sqrt(p * p + k * k)
    ratio = np.where(p >= 0.0, (s + p) / k, k / (s - p))
    rho = mat["rho0"] * ratio
    return rho, 1.0 / s, rho / s, -p / (s * s * s)


def _hdot(H, M):
    """ddot(H, M) per element for a global (3,3) or per-element (E,3,3) structure tensor."""
    H = np.asarray(H)
    return np.einsum("ij,eij->e", H, M) if H.ndim == 2 else np.einsum("eij,eij->e", H, M)


def iso_stress(mat, Ct):
    """NeoHookeanIsochoric::stress (materials.hpp:108) / DispersedFiberIsochoric::stress (materials.cpp:32-41)."""
    S = np.zeros_like(Ct)
    S[:, 0, 0] = S[:, 1, 1] = S[:, 2, 2] = mat["mu"]
    for H in mat.get("H", []):  # H: (3,3) global (materials.cpp:67-80) or (E,3,3) per element (cfg-3 extension)
        E = _hdot(H, Ct) - 1.0
        q = np.minimum(mat["k2"] * E * E, 500.0)
        S = S + (2.0 * mat["k1"] * E * np.exp(q))[:, None, None] * H
    return S


def iso_stress_dir(mat, Ct, dCt):
    """stress_dir (materials.hpp:109, materials.cpp:43-53)."""
    dS = np.zeros_like(Ct)
    for H in mat.get("H", []):
        E = _hdot(H, Ct) - 1.0
        q = np.minimum(mat["k2"] * E * E, 500.0)
        c = 2.0 * mat["k1"] * (1.0 + 2.0 * mat["k2"] * E * E) * np.exp(q)
        dS = dS + (c * _hdot(H, dCt))[:, None, None] * H
    return dS


def frame(mesh, mat, st, body_force):
    """make_frame (assembly.cpp:69-109) + Kinematics::from_F (materials.cpp:82-94)
    + evaluate_stress (:96-106) + per-quadrature-point volumetric data."""
    T, G = mesh["tets"], mesh["grad_n"]  # (E,4), (E,4,3)
    u = st["u"].reshape(-1, 3)[T]
    v = st["v"].reshape(-1, 3)[T]
    vd = st["vdot"].reshape(-1, 3)[T]
    pe, pde = st["p"][T], st["pdot"][T]
    F = np.eye(3)[None] + np.einsum("eai,eaI->eiI", u, G)
    J = np.linalg.det(F)
    if np.any(~(J > 0.0)):
        raise RuntimeError(f"assembly: element {int(np.nonzero(~(J > 0.0))[0][0])} inverted (J <= 0)")
    Finv = np.linalg.inv(F)
    C = np.einsum("eki,ekj->eij", F, F)
    Cinv = np.linalg.inv(C)
    Jm23 = J ** (-2.0 / 3.0)
    Ct = C * Jm23[:, None, None]
    St = iso_stress(mat, Ct)
    sc = np.einsum("eij,eij->e", St, Ct)
    Siso = St * Jm23[:, None, None] - (sc / 3.0)[:, None, None] * Cinv
    Pt = F @ Siso
    g = np.einsum("eIi,eaI->eai", Finv, G)  # F^-T G_a
    divv = np.einsum("eai,eai->e", v, g)
    gp = np.einsum("ea,eai->ei", pe, g)
    L = np.einsum("eai,eaj->eij", v, g)
    pq = pe @ BARY.T          # (E,q)
    pdq = pde @ BARY.T
    vdq = np.einsum("qa,eai->eqi", BARY, vd)
    rho, beta, drho, dbeta = volumetric(mat, pq)
    vmb = vdq - np.asarray(body_force)[None, None, :]
    res = rho[:, :, None] * J[:, None, None] * vmb + J[:, None, None] * gp[:, None, :]
    cont = J[:, None] * (beta * pdq + divv[:, None])
    pbar = (W4 * pq).sum(axis=1)
    return dict(F=F, J=J, Finv=Finv, C=C, Cinv=Cinv, Jm23=Jm23, Ct=Ct, St=St, Siso=Siso, Pt=Pt, g=g,
                divv=divv, gp=gp, L=L, pq=pq, pdq=pdq, vdq=vdq, rho=rho, beta=beta, drho=drho, dbeta=dbeta,
                vmb=vmb, res=res, cont=cont, pbar=pbar)


def assemble_residuals(mesh, dofs, mat, tau, loads, st):
    """assemble_residuals (assembly.cpp:113-185)."""
    f = frame(mesh, mat, st, loads["body_force"])
    T, G, vol = mesh["tets"], mesh["grad_n"], mesh["volume"]
    J = f["J"]
    wq = W4 * vol
    # pressure rows: sum_q wq (N_a cont_q + tau g_a . res_q)
    rp_e = np.einsum("e,qa,eq->ea", wq, BARY, f["cont"]) + \
        tau[:, None] * np.einsum("e,eai,eqi->ea", wq, f["g"], f["res"])
    rm_e = np.einsum("e,qa,eq,e,eqi->eai", wq, BARY, f["rho"], J, f["vmb"])
    PG = np.einsum("eaI,eiI->eai", G, f["Pt"])
    rm_e = rm_e + vol[:, None, None] * (PG - f["g"] * (J * f["pbar"])[:, None, None])
    rp = np.zeros(dofs["np"])
    np.add.at(rp, T, rp_e)
    rm = np.zeros(dofs["nv"])
    rows = dofs["vdof"][T]  # (E,4,3)
    m = rows >= 0
    np.add.at(rm, rows[m], rm_e[m])
    for nodes, third, h in loads["facets"]:
        for n in nodes:
            for i in range(3):
                r = dofs["vdof"][n, i]
                if r >= 0:
                    rm[r] -= third * h[i]
    return rm, rp


def ptilde_dir(f, mat, dF):
    """ptilde_dir (materials.cpp:108-129), vectorised over elements."""
    F, Finv, C, Cinv, Ct, Jm23, St, Siso = (f[k] for k in ("F", "Finv", "C", "Cinv", "Ct", "Jm23", "St", "Siso"))
    t = np.einsum("eji,eij->e", Finv, dF)
    dC = np.einsum("eki,ekj->eij", dF, F) + np.einsum("eki,ekj->eij", F, dF)
    dJm23 = -2.0 / 3.0 * Jm23 * t
    dCt = dC * Jm23[:, None, None] + dJm23[:, None, None] * C
    dS = iso_stress_dir(mat, Ct, dCt)
    dCinv = -(Cinv @ dC @ Cinv)
    sc = np.einsum("eij,eij->e", St, Ct)
    dsc = np.einsum("eij,eij->e", dS, Ct) + np.einsum("eij,eij->e", St, dCt)
    dSiso = St * dJm23[:, None, None] + dS * Jm23[:, None, None] - (dsc / 3.0)[:, None, None] * Cinv \
        - (sc / 3.0)[:, None, None] * dCinv
    return dF @ Siso + F @ dSiso


def element_tangent(mesh, mat, tau, loads, st, ts):
    """Element matrices eA, eM, eB, eC, eK, eD of assemble_tangent (assembly.cpp:207-313)."""
    f = frame(mesh, mat, st, loads["body_force"])
    G, vol = mesh["grad_n"], mesh["volume"]
    E = len(vol)
    am = ts["alpha_m"]
    chi = ts["alpha_f"] * ts["gamma"] * ts["dt"]
    fac2 = chi * chi / am
    J, g, L, gp = f["J"], f["g"], f["L"], f["gp"]
    eA = np.zeros((E, 4, 3, 4, 3))
    eM = np.zeros((E, 4, 3, 4, 3))
    eB = np.zeros((E, 4, 3, 4))
    eC = np.zeros((E, 4, 4, 3))
    eK = np.zeros((E, 4, 4, 3))
    eD = np.zeros((E, 4, 4))
    I3 = np.eye(3)
    for q in range(4):
        N = BARY[q]
        wq = W4 * vol
        rho, beta, drho, dbeta = (f[k][:, q] for k in ("rho", "beta", "drho", "dbeta"))
        vmb, res, cont, pdq = f["vmb"][:, q], f["res"][:, q], f["cont"][:, q], f["pdq"][:, q]
        NN = np.outer(N, N)
        mass = (wq * rho * J)[:, None, None] * NN[None]          # (E,a,b)
        eM += am * mass[:, :, None, :, None] * I3[None, None, :, None, :]
        eA += am * mass[:, :, None, :, None] * I3[None, None, :, None, :]
        eA += fac2 * np.einsum("e,a,ei,ebj->eaibj", wq * rho * J, N, vmb, g)
        eB += chi * (np.einsum("e,ei,ab->eaib", wq * drho * J, vmb, NN)
                     - np.einsum("e,eai,b->eaib", wq * J, g, N))
        gab = np.einsum("eai,ebi->eab", g, g)
        gavmb = np.einsum("eai,ei->ea", g, vmb)
        gbres = np.einsum("ebi,ei->eb", g, res)
        crate = am * np.einsum("e,eaj,b->eabj", wq * tau * rho * J, g, N) + chi * np.einsum("e,a,ebj->eabj", wq * J, N, g)
        eK += crate
        eC += crate
        cu = np.einsum("a,e,ebj->eabj", N, cont, g)
        Lg = np.einsum("eij,ebi->ebj", L, g)
        cu -= np.einsum("e,a,ebj->eabj", J, N, Lg)
        cu -= tau[:, None, None, None] * np.einsum("eaj,eb->eabj", g, gbres)
        ga_gp = np.einsum("eai,ei->ea", g, gp)
        cu += tau[:, None, None, None] * (np.einsum("e,ea,ebj->eabj", rho * J, gavmb, g)
                                          + np.einsum("e,ea,ebj->eabj", J, ga_gp, g)
                                          - np.einsum("e,ej,eab->eabj", J, gp, gab))
        eC += fac2 * wq[:, None, None, None] * cu
        eD += wq[:, None, None] * (am * (J * beta)[:, None, None] * NN[None]
                                   + chi * (J * dbeta * pdq)[:, None, None] * NN[None]
                                   + chi * (tau * J)[:, None, None] * (gab + drho[:, None, None] * gavmb[:, :, None] * N[None, None, :]))
    for bn in range(4):
        for j in range(3):
            dF = np.zeros((E, 3, 3))
            dF[:, j, :] = G[:, bn, :]
            dP = ptilde_dir(f, mat, dF)
            acc = np.einsum("eaI,eiI->eai", G, dP)
            acc -= (J * f["pbar"])[:, None, None] * (g * g[:, bn, j][:, None, None]
                                                     - g[:, :, j][:, :, None] * g[:, bn, :][:, None, :])
            eA[:, :, :, bn, j] += fac2 * vol[:, None, None] * acc
    return eA, eM, eB, eC, eK, eD


def assemble_tangent(mesh, dofs, mat, tau, loads, st, ts):
    """assemble_tangent (assembly.cpp:187-363) -> (A, B, C, D, A_rate, C_rate) as scipy CSR."""
    eA, eM, eB, eC, eK, eD = element_tangent(mesh, mat, tau, loads, st, ts)
    T = mesh["tets"]
    vd = dofs["vdof"][T]  # (E,4,3)
    nv, np_ = dofs["nv"], dofs["np"]
    E = T.shape[0]
    ri = np.broadcast_to(vd[:, :, :, None, None], (E, 4, 3, 4, 3))
    ci = np.broadcast_to(vd[:, None, None, :, :], (E, 4, 3, 4, 3))
    m = (ri >= 0) & (ci >= 0)
    A = sp.coo_matrix((eA[m], (ri[m], ci[m])), shape=(nv, nv)).tocsr()
    Ar = sp.coo_matrix((eM[m], (ri[m], ci[m])), shape=(nv, nv)).tocsr()
    rB = np.broadcast_to(vd[:, :, :, None], (E, 4, 3, 4))
    cB = np.broadcast_to(T[:, None, None, :], (E, 4, 3, 4))
    mB = rB >= 0
    B = sp.coo_matrix((eB[mB], (rB[mB], cB[mB])), shape=(nv, np_)).tocsr()
    rC = np.broadcast_to(T[:, :, None, None], (E, 4, 4, 3))
    cC = np.broadcast_to(vd[:, None, :, :], (E, 4, 4, 3))
    mC = cC >= 0
    Cm = sp.coo_matrix((eC[mC], (rC[mC], cC[mC])), shape=(np_, nv)).tocsr()
    Cr = sp.coo_matrix((eK[mC], (rC[mC], cC[mC])), shape=(np_, nv)).tocsr()
    rD = np.broadcast_to(T[:, :, None], (E, 4, 4))
    cD = np.broadcast_to(T[:, None, :], (E, 4, 4))
    D = sp.coo_matrix((eD.ravel(), (rD.ravel(), cD.ravel())), shape=(np_, np_)).tocsr()
    for M in (A, Ar, B, Cm, Cr, D):
        M.sort_indices()
    return A, B, Cm, D, Ar, Cr


# ---------------------------------------------------------------------------
# blocksystem.cpp / precond.cpp building blocks

def block_scaling(A, D, eps=1e-15):
    """compute_block_scaling (blocksystem.cpp:53-77)."""
    da, dd = A.diagonal(), D.diagonal()
    amax, dmax = np.abs(da).max(initial=0.0), np.abs(dd).max(initial=0.0)
    wv = np.where(np.abs(da) > eps * amax, 1.0 / np.sqrt(np.abs(da)), 1.0)
    wp = np.where(np.abs(dd) > eps * dmax, 1.0 / np.sqrt(np.abs(dd)), 1.0)
    return wv, wp


def build_shat(A, B, Cm, D, eps=1e-300):
    """build_shat (precond.cpp:10-24)."""
    da = A.diagonal()
    bad = np.nonzero(np.abs(da) < eps)[0]
    if bad.size:
        raise RuntimeError(f"build_shat: zero diagonal in momentum block at row {int(bad[0])}")
    S = (D - Cm @ sp.diags(1.0 / da) @ B).tocsr()
    S.sort_indices()
    return S


# ---------------------------------------------------------------------------
# krylov.cpp

def gmres(apply_op, apply_M, b, x, restart, max_iters, rel_tol, abs_tol=1e-50, flexible=False):
    """run_gmres (krylov.cpp:21-176); returns (x, converged, iterations, history)."""
    n = b.size
    r = b - apply_op(x)
    rnorm = np.linalg.norm(r)
    tol = max(rel_tol * rnorm, abs_tol)
    if rnorm <= tol:
        return x, True, 0, []
    m = restart
    hist, total, stag, conv = [], 0, False, False
    while total < max_iters and not stag:
        beta = np.linalg.norm(r)
        if beta == 0.0:
            break
        V = [r / beta]
        Z = []
        H = []
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        j, breakdown = 0, False
        while j < m and total < max_iters:
            if apply_M is not None:
                z = apply_M(V[j])
                if flexible:
                    Z.append(z)
                w = apply_op(z)
            else:
                w = apply_op(V[j])
            h = np.zeros(j + 2)
            for i in range(j + 1):
                h[i] = V[i] @ w
                w = w - h[i] * V[i]
            wnorm = math.sqrt(w @ w)
            corr = np.array([V[i] @ w for i in range(j + 1)])
            if wnorm > 0.0 and np.abs(corr).max() / wnorm > 1e-8:
                h[: j + 1] += corr
                for i in range(j + 1):
                    w = w - corr[i] * V[i]
                wnorm = np.linalg.norm(w)
            h[j + 1] = wnorm
            if wnorm > 1e-300:
                V.append(w / wnorm)
            else:
                breakdown = True
            for i in range(j):
                hi, hi1 = h[i], h[i + 1]
                h[i] = cs[i] * hi + sn[i] * hi1
                h[i + 1] = -sn[i] * hi + cs[i] * hi1
            den = math.hypot(h[j], h[j + 1])
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (h[j] / den, h[j + 1] / den)
            h[j], h[j + 1] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] *= cs[j]
            H.append(h)
            total += 1
            j += 1
            hist.append(abs(g[j]))
            if abs(g[j]) <= tol or breakdown:
                break
        y = np.zeros(j)
        for i in range(j - 1, -1, -1):
            s = g[i] - sum(H[k][i] * y[k] for k in range(i + 1, j))
            y[i] = s / H[i][i] if H[i][i] != 0.0 else 0.0
        if flexible and apply_M is not None:
            for i in range(j):
                x = x + y[i] * Z[i]
        else:
            t = sum((y[i] * V[i] for i in range(j)), np.zeros(n))
            x = x + (apply_M(t) if apply_M is not None else t)
        r = b - apply_op(x)
        rnorm = np.linalg.norm(r)
        if rnorm <= tol:
            conv = True
            break
        if breakdown:
            stag = True
    return x, conv, total, hist


# ---------------------------------------------------------------------------
# amg.cpp

class Amg:
    """AmgHierarchy::build / vcycle (amg.cpp:189-362), SGS smoother, dense coarse solve."""

    def __init__(self, A, block_size=1, theta=0.08, max_levels=12, coarse_max_rows=200, row_to_node=None,
                 row_comp=None):
        A = A.tocsr()
        k = block_size
        if row_to_node is None:
            node = np.arange(A.shape[0]) // k
            comp = np.arange(A.shape[0]) % k
        else:
            node, comp = np.asarray(row_to_node), np.asarray(row_comp)
        Bn = np.zeros((A.shape[0], k))
        Bn[np.arange(A.shape[0]), comp] = 1.0
        self.levels, self.fallback = [], False
        while A.shape[0] > coarse_max_rows and len(self.levels) + 1 < max_levels:
            nn = node[-1] + 1 if node.size else 0
            nbr = self._strength(A, node, nn, theta)
            agg, na = self._aggregate(nbr)
            if na <= 0 or na >= nn:
                if not self.levels:
                    d = A.diagonal()
                    self.fallback, self.fb = True, np.where(d != 0.0, 1.0 / np.where(d != 0, d, 1), 1.0)
                    return
                break
            agg_row = agg[node]
            P, Bc = self._tentative(agg_row, na, Bn, k)
            d = A.diagonal()
            invd = np.where(d != 0.0, 1.0 / np.where(d != 0, d, 1), 1.0)
            lam = self._spectral(A, invd)
            omega = 4.0 / (3.0 * max(lam, 1e-12))
            P = (P - omega * sp.diags(invd) @ (A @ P)).tocsr()
            R = P.T.tocsr()
            Ac = (R @ (A @ P)).tocsr()
            self.levels.append(dict(A=A, P=P, R=R, invd=invd))
            A, Bn = Ac, Bc
            node = np.arange(A.shape[0]) // k
        d = A.diagonal()
        self.levels.append(dict(A=A, invd=np.where(d != 0.0, 1.0 / np.where(d != 0, d, 1), 1.0)))
        self.coarse = np.linalg.pinv(A.toarray(), rcond=1e-12)

    @staticmethod
    def _strength(A, node, nn, theta):  # amg.cpp:32-81
        C = A.tocoo()
        I, J, v2 = node[C.row], node[C.col], C.data * C.data
        S = sp.coo_matrix((v2, (I, J)), shape=(nn, nn)).tocsr()
        dw = S.diagonal()
        S = S.tocoo()
        off = S.row != S.col
        i, j, s2 = S.row[off], S.col[off], S.data[off]
        ok = (dw[i] > 0) & (dw[j] > 0) & (np.sqrt(s2) > theta * np.power(dw[i] * dw[j], 0.25))
        M = sp.coo_matrix((np.ones(ok.sum()), (i[ok], j[ok])), shape=(nn, nn)).tocsr()
        M = ((M + M.T) > 0).tocsr()
        M.sort_indices()
        return [M.indices[M.indptr[r]:M.indptr[r + 1]] for r in range(nn)]

    @staticmethod
    def _aggregate(nbr):  # amg.cpp:85-117
        n = len(nbr)
        agg = -np.ones(n, dtype=np.int64)
        na = 0
        for i in range(n):
            if agg[i] >= 0 or len(nbr[i]) == 0:
                continue
            if np.any(agg[nbr[i]] >= 0):
                continue
            agg[i] = na
            agg[nbr[i]] = na
            na += 1
        for i in range(n):
            if agg[i] >= 0:
                continue
            for j in nbr[i]:
                if agg[j] >= 0:
                    agg[i] = agg[j]
                    break
        for i in range(n):
            if agg[i] < 0:
                agg[i] = na
                na += 1
        return agg, na

    @staticmethod
    def _tentative(agg_row, na, Bn, k):  # amg.cpp:122-168
        rows, cols, vals = [], [], []
        Bc = np.zeros((na * k, k))
        for a in range(na):
            rr = np.nonzero(agg_row == a)[0]
            Q = Bn[rr].copy()
            for c in range(k):
                for c2 in range(c):
                    d = Q[:, c2] @ Q[:, c]
                    Bc[a * k + c2, c] = d
                    Q[:, c] -= d * Q[:, c2]
                nrm = np.linalg.norm(Q[:, c])
                Bc[a * k + c, c] = nrm
                Q[:, c] = Q[:, c] / nrm if nrm > 1e-14 else 0.0
            for c in range(k):
                nz = Q[:, c] != 0.0
                rows += list(rr[nz])
                cols += [a * k + c] * int(nz.sum())
                vals += list(Q[nz, c])
        P = sp.coo_matrix((vals, (rows, cols)), shape=(agg_row.size, na * k)).tocsr()
        return P, Bc

    @staticmethod
    def _spectral(A, invd):  # amg.cpp:170-185
        v = np.ones(A.shape[0])
        lam = 1.0
        for _ in range(10):
            w = (A @ v) * invd
            nrm = np.linalg.norm(w)
            if nrm == 0.0:
                return 1.0
            lam = nrm / np.linalg.norm(v)
            v = w * (1.0 / nrm)
        return lam

    @staticmethod
    def _sgs(A, invd, b, z):  # amg.cpp:309-323: forward then backward, in place
        Dp = sp.diags(1.0 / invd)
        Lo, Up = sp.tril(A, -1, format="csr"), sp.triu(A, 1, format="csr")
        z = spla.spsolve_triangular((Dp + Lo).tocsr(), b - Up @ z, lower=True)
        z = spla.spsolve_triangular((Dp + Up).tocsr(), b - Lo @ z, lower=False)
        return z

    def _cycle(self, l, r):  # amg.cpp:326-352
        lv = self.levels[l]
        if l == len(self.levels) - 1:
            return self.coarse @ r
        z = self._sgs(lv["A"], lv["invd"], r, np.zeros_like(r))
        s = r - lv["A"] @ z
        z = z + lv["P"] @ self._cycle(l + 1, lv["R"] @ s)
        return self._sgs(lv["A"], lv["invd"], r, z)

    def vcycle(self, r):
        if self.fallback:
            return self.fb * r
        return self._cycle(0, r)

    def level_rows(self):
        return [lv["A"].shape[0] for lv in self.levels]


# ---------------------------------------------------------------------------
# precond.cpp

def solve_block_system(A, B, Cm, D, rhs, outer=(200, 200, 1e-6), ta=(500, 500, 1e-4), ts=(200, 200, 1e-4),
                       ti=(500, 500, 1e-2), amg_a_block=3, scale=True):
    """solve_block_system, Nested branch (precond.cpp:157-218) with ScrSolver
    (:44-99), SchurOperator (:26-42) and NestedPrecond (:101-109)."""
    nv = A.shape[0]
    if scale:
        wv, wp = block_scaling(A, D)
        A, B = sp.diags(wv) @ A @ sp.diags(wv), sp.diags(wv) @ B @ sp.diags(wp)
        Cm, D = sp.diags(wp) @ Cm @ sp.diags(wv), sp.diags(wp) @ D @ sp.diags(wp)
        b = rhs * np.concatenate([wv, wp])
    else:
        b = rhs.copy()
    A, B, Cm, D = (M.tocsr() for M in (A, B, Cm, D))
    S = build_shat(A, B, Cm, D)
    amg_a = Amg(A, block_size=amg_a_block)
    amg_s = Amg(S, block_size=1)
    stats = dict(a_solves=0, a_iters=0, s_solves=0, s_iters=0, schur_applies=0, inner_iters=0)

    def a_solve(r, cfg):
        x, _, it, _ = gmres(lambda v: A @ v, amg_a.vcycle, r, np.zeros(nv), *cfg)
        return x, it

    def schur(x):
        z, it = a_solve(B @ x, ti)
        stats["schur_applies"] += 1
        stats["inner_iters"] += it
        return D @ x - Cm @ z

    def nested(r):
        rv, rp = r[:nv], r[nv:]
        xh, it = a_solve(rv, ta)
        stats["a_solves"] += 1
        stats["a_iters"] += it
        rp2 = rp - Cm @ xh
        if ti[2] >= 1.0:
            xp, _, it, _ = gmres(lambda v: S @ v, amg_s.vcycle, rp2, np.zeros(rp.size), *ts)
        else:
            xp, _, it, _ = gmres(schur, amg_s.vcycle, rp2, np.zeros(rp.size), *ts)
        stats["s_solves"] += 1
        stats["s_iters"] += it
        xv, it = a_solve(rv - B @ xp, ta)
        stats["a_solves"] += 1
        stats["a_iters"] += it
        return np.concatenate([xv, xp])

    K = sp.bmat([[A, B], [Cm, D]]).tocsr()
    x, conv, it, hist = gmres(lambda v: K @ v, nested, b, np.zeros(b.size), *outer, flexible=True)
    if scale:
        x = x * np.concatenate([wv, wp])
    stats.update(outer_iters=it, converged=int(conv))
    return x, stats, np.array(hist)


# ---------------------------------------------------------------------------
# timeint.cpp

def step_generalized_alpha(mesh, dofs, mat, tau, loads, st, ts, solver, tol_R=1e-8, tol_A=1e-6, l_max=20,
                           prescribed=None):
    """step_generalized_alpha (timeint.cpp:40-180) on state dict `st` (updated copy returned with
    the step statistics).  `solver` = keyword arguments of solve_block_system.

    `prescribed` = (nodes, u_t) is the cfg-3 extension the reference lacks (homogeneous
    constraints only, assembly.hpp:28-30): after the predictor the iterate at those fully fixed
    nodes is set to the end-of-step displacement u_t [n,3] and to the rates the generalized-alpha
    update formulas give for it: udot = (u_t - u_n)/(gamma dt) + (gamma-1)/gamma udot_n, v = udot,
    vdot = (v - v_n)/(gamma dt) + (gamma-1)/gamma vdot_n."""
    am, af, gam, dt = ts["alpha_m"], ts["alpha_f"], ts["gamma"], ts["dt"]
    chi = af * gam * dt
    gdt = gam * dt
    nv, npn = dofs["nv"], dofs["np"]
    flat = dofs["vdof"].reshape(-1)
    idx = np.empty(nv, dtype=np.int64)
    idx[flat[flat >= 0]] = np.nonzero(flat >= 0)[0]
    keys = ("u", "udot", "p", "pdot", "v", "vdot")
    yn = {k: np.array(st[k], dtype=np.float64) for k in keys}
    cur = {k: yn[k].copy() for k in keys}
    pf = (gam - 1.0) / gam
    for k in ("udot", "pdot", "vdot"):
        cur[k] = cur[k] * pf
    if prescribed is not None:
        nodes, u_t = prescribed
        ii = (3 * np.asarray(nodes, dtype=np.int64)[:, None] + np.arange(3)[None, :]).reshape(-1)
        ut = np.asarray(u_t, dtype=np.float64).reshape(-1)
        cud = (ut - yn["u"][ii]) / gdt + pf * yn["udot"][ii]
        cur["u"][ii] = ut
        cur["udot"][ii] = cud
        cur["v"][ii] = cud
        cur["vdot"][ii] = (cud - yn["v"][ii]) / gdt + pf * yn["vdot"][ii]
    blend = lambda a, b, w: a + w * (b - a)  # noqa: E731  (timeint.cpp:31-36)
    out = dict(converged=False, newton_iters=0, res_history=[], linear=dict(
        outer_iters=0, a_solves=0, a_iters=0, s_solves=0, s_iters=0, schur_applies=0, inner_iters=0))
    norm_prev, prev = np.inf, None
    for l in range(1, l_max + 2):
        halvings = 0
        while True:
            mid = {k: blend(yn[k], cur[k], am if k in ("udot", "pdot", "vdot") else af) for k in keys}
            admissible = True
            try:
                rm, rp = assemble_residuals(mesh, dofs, mat, tau, loads, mid)
            except RuntimeError:
                admissible = False
            if admissible:
                rk = mid["udot"][idx] - mid["v"][idx]
                norm = math.sqrt(rk @ rk + rp @ rp + rm @ rm)
                if np.isfinite(norm) and norm <= 4.0 * norm_prev:
                    break
            if l == 1 or halvings >= 30:
                return cur, out
            cur = {k: blend(prev[k], cur[k], 0.5) for k in keys}
            halvings += 1
        out["res_history"].append(norm)
        norm_prev = norm
        if l == 1:
            res0 = norm
        if norm <= max(tol_R * res0, tol_A):
            out["converged"] = True
            return cur, out
        if l > l_max:
            break
        A, B, Cm, D, Ar, Cr = assemble_tangent(mesh, dofs, mat, tau, loads, mid, ts)
        rhs = np.concatenate([-rm + (A @ rk - Ar @ rk) / chi, -rp + (Cm @ rk - Cr @ rk) / chi])
        x, stats, _ = solve_block_system(A, B, Cm, D, rhs, **solver)
        for k in out["linear"]:
            out["linear"][k] += stats[k]
        out["newton_iters"] += 1
        prev = {k: cur[k].copy() for k in keys}
        dvd = x[:nv]
        dud = (chi / am) * dvd - rk / am
        cur["vdot"][idx] += dvd
        cur["v"][idx] += gdt * dvd
        cur["udot"][idx] += dud
        cur["u"][idx] += gdt * dud
        cur["pdot"] += x[nv:]
        cur["p"] += gdt * x[nv:]
    return cur, out
