"""ORACLE TEST INFRASTRUCTURE -- ctypes access to the compiled reference.

Loads ``oracle/_ref/libelastodyn_ref.so`` (the UNMODIFIED reference library
built from /root/reference/proj/src by ``oracle/Makefile``, plus our harness
``oracle/ref_harness.cpp``).  Only tests/, bench.py's cpu_baseline /
``--impl reference`` leg and ``__graft_entry__.smoke()`` may import this
module, and only as the checker -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libelastodyn_ref.so")

_i32 = C.c_int32
_f64 = C.c_double


class KrylovConfig(C.Structure):
    """krylov.hpp:64-69"""
    _fields_ = [("restart", _i32), ("max_iters", _i32), ("rel_tol", _f64), ("abs_tol", _f64)]


class AmgOptions(C.Structure):
    """amg.hpp:16-37 (+ use_dof_row_maps = set_amg_maps, driver.cpp:32-48)"""
    _fields_ = [("block_size", _i32), ("max_levels", _i32), ("coarse_max_rows", _i32),
                ("smoother", _i32), ("pre_sweeps", _i32), ("post_sweeps", _i32),
                ("smooth_prolongator", _i32), ("use_dof_row_maps", _i32),
                ("strength_theta", _f64), ("jacobi_weight", _f64)]


class SolverOptions(C.Structure):
    """BlockSolverOptions, precond.hpp:167-175"""
    _fields_ = [("precond", _i32), ("scale", _i32), ("outer", KrylovConfig), ("a", KrylovConfig),
                ("s", KrylovConfig), ("inner", KrylovConfig), ("amg_a", AmgOptions),
                ("amg_s", AmgOptions), ("eps_diag", _f64)]


class LinearStats(C.Structure):
    """precond.hpp:19-49"""
    _fields_ = [("outer_iters", C.c_int64), ("a_solves", C.c_int64), ("a_iters", C.c_int64),
                ("s_solves", C.c_int64), ("s_iters", C.c_int64), ("schur_applies", C.c_int64),
                ("inner_iters", C.c_int64), ("converged", _i32), ("pad", _i32), ("t_solve", _f64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class ProblemParams(C.Structure):
    _fields_ = [("n", _i32), ("incompressible", _i32), ("material", _i32), ("pad", _i32),
                ("edge", _f64), ("mu", _f64), ("kappa", _f64), ("rho0", _f64), ("c_m", _f64),
                ("k1", _f64), ("k2", _f64), ("kd", _f64), ("phi_deg", _f64), ("load", _f64),
                ("dt", _f64), ("rho_inf", _f64), ("body_force", _f64 * 3)]


def default_amg(block_size=1, use_maps=0) -> AmgOptions:
    return AmgOptions(block_size, 12, 200, 1, 1, 1, 1, use_maps, 0.08, 2.0 / 3.0)


def default_solver_options(**kw) -> SolverOptions:
    """BlockSolverOptions{} defaults (precond.hpp:84-86,167-175) with the cube
    problem's AMG row maps (set_amg_maps)."""
    o = SolverOptions()
    o.precond = 0
    o.scale = 1
    o.outer = KrylovConfig(200, 200, 1e-6, 1e-50)
    o.a = KrylovConfig(500, 500, 1e-4, 1e-50)
    o.s = KrylovConfig(200, 200, 1e-4, 1e-50)
    o.inner = KrylovConfig(500, 500, 1e-2, 1e-50)
    o.amg_a = default_amg(3, 1)
    o.amg_s = default_amg(1, 0)
    o.eps_diag = 1e-15
    for k, v in kw.items():
        setattr(o, k, v)
    return o


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle library missing: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        dp = C.POINTER(_f64)
        ip = C.POINTER(_i32)
        L.orc_last_error.restype = C.c_char_p
        L.orc_problem_create.restype = P
        L.orc_problem_create.argtypes = [C.POINTER(ProblemParams)]
        L.orc_problem_destroy.argtypes = [P]
        L.orc_problem_sizes.argtypes = [P, ip]
        L.orc_mesh_export.argtypes = [P, dp, ip, dp, dp, dp, dp, ip]
        L.orc_loaded_facets.argtypes = [P, ip, dp]
        L.orc_set_state.argtypes = [P] + [dp] * 6
        L.orc_get_state.argtypes = [P] + [dp] * 6
        L.orc_assemble_residuals.argtypes = [P, dp, dp, dp]
        L.orc_assemble_tangent.argtypes = [P, dp, dp]
        L.orc_tangent_dims.argtypes = [P, _i32, ip]
        L.orc_tangent_export.argtypes = [P, _i32, ip, ip, dp]
        L.orc_solve_tangent.argtypes = [P, dp, C.POINTER(SolverOptions), dp, C.POINTER(LinearStats),
                                        dp, _i32, ip]
        L.orc_newton_first_pass.argtypes = [P, C.POINTER(SolverOptions), dp, dp, dp,
                                            C.POINTER(LinearStats), dp, _i32, ip, dp]
        L.orc_step.argtypes = [P, C.POINTER(SolverOptions), _f64, _f64, _i32, _f64, ip, dp, _i32,
                               C.POINTER(LinearStats), dp]
        L.orc_solve_block_csr.argtypes = [_i32, _i32] + [ip, ip, dp] * 4 + [
            dp, C.POINTER(SolverOptions), dp, C.POINTER(LinearStats), dp, _i32, ip]
        L.orc_gmres_csr.argtypes = [_i32, ip, ip, dp, dp, dp, C.POINTER(KrylovConfig), _i32, _i32,
                                    C.POINTER(AmgOptions), dp, dp, _i32, ip]
        L.orc_amg_vcycle_csr.argtypes = [_i32, ip, ip, dp, C.POINTER(AmgOptions), ip, ip, dp, dp, ip]
        L.orc_build_shat.argtypes = [_i32, _i32] + [ip, ip, dp] * 4 + [ip, ip, ip, dp]
        _lib = L
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(_f64))


def _ip(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(_i32))


def _err():
    return lib().orc_last_error().decode()


@dataclass
class Csr:
    nrows: int
    ncols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @staticmethod
    def from_scipy(m):
        m = m.tocsr()
        m.sort_indices()
        return Csr(m.shape[0], m.shape[1], np.ascontiguousarray(m.indptr, np.int32),
                   np.ascontiguousarray(m.indices, np.int32), np.ascontiguousarray(m.data, np.float64))

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.rowptr), shape=(self.nrows, self.ncols))

    def args(self):
        return [_ip(self.rowptr), _ip(self.col), _dp(self.val)]


def cube_params(n, nu=0.4, incompressible=None, mu=3.0e4, rho0=1.0e3, c_m=1e-3, load=1.0e3,
                dt=1e-3, rho_inf=0.5, edge=1.0, body_force=(0.0, 0.0, 0.0)) -> ProblemParams:
    """The BASELINE.json cube problems (SURVEY.md §8d choices)."""
    p = ProblemParams()
    p.n = n
    if incompressible is None:
        incompressible = nu >= 0.5 - 1e-12
    p.incompressible = 1 if incompressible else 0
    p.material = 0
    p.edge = edge
    p.mu = mu
    p.kappa = 0.0 if incompressible else 2.0 * mu * (1.0 + nu) / (3.0 * (1.0 - 2.0 * nu))
    p.rho0 = rho0
    p.c_m = c_m
    p.load = load
    p.dt = dt
    p.rho_inf = rho_inf
    p.body_force = (_f64 * 3)(*body_force)
    return p


class RefProblem:
    """A reference cube problem (mesh, DofMap, material, tau, loads, state)."""

    def __init__(self, params: ProblemParams):
        self.params = params
        self.h = lib().orc_problem_create(C.byref(params))
        if not self.h:
            raise RuntimeError(_err())
        s = np.zeros(6, np.int32)
        lib().orc_problem_sizes(self.h, _ip(s))
        self.n_nodes, self.n_tets, self.nv, self.np, self.n_loaded, self.n_facets = map(int, s)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_problem_destroy(self.h)
            self.h = None

    def mesh(self):
        N, E = self.n_nodes, self.n_tets
        out = dict(coords=np.zeros(3 * N), tets=np.zeros(4 * E, np.int32), volume=np.zeros(E),
                   h=np.zeros(E), grad_n=np.zeros(12 * E), tau=np.zeros(E),
                   vdof=np.zeros(3 * N, np.int32))
        lib().orc_mesh_export(self.h, _dp(out["coords"]), _ip(out["tets"]), _dp(out["volume"]),
                              _dp(out["h"]), _dp(out["grad_n"]), _dp(out["tau"]), _ip(out["vdof"]))
        return out

    def loaded_facets(self):
        nodes = np.zeros(3 * self.n_loaded, np.int32)
        third = np.zeros(self.n_loaded)
        lib().orc_loaded_facets(self.h, _ip(nodes), _dp(third))
        return nodes.reshape(-1, 3), third

    def set_state(self, u, udot, p, pdot, v, vdot):
        arrs = [np.ascontiguousarray(a, np.float64) for a in (u, udot, p, pdot, v, vdot)]
        lib().orc_set_state(self.h, *[_dp(a) for a in arrs])

    def get_state(self):
        N = self.n_nodes
        arrs = [np.zeros(3 * N), np.zeros(3 * N), np.zeros(N), np.zeros(N), np.zeros(3 * N),
                np.zeros(3 * N)]
        lib().orc_get_state(self.h, *[_dp(a) for a in arrs])
        return dict(zip(("u", "udot", "p", "pdot", "v", "vdot"), arrs))

    def assemble_residuals(self):
        rm, rp, t = np.zeros(self.nv), np.zeros(self.np), np.zeros(1)
        rc = lib().orc_assemble_residuals(self.h, _dp(rm), _dp(rp), _dp(t))
        if rc:
            raise RuntimeError(_err())
        return rm, rp, float(t[0])

    def assemble_tangent(self, ts=None):
        t = np.zeros(1)
        tsa = None if ts is None else np.asarray(ts, np.float64)
        rc = lib().orc_assemble_tangent(self.h, _dp(tsa), _dp(t))
        if rc:
            raise RuntimeError(_err())
        return float(t[0])

    def tangent_plane(self, which) -> Csr:
        """which: 0 A, 1 B, 2 C, 3 D, 4 A_rate, 5 C_rate (TangentBlocks, assembly.hpp:78-82)"""
        d = np.zeros(3, np.int32)
        if lib().orc_tangent_dims(self.h, which, _ip(d)):
            raise RuntimeError("no tangent assembled")
        nr, nc, nnz = map(int, d)
        m = Csr(nr, nc, np.zeros(nr + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz))
        lib().orc_tangent_export(self.h, which, _ip(m.rowptr), _ip(m.col), _dp(m.val))
        return m

    def solve_tangent(self, rhs, opts=None, hist_cap=4096):
        opts = opts or default_solver_options()
        n = self.nv + self.np
        x, st, hist, hl = np.zeros(n), LinearStats(), np.zeros(hist_cap), np.zeros(1, np.int32)
        rc = lib().orc_solve_tangent(self.h, _dp(np.ascontiguousarray(rhs, np.float64)), C.byref(opts),
                                     _dp(x), C.byref(st), _dp(hist), hist_cap, _ip(hl))
        if rc:
            raise RuntimeError(_err())
        return x, st.as_dict(), hist[: int(hl[0])].copy()

    def newton_first_pass(self, opts=None, hist_cap=4096):
        opts = opts or default_solver_options()
        n = self.nv + self.np
        x, rhs, nrm = np.zeros(n), np.zeros(n), np.zeros(1)
        st, hist, hl, times = LinearStats(), np.zeros(hist_cap), np.zeros(1, np.int32), np.zeros(4)
        rc = lib().orc_newton_first_pass(self.h, C.byref(opts), _dp(x), _dp(rhs), _dp(nrm),
                                         C.byref(st), _dp(hist), hist_cap, _ip(hl), _dp(times))
        if rc:
            raise RuntimeError(_err())
        return dict(x=x, rhs=rhs, norm=float(nrm[0]), stats=st.as_dict(),
                    history=hist[: int(hl[0])].copy(), times=times.copy())

    def step(self, opts=None, tol_r=1e-8, tol_a=1e-6, l_max=20, t_n=0.0, res_cap=64):
        """step_generalized_alpha (timeint.cpp:40-180) on the stored state."""
        opts = opts or default_solver_options()
        info, hist = np.zeros(3, np.int32), np.zeros(res_cap)
        st, ta = LinearStats(), np.zeros(1)
        rc = lib().orc_step(self.h, C.byref(opts), tol_r, tol_a, l_max, t_n, _ip(info), _dp(hist), res_cap,
                            C.byref(st), _dp(ta))
        if rc:
            raise RuntimeError(_err())
        return dict(converged=int(info[0]), newton_iters=int(info[1]), res_history=hist[: min(int(info[2]), res_cap)].copy(),
                    linear=st.as_dict(), t_assembly=float(ta[0]))


def gmres_csr(A: Csr, b, x0=None, cfg=(50, 500, 1e-6, 1e-50), flexible=False, precond=0,
              amg: AmgOptions | None = None, hist_cap=100000):
    n = A.nrows
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64)
    kcfg = KrylovConfig(*cfg)
    amg = amg or default_amg()
    res, hist, hl = np.zeros(4), np.zeros(hist_cap), np.zeros(1, np.int32)
    rc = lib().orc_gmres_csr(n, *A.args(), _dp(np.ascontiguousarray(b, np.float64)), _dp(x),
                             C.byref(kcfg), int(flexible), precond, C.byref(amg), _dp(res), _dp(hist),
                             hist_cap, _ip(hl))
    if rc:
        raise RuntimeError(_err())
    return x, dict(converged=bool(res[0]), iterations=int(res[1]), initial_norm=res[2],
                   final_norm=res[3]), hist[: int(hl[0])].copy()


def amg_vcycle_csr(A: Csr, r, amg: AmgOptions | None = None, row_to_node=None, row_comp=None):
    amg = amg or default_amg()
    z = np.zeros(A.nrows)
    info = np.zeros(18, np.int32)
    rtn = None if row_to_node is None else np.ascontiguousarray(row_to_node, np.int32)
    rc_ = None if row_comp is None else np.ascontiguousarray(row_comp, np.int32)
    rc = lib().orc_amg_vcycle_csr(A.nrows, *A.args(), C.byref(amg), _ip(rtn), _ip(rc_),
                                  _dp(np.ascontiguousarray(r, np.float64)), _dp(z), _ip(info))
    if rc:
        raise RuntimeError(_err())
    nl = int(info[0])
    return z, dict(n_levels=nl, fallback=bool(info[1]), level_rows=[int(v) for v in info[2:2 + nl]])


def solve_block_csr(A: Csr, B: Csr, Cm: Csr, D: Csr, rhs, opts: SolverOptions, hist_cap=4096):
    nv, np_ = A.nrows, D.nrows
    x, st, hist, hl = np.zeros(nv + np_), LinearStats(), np.zeros(hist_cap), np.zeros(1, np.int32)
    rc = lib().orc_solve_block_csr(nv, np_, *A.args(), *B.args(), *Cm.args(), *D.args(),
                                   _dp(np.ascontiguousarray(rhs, np.float64)), C.byref(opts), _dp(x),
                                   C.byref(st), _dp(hist), hist_cap, _ip(hl))
    if rc:
        raise RuntimeError(_err())
    return x, st.as_dict(), hist[: int(hl[0])].copy()


def build_shat(A: Csr, B: Csr, Cm: Csr, D: Csr) -> Csr:
    nv, np_ = A.nrows, D.nrows
    dims = np.zeros(1, np.int32)
    args = [nv, np_, *A.args(), *B.args(), *Cm.args(), *D.args()]
    if lib().orc_build_shat(*args, _ip(dims), None, None, None):
        raise RuntimeError(_err())
    nnz = int(dims[0])
    S = Csr(np_, np_, np.zeros(np_ + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz))
    if lib().orc_build_shat(*args, _ip(dims), _ip(S.rowptr), _ip(S.col), _dp(S.val)):
        raise RuntimeError(_err())
    return S
