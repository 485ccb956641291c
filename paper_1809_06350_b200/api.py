"""Reference-shaped host API over the C-ABI (the drop-in surface for Python).

Names, argument meaning and error behaviour mirror the reference C++ API:
``assemble_residuals`` / ``assemble_tangent`` (assembly.hpp:88-94),
``solve_block_system`` (precond.hpp:182-183), ``gmres`` / ``fgmres``
(krylov.hpp:81-88), ``AmgHierarchy::build`` + ``vcycle`` (amg.hpp:39-74),
``build_shat`` (precond.hpp:54), ``BlockMatrix::matvec`` (blocksystem.hpp:27).
Errors raise the reference's exception types: :class:`ElementInversion`
(a ``RuntimeError``, materials.hpp:16-19), ``RuntimeError`` for a zero
momentum diagonal (precond.cpp:15-17), ``ValueError`` for invalid arguments
(``std::invalid_argument``).  Every call runs on the GPU; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .mesh import Mesh


class ElementInversion(RuntimeError):
    """materials.hpp:16-19"""


class Unsupported(RuntimeError):
    """Outside this build's scope (ED_UNSUPPORTED)."""


def _raise(ctx_ptr, rc, what=""):
    if rc == N.ED_OK:
        return
    msg = N.lib().ed_last_error(ctx_ptr).decode() if ctx_ptr else what
    if rc == N.ED_ELEMENT_INVERSION:
        raise ElementInversion(msg)
    if rc == N.ED_ZERO_DIAGONAL:
        raise RuntimeError(msg)
    if rc == N.ED_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == N.ED_UNSUPPORTED:
        raise Unsupported(msg)
    raise RuntimeError(f"elastodyn_b200 error {rc}: {msg}")


def krylov_config(restart=50, max_iters=500, rel_tol=1e-6, abs_tol=1e-50) -> N.KrylovConfig:
    """KrylovConfig defaults (krylov.hpp:64-69)."""
    return N.KrylovConfig(restart, max_iters, rel_tol, abs_tol)


def amg_options(block_size=1, use_dof_row_maps=0, **kw) -> N.AmgOptions:
    """AmgOptions defaults (amg.hpp:16-37)."""
    o = N.AmgOptions(block_size, 12, 200, 1, 1, 1, 1, use_dof_row_maps, 0.08, 2.0 / 3.0)
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def block_solver_options(**kw) -> N.BlockSolverOptions:
    """BlockSolverOptions{} (precond.hpp:84-86,167-175).  The velocity AMG
    carries the DofMap row grouping (set_amg_maps, driver.cpp:32-48)."""
    o = N.BlockSolverOptions()
    o.precond = 0
    o.scale = 1
    o.outer = krylov_config(200, 200, 1e-6)
    o.a = krylov_config(500, 500, 1e-4)
    o.s = krylov_config(200, 200, 1e-4)
    o.inner = krylov_config(500, 500, 1e-2)
    o.amg_a = amg_options(3, 1)
    o.amg_s = amg_options(1, 0)
    o.eps_diag = 1e-15
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def gen_alpha_scalars(rho_inf, dt) -> N.TimeScalars:
    """gen_alpha_params (timeint.cpp:10-21) -> TimeScalars."""
    if rho_inf < 0.0 or rho_inf > 1.0:
        raise ValueError("gen_alpha_params: rho_inf must lie in [0, 1]")
    am = 0.5 * (3.0 - rho_inf) / (1.0 + rho_inf)
    af = 1.0 / (1.0 + rho_inf)
    return N.TimeScalars(dt, am, af, af)


def neo_hookean(mu, kappa, rho0) -> N.Material:
    """make_neo_hookean_material (materials.cpp:55-65)."""
    m = N.Material()
    m.kind, m.incompressible, m.rho0, m.mu, m.kappa = 0, 0, rho0, mu, kappa
    return m


def incompressible_neo_hookean(mu, rho0) -> N.Material:
    """IncompressibleVolumetric + NeoHookeanIsochoric (driver.cpp:332-339)."""
    m = N.Material()
    m.kind, m.incompressible, m.rho0, m.mu, m.kappa = 0, 1, rho0, mu, 0.0
    return m


def dispersed_fiber(mu, k1, k2, kd, phi_deg, rho0, kappa=None) -> N.Material:
    """make_fiber_material (materials.cpp:67-80); structure tensors H_i =
    kd I + (1 - 3 kd) a_i (x) a_i (materials.cpp:8-19)."""
    if kd < 0.0 or kd > 1.0 / 3.0:
        raise ValueError("kd must be in [0, 1/3]")
    phi = phi_deg * np.arccos(-1.0) / 180.0
    dirs = [np.array([np.cos(phi), np.sin(phi), 0.0]), np.array([np.cos(phi), -np.sin(phi), 0.0])]
    m = N.Material()
    m.kind, m.rho0, m.mu, m.k1, m.k2 = 1, rho0, mu, k1, k2
    m.incompressible, m.kappa = (1, 0.0) if kappa is None else (0, kappa)
    for H, a in zip((m.h1, m.h2), dirs):
        I = np.eye(3).ravel()
        outer = np.outer(a, a).ravel()
        vals = I * kd + (1.0 - 3.0 * kd) * outer
        for k in range(9):
            H[k] = vals[k]
    return m


def fiber_structure_tensors(dirs, kd) -> np.ndarray:
    """H = kd I + (1 - 3 kd) a (x) a (materials.cpp:8-19) for an array of unit
    directions dirs[..., 3] -> [..., 3, 3]."""
    dirs = np.asarray(dirs, dtype=np.float64)
    return np.eye(3) * kd + (1.0 - 3.0 * kd) * dirs[..., :, None] * dirs[..., None, :]


def wave_speed(mat: N.Material) -> float:
    """Material::wave_speed (materials.hpp:148-152)."""
    if mat.incompressible:
        return float(np.sqrt(mat.mu / mat.rho0))
    return float(np.sqrt((mat.kappa + 4.0 * mat.mu / 3.0) / mat.rho0))


def compute_tau(mesh: Mesh, mat: N.Material, c_m=1e-3) -> np.ndarray:
    """compute_tau (assembly.cpp:41-50)."""
    c = wave_speed(mat)
    return c_m * mesh.h / (c * mat.rho0)


@dataclass
class State:
    """State (assembly.hpp:31-37): full-length nodal arrays."""
    u: np.ndarray
    udot: np.ndarray
    p: np.ndarray
    pdot: np.ndarray
    v: np.ndarray
    vdot: np.ndarray

    @staticmethod
    def zeros(n_nodes):
        z3, z1 = lambda: np.zeros(3 * n_nodes), lambda: np.zeros(n_nodes)
        return State(z3(), z3(), z1(), z1(), z3(), z3())

    def arrays(self):
        return [N.f64(a) for a in (self.u, self.udot, self.p, self.pdot, self.v, self.vdot)]


@dataclass
class Csr:
    """CsrMatrix (csr.hpp:13-46) view."""
    nrows: int
    ncols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.rowptr), shape=(self.nrows, self.ncols))

    @staticmethod
    def from_scipy(m):
        m = m.tocsr()
        m.sort_indices()
        return Csr(m.shape[0], m.shape[1], N.i32(m.indptr), N.i32(m.indices), N.f64(m.data))


@dataclass
class SolveResult:
    converged: bool
    iterations: int
    initial_norm: float
    final_norm: float
    history: np.ndarray = field(default_factory=lambda: np.zeros(0))


class Context:
    """One GPU context holding a problem (mesh, DofMap, material, loads,
    state) and its device-resident block system."""

    def __init__(self, device: int = 0):
        p = C.c_void_p()
        rc = N.lib().ed_ctx_create(device, C.byref(p))
        if rc != N.ED_OK or not p.value:
            raise RuntimeError("ed_ctx_create failed: no usable CUDA device (there is no CPU fallback)")
        self._p = p
        self.nv = self.np = 0
        self.n_nodes = 0

    def close(self):
        if getattr(self, "_p", None) is not None and self._p.value:
            N.lib().ed_ctx_destroy(self._p)
            self._p = None

    def __del__(self):
        self.close()

    def _chk(self, rc):
        _raise(self._p, rc)

    # ---- problem definition -------------------------------------------
    def set_mesh(self, mesh: Mesh, tau: np.ndarray):
        self.mesh = mesh
        self.n_nodes = mesh.n_nodes
        self._chk(N.lib().ed_mesh_upload(self._p, mesh.n_nodes, mesh.n_tets, N.ip(N.i32(mesh.tets.ravel())),
                                         N.dp(N.f64(mesh.grad_n.ravel())), N.dp(N.f64(mesh.volume)),
                                         N.dp(N.f64(tau))))

    def build_dofs(self, fixed: np.ndarray):
        """DofMap::build (assembly.cpp:11-27); fixed is (N, 3) bool."""
        fx = np.ascontiguousarray(np.asarray(fixed, dtype=np.uint8).reshape(-1))
        if fx.size != 3 * self.n_nodes:
            raise ValueError("DofMap: constraint table size mismatch")
        nv, np_ = C.c_int32(), C.c_int32()
        self._chk(N.lib().ed_dofs_build(self._p, fx.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(nv),
                                        C.byref(np_)))
        self.nv, self.np = nv.value, np_.value
        self.fixed = np.asarray(fixed, dtype=bool).reshape(-1, 3)

    def set_material(self, mat: N.Material):
        self._chk(N.lib().ed_set_material(self._p, C.byref(mat)))

    def set_loads(self, body_force=(0.0, 0.0, 0.0), facet_nodes=None, facet_third=None, facet_h=None):
        """Loads (assembly.hpp:42-50): one entry per (traction, facet) in order."""
        bf = N.f64(body_force)
        if facet_nodes is None or len(facet_nodes) == 0:
            self._chk(N.lib().ed_set_loads(self._p, N.dp(bf), 0, None, None, None))
            return
        fn, th, fh = N.i32(np.asarray(facet_nodes).reshape(-1)), N.f64(facet_third), N.f64(np.asarray(facet_h).reshape(-1))
        self._chk(N.lib().ed_set_loads(self._p, N.dp(bf), len(th), N.ip(fn), N.dp(th), N.dp(fh)))

    def set_fiber_field(self, h):
        """Per-element fibre structure tensors [E, 2, 3, 3] (None: the material's global ones).
        Extension of materials.cpp:67-80 (global fibre constants) for local fibre frames."""
        if h is None:
            self._chk(N.lib().ed_set_fiber_field(self._p, 0, None))
            return
        hh = N.f64(np.asarray(h).reshape(-1))
        self._chk(N.lib().ed_set_fiber_field(self._p, hh.size // 18, N.dp(hh)))

    def set_prescribed_displacement(self, nodes, u):
        """End-of-step displacement [n, 3] of fully fixed nodes for the next step() call
        (inhomogeneous Dirichlet; the reference has homogeneous constraints only, assembly.hpp:28-30)."""
        nn = N.i32(np.asarray(nodes).reshape(-1))
        uu = N.f64(np.asarray(u).reshape(-1))
        if uu.size != 3 * nn.size:
            raise ValueError("prescribed displacement: 3 values per node")
        self._chk(N.lib().ed_set_prescribed_displacement(self._p, nn.size, N.ip(nn) if nn.size else None,
                                                         N.dp(uu) if nn.size else None))

    def set_state(self, s: State):
        arrs = s.arrays()
        self._chk(N.lib().ed_state_upload(self._p, *[N.dp(a) for a in arrs]))

    def get_state(self) -> State:
        s = State.zeros(self.n_nodes)
        arrs = [s.u, s.udot, s.p, s.pdot, s.v, s.vdot]
        self._chk(N.lib().ed_state_download(self._p, *[N.dp(a) for a in arrs]))
        return s

    # ---- assembly (assembly.hpp:88-94) ---------------------------------
    def assemble_residuals(self):
        rm, rp, bad = np.zeros(self.nv), np.zeros(self.np), C.c_int32(-1)
        self._chk(N.lib().ed_assemble_residuals(self._p, N.dp(rm), N.dp(rp), C.byref(bad)))
        return rm, rp

    def assemble_tangent(self, ts: N.TimeScalars, rk=None):
        bad = C.c_int32(-1)
        rka = None if rk is None else N.f64(rk)
        self._chk(N.lib().ed_assemble_tangent(self._p, C.byref(ts), N.dp(rka), C.byref(bad)))

    def tangent_plane(self, which) -> Csr:
        """Plane of the current block system: 0 A, 1 B, 2 C, 3 D."""
        d = np.zeros(3, np.int32)
        self._chk(N.lib().ed_tangent_export(self._p, which, N.ip(d), None, None, None))
        nr, nc, nnz = map(int, d)
        m = Csr(nr, nc, np.zeros(nr + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz))
        self._chk(N.lib().ed_tangent_export(self._p, which, N.ip(d), N.ip(m.rowptr), N.ip(m.col), N.dp(m.val)))
        return m

    def foldin(self):
        fv, fp = np.zeros(self.nv), np.zeros(self.np)
        self._chk(N.lib().ed_foldin_download(self._p, N.dp(fv), N.dp(fp)))
        return fv, fp

    # ---- block system from CSR (BlockMatrix) ---------------------------
    def set_block_system(self, A: Csr, B: Csr, Cm: Csr, D: Csr):
        self.nv, self.np = A.nrows, D.nrows
        self._keep = [N.i32(m.rowptr) for m in (A, B, Cm, D)] + [N.i32(m.col) for m in (A, B, Cm, D)] + \
                     [N.f64(m.val) for m in (A, B, Cm, D)]
        rp, cc, vv = self._keep[0:4], self._keep[4:8], self._keep[8:12]
        args = []
        for k in range(4):
            args += [N.ip(rp[k]), N.ip(cc[k]), N.dp(vv[k])]
        self._chk(N.lib().ed_block_system_upload(self._p, A.nrows, D.nrows, *args))

    # ---- solve (precond.hpp:182-183) -----------------------------------
    def solve_block_system(self, rhs, opts: N.BlockSolverOptions | None = None, hist_cap=4096):
        """Returns (x, stats dict, outer residual history)."""
        opts = opts or block_solver_options()
        n = self.nv + self.np
        x, st, h, hl = np.zeros(n), N.LinearStats(), np.zeros(hist_cap), C.c_int32(0)
        self._chk(N.lib().ed_solve_block_system(self._p, N.dp(N.f64(rhs)), N.dp(x), C.byref(opts), C.byref(st),
                                                N.dp(h), hist_cap, C.byref(hl)))
        return x, st.as_dict(), h[: hl.value].copy()

    def newton_first_pass(self, ts: N.TimeScalars, opts: N.BlockSolverOptions | None = None, hist_cap=4096):
        """First corrector pass of step_generalized_alpha (timeint.cpp:54-176)."""
        opts = opts or block_solver_options()
        n = self.nv + self.np
        x, nrm, st = np.zeros(n), C.c_double(0.0), N.LinearStats()
        h, hl, pt = np.zeros(hist_cap), C.c_int32(0), N.PhaseTimes()
        self._chk(N.lib().ed_newton_first_pass(self._p, C.byref(ts), C.byref(opts), N.dp(x), C.byref(nrm),
                                               C.byref(st), N.dp(h), hist_cap, C.byref(hl), C.byref(pt)))
        return dict(x=x, norm=nrm.value, stats=st.as_dict(), history=h[: hl.value].copy(), times=pt.as_dict())

    def step(self, ts: N.TimeScalars, opts: N.BlockSolverOptions | None = None, tol_r=1e-8, tol_a=1e-6, l_max=20,
             res_cap=64):
        """step_generalized_alpha (timeint.cpp:40-180): one time step from the
        current state (which becomes y_{n+1}); StepStats + accumulated LinearStats."""
        opts = opts or block_solver_options()
        nl = N.NonlinearConfig(tol_r, tol_a, l_max, 0)
        st, lin, h = N.StepStats(), N.LinearStats(), np.zeros(res_cap)
        self._chk(N.lib().ed_step_generalized_alpha(self._p, C.byref(ts), C.byref(nl), C.byref(opts), C.byref(st),
                                                    C.byref(lin), N.dp(h), res_cap))
        out = st.as_dict()
        out["res_history"] = h[: min(st.n_res, res_cap)].copy()
        out["linear"] = lin.as_dict()
        return out

    # ---- debug / parity --------------------------------------------------
    def block_matvec(self, x):
        y = np.zeros(self.nv + self.np)
        self._chk(N.lib().ed_block_matvec(self._p, N.dp(N.f64(x)), N.dp(y)))
        return y

    def coupled_matvec(self, x, opts: N.BlockSolverOptions | None = None):
        """K x on the solver's working copy through the coupled 4x4 BSR operator and through the planes."""
        opts = opts or block_solver_options()
        xx = N.f64(x)
        y1, y2 = np.zeros(xx.size), np.zeros(xx.size)
        self._chk(N.lib().ed_coupled_matvec(self._p, C.byref(opts), N.dp(xx), N.dp(y1), N.dp(y2)))
        return y1, y2

    def gmres_a(self, b, x0=None, cfg=None, flexible=False, precond=0, amg=None, hist_cap=100000):
        """gmres/fgmres (krylov.cpp:180-192) on the A block; precond 0 none,
        1 JacobiPrecond (krylov.hpp:51-62), 2 AmgPrecond (amg.hpp:76-89)."""
        cfg = cfg or krylov_config()
        n = self.nv
        x = np.zeros(n) if x0 is None else N.f64(x0).copy()
        res, h, hl = N.SolveResult(), np.zeros(hist_cap), C.c_int32(0)
        amg_p = C.byref(amg) if amg is not None else None
        self._chk(N.lib().ed_gmres_a(self._p, N.dp(N.f64(b)), N.dp(x), C.byref(cfg), int(flexible), precond, amg_p,
                                     C.byref(res), N.dp(h), hist_cap, C.byref(hl)))
        return x, SolveResult(bool(res.converged), res.iterations, res.initial_norm, res.final_norm,
                              h[: hl.value].copy())

    def amg_vcycle(self, r, which=0, opts=None):
        """AmgHierarchy::build + vcycle on A (which=0) or S_hat (which=1)."""
        opts = opts or block_solver_options()
        n = self.nv if which == 0 else self.np
        z, info = np.zeros(n), np.zeros(18, np.int32)
        self._chk(N.lib().ed_amg_vcycle(self._p, which, C.byref(opts), N.dp(N.f64(r)), N.dp(z), N.ip(info)))
        nl = int(info[0])
        return z, dict(n_levels=nl, fallback=bool(info[1]), level_rows=[int(v) for v in info[2:2 + nl]])

    def build_shat(self, opts=None) -> Csr:
        """build_shat (precond.cpp:10-24) on the solver's (scaled) system."""
        opts = opts or block_solver_options()
        d = np.zeros(3, np.int32)
        self._chk(N.lib().ed_shat_export(self._p, C.byref(opts), N.ip(d), None, None, None))
        nr, nc, nnz = map(int, d)
        m = Csr(nr, nc, np.zeros(nr + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz))
        self._chk(N.lib().ed_shat_export(self._p, C.byref(opts), N.ip(d), N.ip(m.rowptr), N.ip(m.col), N.dp(m.val)))
        return m

    def spmv_bytes(self):
        cb, ab = C.c_double(), C.c_double()
        self._chk(N.lib().ed_spmv_bytes(self._p, C.byref(cb), C.byref(ab)))
        return cb.value, ab.value

    def block_matvec_device(self, d_x_ptr, d_y_ptr, n_rep):
        ms = C.c_float()
        self._chk(N.lib().ed_block_matvec_device(self._p, C.c_void_p(d_x_ptr), C.c_void_p(d_y_ptr), n_rep,
                                                 C.byref(ms)))
        return ms.value

    def solve_block_system_device(self, d_rhs_ptr, d_x_ptr, opts=None, hist_cap=4096):
        opts = opts or block_solver_options()
        st, h, hl = N.LinearStats(), np.zeros(hist_cap), C.c_int32(0)
        self._chk(N.lib().ed_solve_block_system_device(self._p, C.c_void_p(d_rhs_ptr), C.c_void_p(d_x_ptr),
                                                       C.byref(opts), C.byref(st), N.dp(h), hist_cap, C.byref(hl)))
        return st.as_dict(), h[: hl.value].copy()

    def state_save(self):
        self._chk(N.lib().ed_state_save(self._p))

    def state_restore(self):
        self._chk(N.lib().ed_state_restore(self._p))

    def timer_start(self):
        self._chk(N.lib().ed_timer(self._p, 0, None))

    def timer_stop(self) -> float:
        ms = C.c_float()
        self._chk(N.lib().ed_timer(self._p, 1, C.byref(ms)))
        return ms.value

    def bench_kernels(self, opts=None, n_rep=10):
        """Device-timed hot kernels: {name: (ms per launch, algorithmic bytes)}."""
        opts = opts or block_solver_options()
        out = np.zeros(8)
        self._chk(N.lib().ed_bench_kernels(self._p, C.byref(opts), n_rep, N.dp(out)))
        names = ("coupled_spmv", "a_spmv", "sgs_fwd_fine", "shat_spmv")
        return {k: (float(out[2 * i]), float(out[2 * i + 1])) for i, k in enumerate(names)}

    def bench_assembly(self, ts, n_rep=5):
        """Device-timed residual and tangent assembly (after assemble_tangent):
        ms, algorithmic bytes, the FP64 FMA peak GFLOP/s."""
        out = np.zeros(8)
        self._chk(N.lib().ed_bench_assembly(self._p, C.byref(ts), n_rep, N.dp(out)))
        return {"residual_ms": float(out[0]), "residual_bytes": float(out[1]), "tangent_ms": float(out[2]),
                "tangent_bytes": float(out[3]), "fp64_peak_gflops": float(out[4]), "elements": int(out[5]),
                "plane_bytes": float(out[6]), "k4_bytes": float(out[7])}

    def kernel_accounting(self, on: bool):
        """Bracket every sparse launch with CUDA events (bench.py roofline)."""
        self._chk(N.lib().ed_kernel_accounting(self._p, int(on)))

    def kernel_account(self):
        """{"kernel@level": (launches, total ms, total algorithmic bytes)} since accounting was switched on."""
        n = C.c_int(0)
        self._chk(N.lib().ed_kernel_account_count(self._p, C.byref(n)))
        out = {}
        for i in range(n.value):
            name = C.create_string_buffer(128)
            la, ms, by = N._i64(0), C.c_double(0.0), C.c_double(0.0)
            self._chk(N.lib().ed_kernel_account_get(self._p, i, name, 128, C.byref(la), C.byref(ms), C.byref(by)))
            out[name.value.decode()] = (int(la.value), float(ms.value), float(by.value))
        return out

    @staticmethod
    def kernel_launches():
        return int(N.lib().ed_kernel_launches(None))
