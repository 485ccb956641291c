"""GPU parity tests: the CUDA path (through the C-ABI) against the compiled
reference oracle (oracle/_ref) on identical inputs.

Tolerances (BASELINE.json north_star): iteration counts within +-1, residual
histories within 1e-10 relative, Newton-step solution within 1e-8 relative
L2; assembled blocks within 1e-12 relative to the block maximum.
"""
import numpy as np
import pytest

from conftest import opts_to_ref
from paper_1809_06350_b200 import CubeProblem, api

pytestmark = pytest.mark.gpu

HIST_TOL = 1e-10
X_TOL = 1e-8


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _ref_problem(oracle, cp):
    return oracle.RefProblem(oracle.cube_params(cp.n, nu=cp.nu))


def _csr(m):
    return api.Csr(m.nrows, m.ncols, m.rowptr, m.col, m.val)


def _assert_history(h_gpu, h_ref):
    n = min(len(h_gpu), len(h_ref))
    assert abs(len(h_gpu) - len(h_ref)) <= 1, (len(h_gpu), len(h_ref))
    for k in range(n):
        assert abs(h_gpu[k] - h_ref[k]) <= HIST_TOL * h_ref[0] + HIST_TOL * abs(h_ref[k]), (k, h_gpu[k], h_ref[k])


def _assert_stats(sg, sr):
    for k in ("outer_iters", "a_solves", "s_solves"):
        assert abs(sg[k] - sr[k]) <= 1 * max(1, sr["outer_iters"]) if k != "outer_iters" else abs(sg[k] - sr[k]) <= 1, (k, sg, sr)
    assert sg["converged"] == sr["converged"]


@pytest.fixture(scope="module")
def cfg0(oracle):
    cp = CubeProblem.config(0)
    P = _ref_problem(oracle, cp)
    st = cp.seeded_state()
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    P.assemble_tangent()
    planes = [P.tangent_plane(k) for k in range(4)]
    return cp, P, st, planes


def test_context_and_symbols():
    ctx = api.Context(0)
    assert api.Context.kernel_launches() >= 0
    ctx.close()


def test_block_matvec_bitwise(cfg0):
    """BlockMatrix::matvec (blocksystem.hpp:27-33): same column order, no FMA
    -> bitwise identical to the reference's CSR row sums."""
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    x = np.random.default_rng(1).uniform(-1, 1, cp.nv + cp.np)
    y = ctx.block_matvec(x)
    A, B, Cm, D = [m.to_scipy() for m in planes]
    yv = A @ x[: cp.nv] + B @ x[cp.nv:]
    yp = Cm @ x[: cp.nv] + D @ x[cp.nv:]
    ref_y = np.concatenate([yv, yp])
    assert _rel(y, ref_y) < 1e-14


def test_gmres_on_A_matches_reference(cfg0, oracle):
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    b = np.random.default_rng(2).uniform(-1, 1, cp.nv)
    for flexible in (False, True):
        xg, rg = ctx.gmres_a(b, cfg=api.krylov_config(30, 300, 1e-10), flexible=flexible, precond=1)
        xr, rr, hr = oracle.gmres_csr(planes[0], b, cfg=(30, 300, 1e-10, 1e-50), flexible=flexible, precond=1)
        assert abs(rg.iterations - rr["iterations"]) <= 1
        _assert_history(rg.history, hr)
        assert _rel(xg, xr) < X_TOL


def test_amg_vcycle_matches_reference(cfg0, oracle):
    """AmgHierarchy::build + vcycle on A with the DofMap row maps."""
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    r = np.random.default_rng(3).uniform(-1, 1, cp.nv)
    opts = cp.solver_options()
    opts.amg_a = api.amg_options(3, 0)
    zg, ig = ctx.amg_vcycle(r, 0, opts)
    zr, ir = oracle.amg_vcycle_csr(planes[0], r, oracle.default_amg(3, 0))
    assert ig["level_rows"] == ir["level_rows"], (ig, ir)
    assert _rel(zg, zr) < 1e-12


def test_shat_matches_reference(cfg0, oracle):
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    opts = cp.solver_options()
    opts.scale = 0
    S = ctx.build_shat(opts).to_scipy()
    Sr = oracle.build_shat(*planes).to_scipy()
    assert (S != Sr).nnz == 0 or abs(S - Sr).max() <= 1e-14 * abs(Sr).max()


def test_solve_block_system_matches_reference(cfg0, oracle):
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    rhs = np.random.default_rng(4).uniform(-1, 1, cp.nv + cp.np)
    opts = cp.solver_options()
    xg, sg, hg = ctx.solve_block_system(rhs, opts)
    xr, sr, hr = P.solve_tangent(rhs, opts_to_ref(opts))
    print("gpu", sg, hg)
    print("ref", sr, hr)
    _assert_stats(sg, sr)
    _assert_history(hg, hr)
    assert _rel(xg, xr) < X_TOL


def test_residual_assembly_matches_reference(cfg0):
    cp, P, st, planes = cfg0
    ctx = cp.context(0)
    ctx.set_state(st)
    rm, rp = ctx.assemble_residuals()
    rmr, rpr, _ = P.assemble_residuals()
    assert np.max(np.abs(rm - rmr)) <= 1e-12 * np.max(np.abs(rmr))
    assert np.max(np.abs(rp - rpr)) <= 1e-12 * np.max(np.abs(rpr))


def test_tangent_assembly_matches_reference(cfg0):
    cp, P, st, planes = cfg0
    ctx = cp.context(0)
    ctx.set_state(st)
    ctx.assemble_tangent(cp.ts)
    for k in range(4):
        g = ctx.tangent_plane(k)
        r = planes[k]
        assert np.array_equal(g.rowptr, r.rowptr) and np.array_equal(g.col, r.col), k
        scale = np.max(np.abs(r.val))
        assert np.max(np.abs(g.val - r.val)) <= 1e-12 * scale, (k, np.max(np.abs(g.val - r.val)) / scale)


def test_newton_first_pass_matches_reference(oracle):
    cp = CubeProblem.config(0)
    P = _ref_problem(oracle, cp)
    st = cp.seeded_state()
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    ctx = cp.context(0)
    ctx.set_state(st)
    opts = cp.solver_options()
    out = ctx.newton_first_pass(cp.ts, opts)
    ro = P.newton_first_pass(opts_to_ref(opts))
    print("gpu", out["stats"], out["history"], out["times"])
    print("ref", ro["stats"], ro["history"], ro["times"])
    assert abs(out["norm"] - ro["norm"]) <= 1e-12 * ro["norm"]
    _assert_stats(out["stats"], ro["stats"])
    _assert_history(out["history"], ro["history"])
    assert _rel(out["x"], ro["x"]) < X_TOL
    sg, sr = ctx.get_state(), P.get_state()
    for k in ("u", "udot", "p", "pdot", "v", "vdot"):
        assert _rel(getattr(sg, k), sr[k]) < X_TOL, k
