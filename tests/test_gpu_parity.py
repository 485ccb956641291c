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


def _assert_history(h_gpu, h_ref, floor=0.0):
    """Outer residual estimates within 1e-10 relative; `floor` is the
    roundoff floor of a solve that converged to machine precision (estimates
    below ~1e-13 of the right-hand side carry no information)."""
    n = min(len(h_gpu), len(h_ref))
    assert abs(len(h_gpu) - len(h_ref)) <= 1, (len(h_gpu), len(h_ref))
    for k in range(n):
        tol = HIST_TOL * h_ref[0] + HIST_TOL * abs(h_ref[k]) + floor
        assert abs(h_gpu[k] - h_ref[k]) <= tol, (k, h_gpu[k], h_ref[k])


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


def test_device_amg_setup_equals_host_restatement(cfg0, monkeypatch):
    """The GPU hierarchy build (amg_device.cu) and the host restatement
    (amg_host.cpp) produce identical hierarchies -> identical V-cycles."""
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    r = np.random.default_rng(5).uniform(-1, 1, cp.nv)
    opts = cp.solver_options()
    monkeypatch.setenv("ED_HOST_AMG", "1")
    zh, ih = ctx.amg_vcycle(r, 0, opts)
    monkeypatch.delenv("ED_HOST_AMG")
    zd, idv = ctx.amg_vcycle(r, 0, opts)
    assert ih["level_rows"] == idv["level_rows"]
    assert np.array_equal(zh, zd)
    zh, ih = None, None
    monkeypatch.setenv("ED_HOST_AMG", "1")
    sh, i1 = ctx.amg_vcycle(r[: cp.np], 1, opts)
    monkeypatch.delenv("ED_HOST_AMG")
    sd, i2 = ctx.amg_vcycle(r[: cp.np], 1, opts)
    assert i1["level_rows"] == i2["level_rows"] and np.array_equal(sh, sd)


def _random_saddle(nv, np_, seed, d_shift=1.0):
    """random_saddle of test_precond.cpp:43-67 (numpy generator)."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (nv, nv)) + (nv + 2.0) * np.eye(nv)
    B = rng.uniform(-1, 1, (nv, np_))
    Cm = rng.uniform(-1, 1, (np_, nv))
    D = rng.uniform(-1, 1, (np_, np_)) + d_shift * (np_ + 2.0) * np.eye(np_)
    return A, B, Cm, D


@pytest.mark.parametrize("nv,np_,seed,d_shift", [(14, 8, 9, 1.0), (12, 4, 10, 0.0), (30, 11, 3, 1.0)])
def test_solve_block_system_random_saddle(oracle, nv, np_, seed, d_shift):
    """SolveBlockSystemMatchesDirect / HandlesZeroPressureDiagonalBlock
    (test_precond.cpp:228-306): GPU vs reference vs dense LU."""
    import scipy.sparse as sp
    A, B, Cm, D = _random_saddle(nv, np_, seed, d_shift)
    if d_shift == 0.0:
        D = np.zeros_like(D)
    K = np.block([[A, B], [Cm, D]])
    b = np.random.default_rng(seed + 100).uniform(-1, 1, nv + np_)
    blocks = [api.Csr.from_scipy(sp.csr_matrix(M)) for M in (A, B, Cm, D)]
    if d_shift == 0.0:
        blocks[3] = api.Csr(np_, np_, np.zeros(np_ + 1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    opts = api.block_solver_options()
    opts.outer = api.krylov_config(500, 500, 1e-10)
    opts.amg_a = api.amg_options(1, 0)
    if d_shift == 0.0:
        for c in (opts.a, opts.s, opts.inner):
            c.rel_tol = 1e-10
    ctx = api.Context(0)
    ctx.set_block_system(*blocks)
    xg, sg, hg = ctx.solve_block_system(b, opts)
    ref_blocks = [oracle.Csr(m.nrows, m.ncols, m.rowptr, m.col, m.val) for m in blocks]
    xr, sr, hr = oracle.solve_block_csr(*ref_blocks, b, opts_to_ref(opts))
    x_lu = np.linalg.solve(K, b)
    assert sg["converged"] and sr["converged"]
    assert np.max(np.abs(xg - x_lu)) <= 1e-5 * np.linalg.norm(x_lu)
    _assert_stats(sg, sr)
    _assert_history(hg, hr, floor=1e-13 * np.linalg.norm(b))
    assert _rel(xg, xr) < X_TOL


def test_cfg1_newton_first_pass_matches_reference(oracle):
    """BASELINE configs[1]: 40^3 cube, fully incompressible, seeded state."""
    cp = CubeProblem.config(1)
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


def test_fiber_material_assembly_matches_reference(oracle):
    """DispersedFiberIsochoric (HGO-type fibres, materials.cpp:8-53) on the
    device: residuals and all four planes vs the reference, strained state."""
    n = 4
    p = oracle.cube_params(n, nu=0.5)
    p.material, p.mu, p.k1, p.k2, p.kd, p.phi_deg, p.rho0, p.incompressible = 1, 2.0, 1.5, 0.8, 0.1, 40.0, 1.0, 1
    P = oracle.RefProblem(p)
    cp = CubeProblem(n=n, nu=0.5)
    st = cp.seeded_state()
    st.u *= 20.0
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    m = P.mesh()
    ctx = api.Context(0)
    ctx.set_mesh(cp.mesh, m["tau"])
    ctx.build_dofs(cp.fixed)
    ctx.set_material(api.dispersed_fiber(2.0, 1.5, 0.8, 0.1, 40.0, 1.0))
    ctx.set_loads((0.0, 0.0, 0.0), cp.load_facets, cp.load_third, cp.traction_h())
    ctx.set_state(st)
    rm, rp = ctx.assemble_residuals()
    rmr, rpr, _ = P.assemble_residuals()
    assert np.max(np.abs(rm - rmr)) <= 1e-12 * np.max(np.abs(rmr))
    assert np.max(np.abs(rp - rpr)) <= 1e-12 * np.max(np.abs(rpr))
    ctx.assemble_tangent(cp.ts)
    P.assemble_tangent()
    for k in range(4):
        g, r = ctx.tangent_plane(k), P.tangent_plane(k)
        assert np.array_equal(g.col, r.col)
        assert np.max(np.abs(g.val - r.val)) <= 1e-12 * np.max(np.abs(r.val)), k


def test_element_inversion_raises(oracle):
    """ThrowsOnElementInversion (test_assembly.cpp:271-286): collapse x=1 onto x=0."""
    cp = CubeProblem(n=2, nu=0.4)
    ctx = cp.context(0)
    st = api.State.zeros(cp.mesh.n_nodes)
    st.u.reshape(-1, 3)[cp.mesh.nodes[:, 0] > 0.5, 0] = -2.0
    ctx.set_state(st)
    with pytest.raises(api.ElementInversion, match="inverted"):
        ctx.assemble_residuals()
    with pytest.raises(api.ElementInversion):
        ctx.assemble_tangent(cp.ts)


@pytest.mark.parametrize("n", [16, 20])
def test_mid_cube_vcycle_and_newton_pass(oracle, n):
    """Operators big enough for the cluster-ring sweep (>= 4096 block rows)
    and a collapsed dense coarse tail: one V-cycle on A (1e-12 against the
    reference's sequential sweeps) and a whole first Newton pass."""
    cp = CubeProblem(n=n, nu=0.5)
    P = _ref_problem(oracle, cp)
    st = cp.seeded_state()
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    P.assemble_tangent()
    planes = [P.tangent_plane(k) for k in range(4)]
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    r = np.random.default_rng(11).uniform(-1, 1, cp.nv)
    opts = cp.solver_options()
    opts.amg_a = api.amg_options(3, 0)
    zg, ig = ctx.amg_vcycle(r, 0, opts)
    zr, ir = oracle.amg_vcycle_csr(planes[0], r, oracle.default_amg(3, 0))
    assert ig["level_rows"] == ir["level_rows"], (ig, ir)
    assert _rel(zg, zr) < 1e-12
    ctx.close()
    ctx = cp.context(0)
    ctx.set_state(st)
    opts = cp.solver_options()
    out = ctx.newton_first_pass(cp.ts, opts)
    ro = P.newton_first_pass(opts_to_ref(opts))
    assert abs(out["norm"] - ro["norm"]) <= 1e-12 * ro["norm"]
    _assert_stats(out["stats"], ro["stats"])
    _assert_history(out["history"], ro["history"])
    assert _rel(out["x"], ro["x"]) < X_TOL


@pytest.mark.parametrize("case", ["cfg0_rest_5steps", "n8_seeded_2steps"])
def test_time_steps_match_reference(oracle, case):
    """step_generalized_alpha (timeint.cpp:40-180) -- Newton loop, growth
    guard, convergence test -- over BASELINE configs[0] (5 steps from rest) and
    a seeded 8^3 incompressible cube (2 steps): Newton counts, residual
    histories, accumulated linear counts and the final state against the
    reference."""
    if case.startswith("cfg0"):
        cp, steps, st = CubeProblem.config(0), 5, None
    else:
        cp, steps = CubeProblem(n=8, nu=0.5), 2
        st = cp.seeded_state()
    P = _ref_problem(oracle, cp)
    ctx = cp.context(0)
    if st is not None:
        P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
        ctx.set_state(st)
    opts = cp.solver_options()
    for k in range(steps):
        g = ctx.step(cp.ts, opts, tol_r=1e-8, tol_a=1e-6, l_max=20)
        r = P.step(opts_to_ref(opts), tol_r=1e-8, tol_a=1e-6, l_max=20, t_n=k * cp.dt)
        print(k, "gpu", g["newton_iters"], g["res_history"], g["linear"])
        print(k, "ref", r["newton_iters"], r["res_history"], r["linear"])
        assert g["converged"] == r["converged"]
        assert abs(g["newton_iters"] - r["newton_iters"]) <= 1
        h0 = r["res_history"][0]
        n = min(len(g["res_history"]), len(r["res_history"]))
        for i in range(n):
            assert abs(g["res_history"][i] - r["res_history"][i]) <= 1e-8 * h0 + 1e-6 * r["res_history"][i], (k, i)
        sg, sr = ctx.get_state(), P.get_state()
        for key in ("u", "udot", "p", "pdot", "v", "vdot"):
            assert _rel(getattr(sg, key), sr[key]) < 1e-7, (k, key, _rel(getattr(sg, key), sr[key]))


@pytest.mark.parametrize("kind", [1, 2, 3, 4])
def test_solve_block_system_variants(cfg0, oracle, kind):
    """solve_block_system's other PrecondKinds (precond.cpp:157-218): Simple
    (FGMRES + SimplePrecond, :111-155), Ilu0 (GMRES + Ilu0Precond on the
    monolithic matrix), Jacobi (GMRES + monolithic JacobiPrecond) and None
    (plain GMRES) against the reference."""
    cp, P, st, planes = cfg0
    ctx = api.Context(0)
    ctx.set_block_system(*[_csr(m) for m in planes])
    rhs = np.random.default_rng(40 + kind).uniform(-1, 1, cp.nv + cp.np)
    opts = cp.solver_options()
    opts.precond = kind
    if kind in (2, 3, 4):
        opts.outer = api.krylov_config(100, 400, 1e-4)
    xg, sg, hg = ctx.solve_block_system(rhs, opts)
    xr, sr, hr = P.solve_tangent(rhs, opts_to_ref(opts))
    print(kind, "gpu", sg, len(hg), "ref", sr, len(hr))
    _assert_stats(sg, sr)
    _assert_history(hg, hr)
    assert _rel(xg, xr) < X_TOL
