"""CPU tests (no GPU): the oracle pinned against the compiled reference and
the committed golden vectors, the numpy restatement against both, the mesh
host logic bitwise against the reference, and the C-ABI library (loads,
exports every declared symbol, refuses to run without a GPU).
"""
import json
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import ref
from oracle import restate as R
from paper_1809_06350_b200 import CubeProblem, _native, api
from paper_1809_06350_b200.problem import splitmix64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _setup(n, nu, seeded=True):
    cp = CubeProblem(n=n, nu=nu)
    P = ref.RefProblem(ref.cube_params(n, nu=nu))
    st = cp.seeded_state() if seeded else api.State.zeros(cp.mesh.n_nodes)
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    return cp, P, st


def _restate_problem(cp, P, st):
    m = P.mesh()
    mesh = dict(tets=m["tets"].reshape(-1, 4), grad_n=m["grad_n"].reshape(-1, 4, 3), volume=m["volume"])
    dofs = dict(vdof=m["vdof"].reshape(-1, 3), nv=P.nv, np=P.np)
    mat = dict(incompressible=cp.incompressible, rho0=cp.rho0, mu=cp.mu, kappa=cp.material.kappa)
    fn, th = P.loaded_facets()
    loads = dict(body_force=(0.0, 0.0, 0.0), facets=[(fn[i], th[i], (0.0, 0.0, -cp.load)) for i in range(len(th))])
    sd = dict(u=st.u, udot=st.udot, p=st.p, pdot=st.pdot, v=st.v, vdot=st.vdot)
    ts = dict(dt=cp.ts.dt, alpha_m=cp.ts.alpha_m, alpha_f=cp.ts.alpha_f, gamma=cp.ts.gamma)
    return mesh, dofs, mat, m["tau"], loads, sd, ts


# ---------------------------------------------------------------- golden pins
def test_reference_build_matches_golden_cfg0():
    """oracle/_ref (the reference compiled here) reproduces the committed cfg0 vectors."""
    for name, seeded in (("cfg0.json", True), ("cfg0_zero.json", False)):
        with open(os.path.join(GOLD, name)) as f:
            g = json.load(f)
        cp, P, st = _setup(10, 0.4, seeded)
        out = P.newton_first_pass(ref.SolverOptions.from_buffer_copy(bytes(cp.solver_options())))
        assert out["norm"] == pytest.approx(g["norm"], rel=1e-13)
        for k, v in g["stats"].items():
            assert out["stats"][k] == v, k
        np.testing.assert_allclose(out["history"], g["history"], rtol=1e-10)
        assert np.linalg.norm(out["x"]) == pytest.approx(g["x_norm"], rel=1e-10)
        np.testing.assert_allclose(out["x"][:8], g["x_first"], rtol=1e-9, atol=1e-9 * g["x_norm"])


def test_restatement_matches_golden_n3():
    """The numpy restatement against the golden 3^3 arrays (residuals, all six
    tangent planes incl. A_rate/C_rate, the first-pass solution)."""
    g = np.load(os.path.join(GOLD, "cube_n3.npz"))
    cp, P, st = _setup(3, 0.4)
    mesh, dofs, mat, tau, loads, sd, ts = _restate_problem(cp, P, st)
    rm, rp = R.assemble_residuals(mesh, dofs, mat, tau, loads, sd)
    assert np.max(np.abs(rm - g["rm"])) <= 1e-12 * np.max(np.abs(g["rm"]))
    assert np.max(np.abs(rp - g["rp"])) <= 1e-12 * np.max(np.abs(g["rp"]))
    planes = R.assemble_tangent(mesh, dofs, mat, tau, loads, sd, ts)
    for k, name in enumerate(("A", "B", "C", "D", "A_rate", "C_rate")):
        Mg = sp.csr_matrix((g[f"{name}_val"], g[f"{name}_col"], g[f"{name}_rowptr"]), shape=planes[k].shape)
        assert planes[k].nnz == Mg.nnz, name
        assert abs(planes[k] - Mg).max() <= 1e-12 * abs(Mg).max(), name


# ------------------------------------------------ restatement vs reference
@pytest.mark.parametrize("n,nu", [(3, 0.4), (4, 0.5)])
def test_restated_solve_matches_reference(n, nu):
    cp, P, st = _setup(n, nu)
    P.assemble_tangent()
    A, B, Cm, D = [P.tangent_plane(k).to_scipy() for k in range(4)]
    rhs = np.random.default_rng(n).uniform(-1, 1, P.nv + P.np)
    x, s, h = R.solve_block_system(A, B, Cm, D, rhs, ta=(500, 500, 1e-2), ts=(200, 200, 1e-2))
    xr, sr, hr = P.solve_tangent(rhs, ref.SolverOptions.from_buffer_copy(bytes(cp.solver_options())))
    for k in ("outer_iters", "a_solves", "a_iters", "s_solves", "s_iters", "schur_applies", "inner_iters"):
        assert abs(s[k] - sr[k]) <= 1, (k, s, sr)
    np.testing.assert_allclose(h, hr, rtol=1e-10)
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


def test_restated_gmres_matches_reference_on_random_systems():
    """krylov.cpp on random diagonally shifted systems (test_krylov.cpp:59-85 restated)."""
    rng = np.random.default_rng(12345)
    for trial in range(12):
        n = 5 + int(rng.integers(0, 60))
        Ad = rng.uniform(-1, 1, (n, n)) + n * np.eye(n)
        b = rng.uniform(-1, 1, n)
        A = ref.Csr.from_scipy(sp.csr_matrix(Ad))
        flexible = trial % 2 == 1
        xr, rr, hr = ref.gmres_csr(A, b, cfg=(min(n, 30), 400, 1e-10, 1e-50), flexible=flexible, precond=1)
        invd = 1.0 / np.diag(Ad)
        x, conv, it, h = R.gmres(lambda v: Ad @ v, lambda v: invd * v, b, np.zeros(n), min(n, 30), 400, 1e-10,
                                 flexible=flexible)
        assert conv and rr["converged"]
        assert abs(it - rr["iterations"]) <= 1
        np.testing.assert_allclose(h[:len(hr)], hr[:len(h)], rtol=1e-8, atol=1e-14 * hr[0])
        assert np.linalg.norm(x - np.linalg.solve(Ad, b)) <= 1e-8 * np.linalg.norm(np.linalg.solve(Ad, b))


def _poisson2d(n):
    T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n))
    return (sp.kron(sp.eye(n), T) + sp.kron(T, sp.eye(n))).tocsr()


def test_restated_amg_vcycle_matches_reference():
    """AmgHierarchy::build + vcycle on the 2-D Poisson model (test_amg.cpp:14-35)
    and on a 6^3 cube velocity block (multi-level, block size 3)."""
    A = _poisson2d(24)
    r = np.random.default_rng(1).uniform(-1, 1, A.shape[0])
    zr, info = ref.amg_vcycle_csr(ref.Csr.from_scipy(A), r, ref.default_amg(1))
    amg = R.Amg(A, block_size=1)
    assert amg.level_rows() == info["level_rows"]
    assert np.linalg.norm(amg.vcycle(r) - zr) <= 1e-12 * np.linalg.norm(zr)
    cp, P, st = _setup(6, 0.4)
    P.assemble_tangent()
    A = P.tangent_plane(0).to_scipy()
    r = np.random.default_rng(2).uniform(-1, 1, A.shape[0])
    zr, info = ref.amg_vcycle_csr(ref.Csr.from_scipy(A), r, ref.default_amg(3))
    amg = R.Amg(A, block_size=3)
    assert amg.level_rows() == info["level_rows"] and len(info["level_rows"]) > 1
    assert np.linalg.norm(amg.vcycle(r) - zr) <= 1e-11 * np.linalg.norm(zr)


def test_restated_shat_matches_reference():
    cp, P, st = _setup(4, 0.5)
    P.assemble_tangent()
    A, B, Cm, D = [P.tangent_plane(k) for k in range(4)]
    S = ref.build_shat(A, B, Cm, D).to_scipy()
    Sr = R.build_shat(*(m.to_scipy() for m in (A, B, Cm, D)))
    assert S.nnz == Sr.nnz
    assert abs(S - Sr).max() <= 1e-13 * abs(S).max()


def test_reference_rejects_zero_momentum_diagonal():
    """build_shat throws on |A_ii| < 1e-300 (precond.cpp:15-17, test_precond.cpp:102-109)."""
    rng = np.random.default_rng(2)
    Ad = rng.uniform(-1, 1, (4, 4)) + 6 * np.eye(4)
    Ad[2, 2] = 0.0
    Bm, Cm, Dm = (sp.csr_matrix(rng.uniform(-1, 1, s)) for s in ((4, 2), (2, 4), (2, 2)))
    with pytest.raises(RuntimeError):
        ref.build_shat(*(ref.Csr.from_scipy(m) for m in (sp.csr_matrix(Ad), Bm, Cm, Dm)))
    with pytest.raises(RuntimeError):
        R.build_shat(sp.csr_matrix(Ad), Bm, Cm, Dm)


# ------------------------------------------------------------- host logic
@pytest.mark.parametrize("n,nu", [(3, 0.4), (10, 0.4), (7, 0.5)])
def test_mesh_tau_loads_bitwise_equal_to_reference(n, nu):
    """paper_1809_06350_b200.mesh restates mesh.cpp bit for bit."""
    cp = CubeProblem(n=n, nu=nu)
    P = ref.RefProblem(ref.cube_params(n, nu=nu))
    m = P.mesh()
    assert np.array_equal(m["coords"], cp.mesh.nodes.ravel())
    assert np.array_equal(m["tets"], cp.mesh.tets.ravel())
    assert np.array_equal(m["volume"], cp.mesh.volume)
    assert np.array_equal(m["h"], cp.mesh.h)
    assert np.array_equal(m["grad_n"], cp.mesh.grad_n.ravel())
    assert np.array_equal(m["tau"], cp.tau)
    fn, th = P.loaded_facets()
    assert np.array_equal(fn, cp.load_facets) and np.array_equal(th, cp.load_third)
    assert cp.nv == P.nv and cp.np == P.np


def test_mesh_counts_and_facets():
    """test_mesh.cpp:24-43: 6 n^3 tets, (n+1)^3 nodes, 12 n^2 facets."""
    for n in (1, 2, 5):
        cp = CubeProblem(n=n)
        assert cp.mesh.n_tets == 6 * n ** 3 and cp.mesh.n_nodes == (n + 1) ** 3
        assert len(cp.mesh.facet_nodes) == 12 * n * n
        assert np.all(cp.mesh.volume > 0) and abs(cp.mesh.volume.sum() - 1.0) < 1e-12


def test_seeded_state_is_reproducible_and_bounded():
    a = splitmix64(0x1809063500, 5)
    assert a.dtype == np.uint64 and len(set(a.tolist())) == 5
    cp = CubeProblem(n=4)
    s1, s2 = cp.seeded_state(), cp.seeded_state()
    assert np.array_equal(s1.u, s2.u) and np.array_equal(s1.p, s2.p)
    assert np.abs(s1.u).max() <= 1e-3 and np.abs(s1.p).max() <= 1e2
    assert np.all(s1.u.reshape(-1, 3)[cp.fixed[:, 0]] == 0.0)


def test_gen_alpha_scalars():
    """gen_alpha_params (timeint.cpp:10-21): rho_inf 0.5 -> 5/6, 2/3, 2/3."""
    ts = api.gen_alpha_scalars(0.5, 1e-3)
    assert ts.alpha_m == pytest.approx(5 / 6) and ts.alpha_f == pytest.approx(2 / 3)
    assert ts.chi() == pytest.approx(2 / 3 * 2 / 3 * 1e-3)
    with pytest.raises(ValueError):
        api.gen_alpha_scalars(1.5, 1e-3)


# ---------------------------------------------------------------- C-ABI
def test_library_exports_every_declared_symbol():
    L = _native.lib()
    with open(os.path.join(ROOT, "include", "elastodyn_b200.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(ed_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_native.EXPORTED), declared ^ set(_native.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        api.Context(0)


def _fiber_params(n):
    """make_fiber_material (materials.cpp:67-80) with the reference test's
    fibre_test_material constants (test_assembly.cpp:34-37)."""
    p = ref.cube_params(n, nu=0.5)
    p.material, p.mu, p.k1, p.k2, p.kd, p.phi_deg, p.rho0 = 1, 2.0, 1.5, 0.8, 0.1, 40.0, 1.0
    p.incompressible = 1
    return p


def _fiber_restate_mat(p):
    phi = p.phi_deg * np.arccos(-1.0) / 180.0
    H = []
    for a in (np.array([np.cos(phi), np.sin(phi), 0.0]), np.array([np.cos(phi), -np.sin(phi), 0.0])):
        H.append(np.eye(3) * p.kd + (1.0 - 3.0 * p.kd) * np.outer(a, a))
    return dict(incompressible=True, rho0=p.rho0, mu=p.mu, kappa=0.0, k1=p.k1, k2=p.k2, H=H)


def test_restated_fiber_material_assembly_matches_reference():
    """DispersedFiberIsochoric stress and stress_dir (materials.cpp:21-53)
    through residual and tangent assembly, seeded state, 3^3 cube."""
    p = _fiber_params(3)
    P = ref.RefProblem(p)
    cp = CubeProblem(n=3, nu=0.5)
    st = cp.seeded_state()
    st.u *= 20.0  # engage the exponential fibre stiffening
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    mesh, dofs, _, tau, loads, sd, ts = _restate_problem(cp, P, st)
    mat = _fiber_restate_mat(p)
    rm, rp = R.assemble_residuals(mesh, dofs, mat, tau, loads, sd)
    rmr, rpr, _ = P.assemble_residuals()
    assert np.max(np.abs(rm - rmr)) <= 1e-12 * np.max(np.abs(rmr))
    assert np.max(np.abs(rp - rpr)) <= 1e-12 * np.max(np.abs(rpr))
    planes = R.assemble_tangent(mesh, dofs, mat, tau, loads, sd, ts)
    P.assemble_tangent()
    for k in range(6):
        Mr = P.tangent_plane(k).to_scipy()
        assert abs(planes[k] - Mr).max() <= 1e-12 * abs(Mr).max(), k


def test_reference_side_cpp_binding_builds():
    """INTEGRATION.md's reference-side C++ binding (tests/integration/first_pass_shim.cpp)
    compiles against the reference's own headers and links against the
    reference library and ours (oracle/Makefile); without a GPU it stops at
    ed_ctx_create with exit code 2 (no CPU fallback)."""
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "first_pass_shim")
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if not os.path.exists(exe):
        pytest.skip("reference headers absent and no prebuilt binding")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "no CUDA device" in r.stdout, (r.returncode, r.stdout, r.stderr)


# ------------------------------------------------ cfg-3 enablers
SOLVER_KW = dict(outer=(200, 200, 1e-6), ta=(500, 500, 1e-2), ts=(200, 200, 1e-2), ti=(500, 500, 1e-2))


def test_restated_time_step_matches_reference():
    """restate.step_generalized_alpha (timeint.cpp:40-180 restated) against the compiled reference:
    two steps of the seeded 3^3 cube -- Newton counts, residual histories, linear counts, final state.
    This pins the restated step that the prescribed-displacement GPU test compares with."""
    cp, P, st = _setup(3, 0.4)
    mesh, dofs, mat, tau, loads, sd, ts = _restate_problem(cp, P, st)
    opts = ref.SolverOptions.from_buffer_copy(bytes(cp.solver_options()))
    for k in range(2):
        r = P.step(opts, tol_r=1e-8, tol_a=1e-6, l_max=20, t_n=k * cp.dt)
        sd, g = R.step_generalized_alpha(mesh, dofs, mat, tau, loads, sd, ts, SOLVER_KW)
        assert g["converged"] == bool(r["converged"])
        assert g["newton_iters"] == r["newton_iters"]
        for key in ("outer_iters", "a_solves", "a_iters", "s_solves", "s_iters", "schur_applies", "inner_iters"):
            assert abs(g["linear"][key] - r["linear"][key]) <= 1, key
        n = len(r["res_history"])
        assert len(g["res_history"]) == n
        h0 = r["res_history"][0]
        for a, b in zip(g["res_history"], r["res_history"]):
            assert abs(a - b) <= 1e-8 * b + 1e-13 * h0
        sr = P.get_state()
        for key in ("u", "udot", "p", "pdot", "v", "vdot"):
            assert np.linalg.norm(sd[key] - sr[key]) <= 1e-8 * max(np.linalg.norm(sr[key]), 1e-300), key


def test_cylinder_mesh_is_a_conforming_tube():
    """generate_cylinder_mesh (cfg-3 geometry; the reference has boxes only, mesh.hpp:52-60):
    positive volumes summing to the polygonal tube, conforming across the periodic seam, facet tags."""
    from collections import Counter
    from paper_1809_06350_b200.mesh import FACE, circumferential_fiber_dirs, generate_cylinder_mesh
    nr, nt, nz, ri, th, L = 2, 12, 3, 1.0, 0.1, 0.5
    m = generate_cylinder_mesh(nr, nt, nz, ri, th, L)
    assert m.n_nodes == (nr + 1) * nt * (nz + 1) and m.n_tets == 6 * nr * nt * nz
    assert (m.volume > 0).all()
    ring = 0.5 * nt * np.sin(2 * np.pi / nt) * ((ri + th) ** 2 - ri ** 2)
    assert m.volume.sum() == pytest.approx(ring * L, rel=1e-13)
    np.testing.assert_allclose(m.grad_n.sum(axis=1), 0.0, atol=1e-11)
    faces = Counter(map(tuple, np.sort(m.tets[:, FACE].reshape(-1, 3), axis=1)))
    assert set(faces.values()) == {1, 2}
    assert sum(1 for c in faces.values() if c == 1) == len(m.facet_nodes)
    for tag, area in (("zmin", ring), ("zmax", ring), ("rmin", 2 * nt * ri * np.sin(np.pi / nt) * L)):
        assert m.facet_area(m.facets_with_tag(m.tag_id(tag))).sum() == pytest.approx(area, rel=1e-12)
    d = circumferential_fiber_dirs(m, 49.98)
    np.testing.assert_allclose(np.linalg.norm(d, axis=-1), 1.0, atol=1e-15)
    c = m.nodes[m.tets].mean(axis=1)
    radial = c[:, :2] / np.linalg.norm(c[:, :2], axis=1)[:, None]
    assert np.abs(np.einsum("efi,ei->ef", d[:, :, :2], radial)).max() < 1e-15  # fibres lie in the tangent plane
    np.testing.assert_allclose(d[:, 0, 2], np.sin(np.deg2rad(49.98)), atol=1e-15)
    np.testing.assert_allclose(d[:, 1, 2], -np.sin(np.deg2rad(49.98)), atol=1e-15)


def test_restated_uniform_fiber_field_equals_global_fibers():
    """A per-element fibre field whose every entry is the global structure tensor gives the
    reference-pinned global-fibre assembly (ties the extension to materials.cpp:67-80)."""
    p = _fiber_params(3)
    P = ref.RefProblem(p)
    cp = CubeProblem(n=3, nu=0.5)
    st = cp.seeded_state()
    st.u *= 20.0
    P.set_state(st.u, st.udot, st.p, st.pdot, st.v, st.vdot)
    mesh, dofs, _, tau, loads, sd, ts = _restate_problem(cp, P, st)
    mat = _fiber_restate_mat(p)
    E = mesh["tets"].shape[0]
    mat_e = dict(mat, H=[np.tile(H, (E, 1, 1)) for H in mat["H"]])
    for a, b in zip(R.assemble_residuals(mesh, dofs, mat, tau, loads, sd),
                    R.assemble_residuals(mesh, dofs, mat_e, tau, loads, sd)):
        assert np.array_equal(a, b)
    for a, b in zip(R.assemble_tangent(mesh, dofs, mat, tau, loads, sd, ts),
                    R.assemble_tangent(mesh, dofs, mat_e, tau, loads, sd, ts)):
        assert abs(a - b).max() <= 1e-15 * abs(a).max()
