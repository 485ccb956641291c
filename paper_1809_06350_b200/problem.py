"""The BASELINE.json cube problems on the GPU path.

Unit cube [0, L]^3 meshed n^3 x 6 tets, bottom face z = 0 fully clamped,
dead traction (0, 0, -load) on top-face facets whose centroid lies in the
central quarter [L/4, 3L/4]^2, Neo-Hookean mu = 3e4 Pa with the Gibbs
volumetric energy (kappa from nu; nu = 0.5 -> incompressible), rho0 = 1e3,
c_m = 1e-3, generalized-alpha rho_inf = 0.5, dt = 1e-3, solver FGMRES(200)
outer 1e-6 with SCR a/s/inner rel 1e-2.  Seeded states use one splitmix64
stream (seed 0x1809063500) drawn u, v, p in that order.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import api
from .mesh import Mesh, circumferential_fiber_dirs, generate_cube_mesh, generate_cylinder_mesh

CONFIGS = {
    0: dict(n=10, nu=0.4, steps=5, seeded=False),
    1: dict(n=40, nu=0.5, steps=3, seeded=False),
    2: dict(n=100, nu=0.45, steps=1, seeded=True),
    4: dict(n=160, nu=0.5, steps=2, seeded=True),
}

SEED = 0x1809063500


def kappa_from_nu(mu, nu):
    """materials.hpp:160-163"""
    return 2.0 * mu * (1.0 + nu) / (3.0 * (1.0 - 2.0 * nu))


def splitmix64(seed: int, count: int) -> np.ndarray:
    """count successive outputs of splitmix64 starting from `seed`."""
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(bits: np.ndarray, lo: float, hi: float) -> np.ndarray:
    return lo + (hi - lo) * ((bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)


@dataclass
class CubeProblem:
    n: int
    nu: float = 0.4
    mu: float = 3.0e4
    rho0: float = 1.0e3
    c_m: float = 1e-3
    load: float = 1.0e3
    dt: float = 1e-3
    rho_inf: float = 0.5
    edge: float = 1.0

    def __post_init__(self):
        L = self.edge
        self.mesh: Mesh = generate_cube_mesh(self.n, L)
        tol = 1e-9 * L
        self.fixed = np.zeros((self.mesh.n_nodes, 3), dtype=bool)
        self.fixed[self.mesh.nodes[:, 2] < tol] = True
        self.incompressible = self.nu >= 0.5 - 1e-12
        if self.incompressible:
            self.material = api.incompressible_neo_hookean(self.mu, self.rho0)
        else:
            self.material = api.neo_hookean(self.mu, kappa_from_nu(self.mu, self.nu), self.rho0)
        self.tau = api.compute_tau(self.mesh, self.material, self.c_m)
        zmax = self.mesh.tag_id("zmax")

        def quarter(c):
            return ((c[:, 0] >= 0.25 * L - tol) & (c[:, 0] <= 0.75 * L + tol) & (c[:, 1] >= 0.25 * L - tol)
                    & (c[:, 1] <= 0.75 * L + tol))

        self.mesh.retag_facets(zmax, quarter, "top_load")
        fl = self.mesh.facets_with_tag(self.mesh.tag_id("top_load"))
        self.load_facets = self.mesh.facet_nodes[fl]
        self.load_third = self.mesh.facet_area(fl) / 3.0
        self.ts = api.gen_alpha_scalars(self.rho_inf, self.dt)
        self.n_free = int((~self.fixed[:, 0]).sum())
        self.nv = 3 * self.n_free
        self.np = self.mesh.n_nodes

    @staticmethod
    def config(cfg: int) -> "CubeProblem":
        c = CONFIGS[cfg]
        return CubeProblem(n=c["n"], nu=c["nu"])

    def seeded_state(self, seed: int = SEED) -> api.State:
        """u, v ~ U[-1e-3, 1e-3], p ~ U[-1e2, 1e2], rates 0,
        fixed components zero."""
        N = self.mesh.n_nodes
        bits = splitmix64(seed, 7 * N)
        s = api.State.zeros(N)
        s.u = uniform(bits[: 3 * N], -1e-3, 1e-3)
        s.v = uniform(bits[3 * N: 6 * N], -1e-3, 1e-3)
        s.p = uniform(bits[6 * N: 7 * N], -1e2, 1e2)
        fx = self.fixed.reshape(-1)
        s.u[fx] = 0.0
        s.v[fx] = 0.0
        return s

    def solver_options(self, **kw):
        """Outer FGMRES 1e-6; SCR a/s/inner rel 1e-2 (BASELINE cfg 0 / SURVEY §8d)."""
        o = api.block_solver_options(**kw)
        o.outer = api.krylov_config(200, 200, 1e-6)
        o.a = api.krylov_config(500, 500, 1e-2)
        o.s = api.krylov_config(200, 200, 1e-2)
        o.inner = api.krylov_config(500, 500, 1e-2)
        return o

    def traction_h(self):
        return np.tile(np.array([0.0, 0.0, -self.load]), (len(self.load_third), 1))

    def context(self, device: int = 0) -> api.Context:
        ctx = api.Context(device)
        ctx.set_mesh(self.mesh, self.tau)
        ctx.build_dofs(self.fixed)
        ctx.set_material(self.material)
        ctx.set_loads((0.0, 0.0, 0.0), self.load_facets, self.load_third, self.traction_h())
        return ctx


@dataclass
class CylinderProblem:
    """BASELINE configs[3]: tensile test of an anisotropic arterial wall.

    Thick-walled cylinder (inner radius 1 cm, wall 0.1 cm, length 1 cm, SI units),
    n_r x n_theta x n_z hexes split into six tets; fully incompressible
    Neo-Hookean ground matrix mu with two fibre families at +-phi to the
    circumferential direction in the local tangent plane (per-element structure
    tensors H = kd I + (1 - 3 kd) a (x) a, the reference's DispersedFiberIsochoric
    energy, materials.cpp:21-53, evaluated with the element's own a); the z = 0
    end is clamped, the z = L end carries a prescribed axial displacement ramped
    linearly to `stretch` L over `n_steps` generalized-alpha steps.

    The reference cannot run this configuration (boxes only, global fibres,
    homogeneous constraints), so it is pinned by oracle/restate.py alone.
    Choices BASELINE leaves open: kd = 0 (no dispersion), no fibre tension switch
    (as in the reference's energy), both ends fully clamped in all three
    components (nodes here are fully free or fully fixed), dt = 1e-3.
    """
    n_r: int = 8
    n_theta: int = 128
    n_z: int = 64
    r_in: float = 1.0e-2
    thickness: float = 1.0e-3
    length: float = 1.0e-2
    mu: float = 3.0e4
    k1: float = 2.3632e5
    k2: float = 0.8393
    kd: float = 0.0
    phi_deg: float = 49.98
    rho0: float = 1.0e3
    c_m: float = 1e-3
    stretch: float = 0.10
    n_steps: int = 10
    dt: float = 1e-3
    rho_inf: float = 0.5

    def __post_init__(self):
        self.mesh: Mesh = generate_cylinder_mesh(self.n_r, self.n_theta, self.n_z, self.r_in, self.thickness,
                                                 self.length)
        kz = np.arange(self.mesh.n_nodes) // ((self.n_r + 1) * self.n_theta)
        self.bottom_nodes = np.nonzero(kz == 0)[0].astype(np.int32)
        self.top_nodes = np.nonzero(kz == self.n_z)[0].astype(np.int32)
        self.fixed = np.zeros((self.mesh.n_nodes, 3), dtype=bool)
        self.fixed[self.bottom_nodes] = True
        self.fixed[self.top_nodes] = True
        self.material = api.dispersed_fiber(self.mu, self.k1, self.k2, self.kd, self.phi_deg, self.rho0)
        self.fiber_dirs = circumferential_fiber_dirs(self.mesh, self.phi_deg)           # [E, 2, 3]
        self.fiber_field = api.fiber_structure_tensors(self.fiber_dirs, self.kd)        # [E, 2, 3, 3]
        self.tau = api.compute_tau(self.mesh, self.material, self.c_m)
        self.ts = api.gen_alpha_scalars(self.rho_inf, self.dt)
        self.n_free = int((~self.fixed[:, 0]).sum())
        self.nv = 3 * self.n_free
        self.np = self.mesh.n_nodes

    def top_displacement(self, step: int) -> np.ndarray:
        """Prescribed displacement [n_top, 3] at the end of time step `step` (1-based), linear ramp."""
        u = np.zeros((len(self.top_nodes), 3))
        u[:, 2] = self.stretch * self.length * min(step, self.n_steps) / self.n_steps
        return u

    solver_options = CubeProblem.solver_options

    def context(self, device: int = 0) -> api.Context:
        ctx = api.Context(device)
        ctx.set_mesh(self.mesh, self.tau)
        ctx.build_dofs(self.fixed)
        ctx.set_material(self.material)
        ctx.set_fiber_field(self.fiber_field)
        ctx.set_loads((0.0, 0.0, 0.0))
        return ctx
