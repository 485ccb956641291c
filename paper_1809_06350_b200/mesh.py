"""Structured box meshes (host-side setup input of the hot path).

A vectorised numpy restatement of the reference mesh generator
(mesh.cpp:64-200): lexicographic nodes ``i + mx (j + my k)`` (:166-172), six
tets per cell sharing the 0-7 diagonal (:68-75), orientation fixed by
swapping t[2] and t[3] (:94-103), ``volume = det/6``, shape-function gradients
from the rows of the inverse edge matrix (:106-115), ``h`` = longest edge
(:117-121) and boundary facets per local face (:125-154).  Every expression
keeps the reference's operation order, so the arrays are bitwise identical
to the reference's (checked by tests/test_oracle_cpu.py::test_mesh_tau_loads_bitwise_equal_to_reference
against oracle/_ref).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CELL_TETS = np.array([[0, 1, 3, 7], [0, 1, 5, 7], [0, 2, 3, 7], [0, 2, 6, 7], [0, 4, 5, 7],
                      [0, 4, 6, 7]], dtype=np.int64)
FACE = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]], dtype=np.int64)
TAGS = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def _det3(m):
    m0, m1, m2, m3, m4, m5, m6, m7, m8 = (m[:, k] for k in range(9))
    return m0 * (m4 * m8 - m5 * m7) - m1 * (m3 * m8 - m5 * m6) + m2 * (m3 * m7 - m4 * m6)


def _inv3(m):
    d = _det3(m)
    i = 1.0 / d
    m0, m1, m2, m3, m4, m5, m6, m7, m8 = (m[:, k] for k in range(9))
    return np.stack([(m4 * m8 - m5 * m7) * i, (m2 * m7 - m1 * m8) * i, (m1 * m5 - m2 * m4) * i,
                     (m5 * m6 - m3 * m8) * i, (m0 * m8 - m2 * m6) * i, (m2 * m3 - m0 * m5) * i,
                     (m3 * m7 - m4 * m6) * i, (m1 * m6 - m0 * m7) * i, (m0 * m4 - m1 * m3) * i], axis=1)


def _norm(v):
    return np.sqrt(v[..., 0] * v[..., 0] + v[..., 1] * v[..., 1] + v[..., 2] * v[..., 2])


@dataclass
class Mesh:
    """Mesh (mesh.hpp:24-50) as flat numpy arrays."""
    nodes: np.ndarray      # (N, 3)
    tets: np.ndarray       # (E, 4) int32, positively oriented
    volume: np.ndarray     # (E,)
    h: np.ndarray          # (E,)
    grad_n: np.ndarray     # (E, 4, 3)
    facet_nodes: np.ndarray  # (F, 3)
    facet_tet: np.ndarray    # (F,)
    facet_tag: np.ndarray    # (F,) index into tag_names
    tag_names: list

    @property
    def n_nodes(self):
        return self.nodes.shape[0]

    @property
    def n_tets(self):
        return self.tets.shape[0]

    def tag_id(self, name):
        return self.tag_names.index(name) if name in self.tag_names else -1

    def facet_area(self, f=None):
        fn = self.facet_nodes if f is None else self.facet_nodes[f]
        a, b, c = (self.nodes[fn[..., k]] for k in range(3))
        e1, e2 = b - a, c - a
        cr = np.stack([e1[..., 1] * e2[..., 2] - e1[..., 2] * e2[..., 1],
                       e1[..., 2] * e2[..., 0] - e1[..., 0] * e2[..., 2],
                       e1[..., 0] * e2[..., 1] - e1[..., 1] * e2[..., 0]], axis=-1)
        return 0.5 * _norm(cr)

    def facet_centroid(self, f=None):
        fn = self.facet_nodes if f is None else self.facet_nodes[f]
        a, b, c = (self.nodes[fn[..., k]] for k in range(3))
        return (a + b + c) / 3.0

    def retag_facets(self, from_tag, pred, name):
        """Mesh::retag_facets (mesh.cpp:25-38)."""
        if name not in self.tag_names:
            self.tag_names.append(name)
        to = self.tag_names.index(name)
        sel = (self.facet_tag == from_tag) & pred(self.facet_centroid())
        self.facet_tag = np.where(sel, to, self.facet_tag)
        return int(sel.sum())

    def facets_with_tag(self, tag):
        return np.nonzero(self.facet_tag == tag)[0]


def generate_box_mesh(nx, ny, nz, lx, ly, lz) -> Mesh:
    """generate_box_mesh (mesh.cpp:158-188)."""
    if min(nx, ny, nz) < 1:
        raise ValueError("divisions must be >= 1")
    if min(lx, ly, lz) <= 0.0:
        raise ValueError("edge lengths must be positive")
    mx, my, mz = nx + 1, ny + 1, nz + 1
    k, j, i = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    nodes = np.stack([lx * i.ravel() / nx, ly * j.ravel() / ny, lz * k.ravel() / nz], axis=1)

    ck, cj, ci = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    corner = np.empty((ci.size, 8), dtype=np.int64)
    for b in range(8):
        corner[:, b] = (ci + (b & 1)) + mx * ((cj + ((b >> 1) & 1)) + my * (ck + ((b >> 2) & 1)))
    tets = corner[:, CELL_TETS].reshape(-1, 4)
    tets, volume, grad, h = _finalize_geometry(nodes, tets)

    # collect_boundary_facets (mesh.cpp:125-154)
    tol = 1e-12 * max(lx, ly, lz, 1.0)
    lims = (lx, ly, lz)
    tri = tets[:, FACE]  # (E, 4, 3)
    pts = nodes[tri]     # (E, 4, 3, 3)
    plane = np.full(tri.shape[:2], -1, dtype=np.int64)
    for d in range(2, -1, -1):  # first matching d wins in the reference -> iterate reversed
        lo = np.all(np.abs(pts[..., d]) < tol, axis=-1)
        hi = np.all(np.abs(pts[..., d] - lims[d]) < tol, axis=-1)
        plane = np.where(hi, 2 * d + 1, plane)
        plane = np.where(lo, 2 * d, plane)
    e_idx, f_idx = np.nonzero(plane >= 0)
    order = np.lexsort((f_idx, e_idx))
    e_idx, f_idx = e_idx[order], f_idx[order]
    return Mesh(nodes=nodes, tets=tets.astype(np.int32), volume=volume, h=h, grad_n=grad,
                facet_nodes=tri[e_idx, f_idx].astype(np.int32), facet_tet=e_idx.astype(np.int32),
                facet_tag=plane[e_idx, f_idx].astype(np.int32), tag_names=list(TAGS))


def _finalize_geometry(nodes, tets):
    """finalize_geometry (mesh.cpp:77-123): orientation, volume, shape-function gradients, h."""
    def edge_mat(t):
        x0 = nodes[t[:, 0]]
        dm = np.empty((t.shape[0], 9))
        for a in range(3):
            d = nodes[t[:, a + 1]] - x0
            dm[:, a], dm[:, 3 + a], dm[:, 6 + a] = d[:, 0], d[:, 1], d[:, 2]
        return dm

    dm = edge_mat(tets)
    det = _det3(dm)
    neg = det < 0.0
    if neg.any():
        tets[neg, 2], tets[neg, 3] = tets[neg, 3].copy(), tets[neg, 2].copy()
        dm[neg] = edge_mat(tets[neg])
        det[neg] = _det3(dm[neg])
    if (det <= 0.0).any():
        raise RuntimeError("degenerate tetrahedron in mesh")
    volume = det / 6.0
    inv = _inv3(dm)
    grad = np.empty((tets.shape[0], 4, 3))
    g0 = np.zeros((tets.shape[0], 3))
    for a in range(1, 4):
        g = inv[:, 3 * (a - 1):3 * (a - 1) + 3]
        grad[:, a] = g
        g0 = g0 - g
    grad[:, 0] = g0
    h = np.zeros(tets.shape[0])
    for a in range(4):
        for b in range(a + 1, 4):
            h = np.maximum(h, _norm(nodes[tets[:, a]] - nodes[tets[:, b]]))

    return tets, volume, grad, h


def generate_cube_mesh(n, edge_length) -> Mesh:
    """generate_cube_mesh (mesh.cpp:190-193)."""
    return generate_box_mesh(n, n, n, edge_length, edge_length, edge_length)


CYL_TAGS = ("rmin", "rmax", "zmin", "zmax")


def generate_cylinder_mesh(n_r, n_theta, n_z, r_in, thickness, length) -> Mesh:
    """Thick-walled cylinder about the z axis (BASELINE configs[3]; the reference
    has boxes only, mesh.hpp:52-60): n_r x n_theta x n_z hexes in (r, theta, z),
    periodic in theta, each split into six tets on its 0-7 diagonal exactly like
    the box generator (cell corner bit 0 = r, bit 1 = theta, bit 2 = z), then
    the reference's finalize_geometry.  Nodes are numbered
    ``i_r + (n_r + 1) (j_theta + n_theta k_z)``.  Boundary facets are tagged
    rmin / rmax / zmin / zmax."""
    if min(n_r, n_z) < 1 or n_theta < 3:
        raise ValueError("divisions must be >= 1 (>= 3 around the circumference)")
    if r_in <= 0.0 or thickness <= 0.0 or length <= 0.0:
        raise ValueError("radii and length must be positive")
    mr, mz = n_r + 1, n_z + 1
    k, j, i = np.meshgrid(np.arange(mz), np.arange(n_theta), np.arange(mr), indexing="ij")
    r = r_in + thickness * i.ravel() / n_r
    th = 2.0 * np.pi * j.ravel() / n_theta
    nodes = np.stack([r * np.cos(th), r * np.sin(th), length * k.ravel() / n_z], axis=1)
    ck, cj, ci = np.meshgrid(np.arange(n_z), np.arange(n_theta), np.arange(n_r), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    corner = np.empty((ci.size, 8), dtype=np.int64)
    for b in range(8):
        corner[:, b] = (ci + (b & 1)) + mr * (((cj + ((b >> 1) & 1)) % n_theta) + n_theta * (ck + ((b >> 2) & 1)))
    tets = corner[:, CELL_TETS].reshape(-1, 4)
    tets, volume, grad, h = _finalize_geometry(nodes, tets)
    # boundary facets from the logical coordinates of the facet's nodes
    tri = tets[:, FACE]
    ir = tri % mr
    kz = tri // (mr * n_theta)
    plane = np.full(tri.shape[:2], -1, dtype=np.int64)
    plane = np.where(np.all(kz == n_z, axis=-1), 3, plane)
    plane = np.where(np.all(kz == 0, axis=-1), 2, plane)
    plane = np.where(np.all(ir == n_r, axis=-1), 1, plane)
    plane = np.where(np.all(ir == 0, axis=-1), 0, plane)
    e_idx, f_idx = np.nonzero(plane >= 0)
    order = np.lexsort((f_idx, e_idx))
    e_idx, f_idx = e_idx[order], f_idx[order]
    return Mesh(nodes=nodes, tets=tets.astype(np.int32), volume=volume, h=h, grad_n=grad,
                facet_nodes=tri[e_idx, f_idx].astype(np.int32), facet_tet=e_idx.astype(np.int32),
                facet_tag=plane[e_idx, f_idx].astype(np.int32), tag_names=list(CYL_TAGS))


def circumferential_fiber_dirs(mesh: Mesh, phi_deg: float) -> np.ndarray:
    """Two fibre families per element at +-phi to the circumferential direction in the
    (theta, z) tangent plane of a cylinder about the z axis, evaluated at the element
    centroid: a = cos(phi) e_theta +- sin(phi) e_z.  Returns [E, 2, 3] unit vectors."""
    c = mesh.nodes[mesh.tets].mean(axis=1)
    rr = np.sqrt(c[:, 0] * c[:, 0] + c[:, 1] * c[:, 1])
    e_t = np.stack([-c[:, 1] / rr, c[:, 0] / rr, np.zeros_like(rr)], axis=1)
    e_z = np.array([0.0, 0.0, 1.0])
    phi = phi_deg * np.pi / 180.0
    return np.stack([np.cos(phi) * e_t + np.sin(phi) * e_z, np.cos(phi) * e_t - np.sin(phi) * e_z], axis=1)
