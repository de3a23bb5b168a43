"""Hexahedral cube meshes, trilinear element maps and geometric factors.

Mirrors reference ``mesh.py``.  Mesh construction and the seeded corner
perturbation reproduce the reference bit for bit (same numpy generator calls
and the same floating-point expression order), so a mesh built here is
identical to ``hexbench.mesh.perturb_mesh(build_cube_mesh(...))``.

Geometric factors exist in two forms:

* :func:`geometric_factors` -- host numpy, batched over elements, returning
  the reference ``(E, 7, m, m, m)`` array (reference ``mesh.py:101-139``);
* the device generator ``hx_geometric_factors`` in the native library, which
  writes straight into the packed device layout the kernels read (used by
  :func:`~paper_1711_00903_b200.operators.make_operator`).
"""

import itertools
from dataclasses import dataclass, field

import numpy as np

# reference corners, lexicographic (r, s, t) with r slowest (reference mesh.py:9)
CORNERS = np.array(list(itertools.product((-1.0, 1.0), repeat=3)))

# slot order of the 7-wide factor array (reference mesh.py:12)
FACTOR_NAMES = ("Grr", "Grs", "Grt", "Gss", "Gst", "Gtt", "GwJ")

DEGENERATE_DET = 1e-14


class DegenerateGeometryError(ValueError):
    """A trilinear element map folds over (non-positive Jacobian)."""


@dataclass(frozen=True)
class HexMesh:
    n_el: int
    vertices: np.ndarray = field(repr=False)  # (n_el, 8, 3)
    extent: float

    def __post_init__(self):
        v = np.array(self.vertices, dtype=np.float64)
        v.setflags(write=False)
        object.__setattr__(self, "vertices", v)


class GeometricFactors:
    """Weighted metric and Jacobian at the tensor quadrature points.

    ``data`` is the reference layout ``(n_el, 7, m, m, m)`` (point order
    (k, j, i)).  Instances produced by ``make_operator`` are device-resident
    and materialise ``data`` on the host only when it is first read.
    """

    def __init__(self, point_set, n_per_axis, weights_1d, data=None, loader=None):
        self.point_set = point_set
        self.n_per_axis = n_per_axis
        self.weights_1d = np.asarray(weights_1d, dtype=np.float64)
        self._data = data
        self._loader = loader

    @property
    def data(self):
        if self._data is None:
            self._data = self._loader()
        return self._data

    def element(self, e):
        return self.data[e]

    @property
    def gwj(self):
        return self.data[:, 6]


def build_cube_mesh(elements_per_side, extent):
    """elements_per_side**3 congruent hexahedra tiling [0, extent]^3."""
    if elements_per_side < 1:
        raise ValueError("elements_per_side must be >= 1")
    if extent <= 0:
        raise ValueError("extent must be positive")
    s = int(elements_per_side)
    h = extent / s
    idx = np.arange(s, dtype=np.float64)
    cx, cy, cz = np.meshgrid(idx, idx, idx, indexing="ij")  # cx slowest
    origins = np.stack([cx.ravel(), cy.ravel(), cz.ravel()], axis=1) * h
    verts = origins[:, None, :] + (CORNERS + 1.0)[None, :, :] * (h / 2.0)
    return HexMesh(s ** 3, verts, float(extent))


def _shape_gradients(r, s, t):
    """d(phi_c)/d(r,s,t) for the 8 trilinear shape functions at points
    (r, s, t) (arrays of length P) -> (P, 8, 3)."""
    rc, sc, tc = CORNERS[:, 0], CORNERS[:, 1], CORNERS[:, 2]
    r, s, t = (np.asarray(v, dtype=np.float64).reshape(-1) for v in (r, s, t))
    return np.stack([
        rc * (1 + np.outer(s, sc)) * (1 + np.outer(t, tc)) / 8.0,
        (1 + np.outer(r, rc)) * sc * (1 + np.outer(t, tc)) / 8.0,
        (1 + np.outer(r, rc)) * (1 + np.outer(s, sc)) * tc / 8.0,
    ], axis=2)


def trilinear_jacobian(element, r, s, t):
    """Forward Jacobian A = d(x,y,z)/d(r,s,t) and det(A) at one point."""
    element = np.asarray(element, dtype=np.float64)
    g = _shape_gradients([r], [s], [t])[0]  # (8, 3)
    a = element.T @ g
    det = float(np.linalg.det(a))
    if abs(det) <= DEGENERATE_DET:
        raise DegenerateGeometryError("trilinear map is degenerate")
    return a, det


def trilinear_map(element, r, s, t):
    element = np.asarray(element, dtype=np.float64)
    rc, sc, tc = CORNERS[:, 0], CORNERS[:, 1], CORNERS[:, 2]
    phi = (1 + r * rc) * (1 + s * sc) * (1 + t * tc) / 8.0
    return element.T @ phi


def perturb_mesh(mesh, amplitude=0.15, seed=0):
    """Seeded independent corner jiggle (reference mesh.py:61-74).

    Same generator draw and expression order as the reference, so the
    vertices are bit-identical; the 27-point fold check is batched.
    """
    rng = np.random.default_rng(seed)
    h = mesh.extent / round(mesh.n_el ** (1 / 3))
    verts = mesh.vertices + rng.uniform(-1, 1, mesh.vertices.shape) * amplitude * h / 2
    probe = np.array(list(itertools.product((-0.9, 0.0, 0.9), repeat=3)))
    g = _shape_gradients(probe[:, 0], probe[:, 1], probe[:, 2])  # (27, 8, 3)
    for lo in range(0, mesh.n_el, 65536):
        if np.any(np.abs(_det3(_jacobians(verts[lo:lo + 65536], g))) <= DEGENERATE_DET):
            raise DegenerateGeometryError("trilinear map is degenerate")
    return HexMesh(mesh.n_el, verts, mesh.extent)


def _jacobians(verts, g):
    """A[e, p, x, b] = sum_c verts[e, c, x] g[p, c, b] as one BLAS product."""
    e, p = verts.shape[0], g.shape[0]
    a = np.matmul(verts.transpose(0, 2, 1), g.transpose(1, 0, 2).reshape(8, p * 3))
    return a.reshape(e, 3, p, 3).transpose(0, 2, 1, 3)


def _det3(a):
    return (a[..., 0, 0] * (a[..., 1, 1] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 1])
            - a[..., 0, 1] * (a[..., 1, 0] * a[..., 2, 2] - a[..., 1, 2] * a[..., 2, 0])
            + a[..., 0, 2] * (a[..., 1, 0] * a[..., 2, 1] - a[..., 1, 1] * a[..., 2, 0]))


def tensor_points(rule):
    """(r, s, t) of the m^3 tensor points in (k, j, i) order, r fastest."""
    tt, ss, rr = np.meshgrid(rule.nodes, rule.nodes, rule.nodes, indexing="ij")
    return rr.ravel(), ss.ravel(), tt.ravel()


def geometric_factors(mesh, rule, chunk=2048):
    """Host-side factors, reference layout (n_el, 7, m, m, m).

    G = det(A) A^-1 A^-T and GwJ = det(A), each scaled by w_i w_j w_k
    (reference mesh.py:101-139), batched over element chunks.
    """
    m = rule.n
    w = rule.weights
    g = _shape_gradients(*tensor_points(rule))
    w3 = (w[:, None, None] * w[None, :, None] * w[None, None, :]).ravel()
    data = np.empty((mesh.n_el, 7, m ** 3))
    for lo in range(0, mesh.n_el, chunk):
        a = _jacobians(mesh.vertices[lo:lo + chunk], g)
        det = np.linalg.det(a)
        if np.any(det <= DEGENERATE_DET):
            raise DegenerateGeometryError("non-positive Jacobian determinant")
        inv = np.linalg.inv(a)
        gm = det[..., None, None] * np.einsum("epxb,epyb->epxy", inv, inv)
        blk = data[lo:lo + chunk]
        for slot, (x, y) in enumerate(((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))):
            blk[:, slot] = w3 * gm[..., x, y]
        blk[:, 6] = w3 * det
    return GeometricFactors(rule.kind, m, w, data.reshape(mesh.n_el, 7, m, m, m))
