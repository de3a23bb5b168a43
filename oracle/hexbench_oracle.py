"""CPU ORACLE -- test infrastructure only, never part of the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed CPU
reference.  It restates the reference algorithm of the three element matvecs
(``/root/reference/pkg/src/hexbench/operators.py``) in batched numpy: the
same sequence of 1-D contractions in the same axis order, vectorised over
elements instead of the reference's per-element Python loop
(operators.py:296-303).

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by the reference itself (``tests/golden/make_golden.py``,
committed fixtures ``tests/golden/*.npz``) to <= 1e-13 relative; the
reference's own oracles (dense assembly, dense.py) pinned those vectors to
1e-12 / 1e-11 / 1e-10 when they were generated.

Layouts: q, out (E, n^3) with point order (k, j, i); factors (E, 7, m^3) in
the reference order (mesh.py:12: Grr, Grs, Grt, Gss, Gst, Gtt, GwJ).
"""

import numpy as np

BP1, BP35, BP3 = "BP1.0", "BP3.5", "BP3.0"


def contract(mat, t, axis):
    """Batched contract_dim (reference_ops.py:68-85): t is (E, a0, a1, a2),
    contract tensor axis `axis` (0=k, 1=j, 2=i) with mat[a, b]."""
    mat = np.asarray(mat, dtype=np.float64)
    if axis == 2:                                   # i: t @ M^T on the last axis
        return t @ mat.T
    if axis == 1:                                   # j: M @ t over (.., b, i)
        return np.matmul(mat, t)
    e, b, a1, a2 = t.shape                          # k: M @ t reshaped (E, b, a1*a2)
    return np.matmul(mat, t.reshape(e, b, a1 * a2)).reshape(e, mat.shape[0], a1, a2)


def interp_passes(interp, q):
    """Reference operators.py:208-219: axis 1, then 2, then 0."""
    t = contract(interp, q, 1)
    t = contract(interp, t, 2)
    return contract(interp, t, 0)


def project_passes(interp, t):
    """Reference operators.py:222-232 with I^T, same axis order."""
    it = np.asarray(interp).T
    t = contract(it, t, 1)
    t = contract(it, t, 2)
    return contract(it, t, 0)


def diff_chain_combine(diff, lam, t, extra, facs):
    """Reference operators.py:235-268 (the k term uses rqt)."""
    qr = contract(diff, t, 2)
    qs = contract(diff, t, 1)
    qt = contract(diff, t, 0)
    grr, grs, grt, gss, gst, gtt, gwj = (facs[:, s] for s in range(7))
    rqr = grr * qr + grs * qs + grt * qt
    rqs = grs * qr + gss * qs + gst * qt
    rqt = grt * qr + gst * qs + gtt * qt
    dt = np.asarray(diff).T
    out = lam * gwj * extra
    out = out + contract(dt, rqr, 2)
    out = out + contract(dt, rqs, 1)
    out = out + contract(dt, rqt, 0)
    return out


def apply(bp, degree, lam, interp, diff, factors, q):
    """out = A q for all elements (reference operators.py:271-293).

    interp: (m, n) or None; diff: (n, n) for BP3.5, (m, m) for BP3.0;
    factors: (E, 7, m^3) or (E, 7, m, m, m); q: (E, n^3).
    """
    n, m = degree + 1, degree + 2
    q = np.asarray(q, dtype=np.float64)
    e = q.shape[0]
    qe = q.reshape(e, n, n, n)
    p = n if bp == BP35 else m
    facs = np.asarray(factors, dtype=np.float64).reshape(e, 7, p, p, p)
    if bp == BP1:
        t = interp_passes(interp, qe)
        t = facs[:, 6] * t
        out = project_passes(interp, t)
    elif bp == BP35:
        out = diff_chain_combine(diff, lam, qe, qe, facs)
    elif bp == BP3:
        t = interp_passes(interp, qe)
        a = diff_chain_combine(diff, lam, t, t, facs)
        out = project_passes(interp, a)
    else:
        raise ValueError(f"unknown benchmark {bp!r}")
    return out.reshape(e, n ** 3)


def apply_chunked(bp, degree, lam, interp, diff, factors, q, chunk=512):
    """Same as ``apply`` in element chunks (bounded temporaries)."""
    q = np.asarray(q)
    out = np.empty_like(q, dtype=np.float64)
    for lo in range(0, q.shape[0], chunk):
        out[lo:lo + chunk] = apply(bp, degree, lam, interp, diff,
                                   factors[lo:lo + chunk], q[lo:lo + chunk])
    return out


def rel_l2(a, b):
    """Relative L2 error ||a - b|| / ||b|| (the north-star parity metric)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def rel_inf(a, b):
    """max|a - b| / max(1, max|b|) -- the reference tests' metric
    (test_acceptance.py:62)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


# ---- assembly on the structured cube mesh (checker for csrc/hx_dss.cu) ------
# The reference has no assembly, so nothing here is pinned to a
# reference output: these restate Q / Q^T as plain index arithmetic on
# build_cube_mesh's element order (mesh.py:44-56: e = (cx*side + cy)*side + cz,
# r/s/t = x/y/z) and are checked in tests against dense linear algebra.

def cube_global_index(side, degree):
    """(E, n^3) global node id of every element-local node."""
    n, N = degree + 1, degree
    g1 = side * N + 1
    e = np.arange(side ** 3)
    cx, cy, cz = e // (side * side), (e // side) % side, e % side
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    gx = cx[:, None] * N + i.ravel()[None, :]
    gy = cy[:, None] * N + j.ravel()[None, :]
    gz = cz[:, None] * N + k.ravel()[None, :]
    return (gx * g1 + gy) * g1 + gz


def cube_boundary(side, degree):
    """(n_global,) bool: node lies on the cube boundary."""
    g1 = side * degree + 1
    gx, gy, gz = np.meshgrid(np.arange(g1), np.arange(g1), np.arange(g1), indexing="ij")
    b = (gx == 0) | (gx == g1 - 1) | (gy == 0) | (gy == g1 - 1) | (gz == 0) | (gz == g1 - 1)
    return b.ravel()


def scatter_add(u, gidx, n_global):
    """Q^T u: sum element-local values into global nodes."""
    out = np.zeros(n_global)
    np.add.at(out, gidx.ravel(), np.asarray(u, dtype=np.float64).ravel())
    return out


def dss(u, side, degree, mask=False):
    """mask . Q Q^T u, element-local in and out."""
    gidx = cube_global_index(side, degree)
    ng = (side * degree + 1) ** 3
    s = scatter_add(u, gidx, ng)
    if mask:
        s[cube_boundary(side, degree)] = 0.0
    return s[gidx].reshape(np.shape(u))


def multiplicity(side, degree):
    gidx = cube_global_index(side, degree)
    cnt = np.bincount(gidx.ravel(), minlength=(side * degree + 1) ** 3)
    return cnt[gidx]


_CORNERS = np.array([[a, b, c] for a in (-1.0, 1.0) for b in (-1.0, 1.0) for c in (-1.0, 1.0)])


def node_coords(vertices, nodes):
    """(E, n^3, 3) physical coordinates of every element-local node under the
    trilinear map (reference mesh.py:93-98, corner order mesh.py:9), batched:
    node (k, j, i) sits at reference point (nodes[i], nodes[j], nodes[k])."""
    v = np.asarray(vertices, dtype=np.float64)
    r = np.asarray(nodes, dtype=np.float64)
    n = r.size
    t, s, q = np.meshgrid(r, r, r, indexing="ij")          # (k, j, i) grids
    pts = np.stack([q.ravel(), s.ravel(), t.ravel()], axis=1)  # (n^3, 3) = (r, s, t)
    phi = np.prod(1 + pts[:, None, :] * _CORNERS[None, :, :], axis=2) / 8.0  # (n^3, 8)
    return np.einsum("pc,ecd->epd", phi, v).reshape(v.shape[0], n ** 3, 3)


def assembled_cg(apply, b, side, degree, mask, tol=1e-13, maxiter=2000):
    """CG on mask Q^T A_L Q with continuous element-local representatives (the
    algorithm of cg.cg_solve_assembled, in numpy).  Returns (x, iterations)."""
    mult = multiplicity(side, degree)
    r = dss(b, side, degree, mask)
    x = np.zeros_like(r)
    p = r.copy()
    rr = np.sum(r * r / mult)
    r0 = np.sqrt(rr)
    for it in range(maxiter):
        ap = apply(p)
        alpha = rr / np.sum(p * ap)
        x += alpha * p
        r -= alpha * dss(ap, side, degree, mask)
        rn = np.sum(r * r / mult)
        if np.sqrt(rn) < tol * r0:
            return x, it + 1
        p = r + rn / rr * p
        rr = rn
    return x, maxiter


def dss_range(pad, side, degree, e_begin, e_end, base, mask=False):
    """mask . Q Q^T restricted to elements [e_begin, e_end), computed ONLY from
    the padded vector ``pad`` holding elements [base, base + len(pad)) -- the
    rank-local view of csrc/hx_dss.cu's range semantics (checks that the halo
    holds every copy of every own node)."""
    gidx = cube_global_index(side, degree)
    ng = (side * degree + 1) ** 3
    top = base + pad.shape[0]
    s = scatter_add(pad, gidx[base:top], ng)
    if mask:
        s[cube_boundary(side, degree)] = 0.0
    return s[gidx[e_begin:e_end]]


def dss_passes(u, side, degree):
    """Q Q^T as three per-axis face passes (csrc/hx_dss.cu dss_pass_kernel):
    for every interior face normal to x, then y, then z, both copies of each
    face node become (lower-element copy + upper-element copy)."""
    n, N = degree + 1, degree
    t = np.array(u, dtype=np.float64).reshape(side, side, side, n, n, n)  # cx,cy,cz,k,j,i
    # x: element axis 0, local i (axis 5); y: axis 1, local j (axis 4); z: axis 2, k (axis 3)
    for eax, lax in ((0, 5), (1, 4), (2, 3)):
        lo = [slice(None)] * 6
        hi = [slice(None)] * 6
        lo[eax], lo[lax] = slice(0, side - 1), N       # lower element's upper face
        hi[eax], hi[lax] = slice(1, side), 0           # upper element's lower face
        s = t[tuple(lo)] + t[tuple(hi)]
        t[tuple(lo)] = s
        t[tuple(hi)] = s
    return t.reshape(np.shape(u))
