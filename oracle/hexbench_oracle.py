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
