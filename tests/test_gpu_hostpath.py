"""GPU: the host-memory entry points and apply_operator's argument contract.

* hx_apply_host is stream-ordered: a call may read host input that earlier
  work on the same stream produces (chained out -> in without a sync);
* hx_apply_host_staged (apply_operator on plain numpy arrays) streams
  pageable memory through a pinned ring and is bitwise the device apply;
* a caller-supplied ``out`` is validated and left untouched on non-finite
  input (the reference scans q before any work, operators.py:317-318);
* several devices in one process (skipped on a one-GPU box)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1711_00903_b200 as hx  # noqa: E402
from oracle import hexbench_oracle as orc  # noqa: E402
from paper_1711_00903_b200 import _native, operators  # noqa: E402

pytestmark = pytest.mark.gpu

BPS = (hx.BP1, hx.BP35, hx.BP3)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def mesh3():
    return hx.perturb_mesh(hx.build_cube_mesh(3, 2.0), amplitude=0.15, seed=7)


def dev_apply(op, q):
    qd = torch.from_numpy(np.ascontiguousarray(q)).to(op.device)
    out = torch.empty_like(qd)
    hx.apply_device(op, qd, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def pinned(shape):
    return torch.empty(shape, dtype=torch.float64).pin_memory().numpy()


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("chunks", [1, 2, 3, 5])
def test_apply_host_chains_out_into_in_without_sync(bp, chunks, mesh3):
    """x1 = A x0 and x2 = A x1 queued back to back on one stream with one
    workspace: the second call's H2D must see the first call's D2H (ADVICE
    r1: the old cross-call slot sequence read x1 before it was written)."""
    op = hx.make_operator(bp, 7, mesh3, lam=1.0)
    chunk = -(-op.n_el // chunks)
    work = operators._device_work(op, chunk)
    x0 = pinned((op.n_el, op.n_p))
    x0[:] = np.random.default_rng(5).standard_normal(x0.shape)
    x1, x2, x3 = (pinned(x0.shape) for _ in range(3))
    x1[:] = np.nan  # stale contents must never be read
    x2[:] = np.nan
    for _ in range(3):
        hx.apply_host(op, x0, x1, chunk_el=chunk, work=work)
        hx.apply_host(op, x1, x2, chunk_el=chunk, work=work)
        hx.apply_host(op, x2, x3, chunk_el=chunk, work=work)
        torch.cuda.synchronize()
        ref1 = dev_apply(op, x0)
        ref2 = dev_apply(op, ref1)
        np.testing.assert_array_equal(x1, ref1)
        np.testing.assert_array_equal(x2, ref2)
        np.testing.assert_array_equal(x3, dev_apply(op, ref2))
        x1[:] = np.nan
        x2[:] = np.nan


def test_apply_host_same_plan_two_streams_one_workspace(mesh3):
    """Calls on one plan from two streams serialise on the plan's pipeline."""
    op = hx.make_operator(hx.BP35, 7, mesh3, lam=1.0)
    rng = np.random.default_rng(2)
    work = operators._device_work(op, 4)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    qs = [pinned((op.n_el, op.n_p)) for _ in range(6)]
    outs = [pinned((op.n_el, op.n_p)) for _ in range(6)]
    for i, (q, o) in enumerate(zip(qs, outs)):
        q[:] = rng.standard_normal(q.shape)
        hx.apply_host(op, q, o, stream=streams[i % 2].cuda_stream, chunk_el=4, work=work)
    torch.cuda.synchronize()
    for q, o in zip(qs, outs):
        np.testing.assert_array_equal(o, dev_apply(op, q))


@pytest.mark.parametrize("bp", BPS)
@pytest.mark.parametrize("chunks", [1, 2, 4, 7])
def test_apply_host_overlap_back_to_back_bitwise(bp, chunks, mesh3):
    """HX_HOST_OVERLAP: independent calls queued back to back pipeline into
    each other (the slot sequence continues across calls); every output is
    bitwise the device apply, including across a change of chunking (full
    drain), an interleaved stream-ordered call and a staged call."""
    op = hx.make_operator(bp, 7, mesh3, lam=0.7)
    rng = np.random.default_rng(11)
    chunk = -(-op.n_el // chunks)
    work = operators._device_work(op, max(chunk, 3))
    qs = [pinned((op.n_el, op.n_p)) for _ in range(8)]
    outs = [pinned((op.n_el, op.n_p)) for _ in range(8)]
    for q, o in zip(qs, outs):
        q[:] = rng.standard_normal(q.shape)
        o[:] = np.nan
    for i, (q, o) in enumerate(zip(qs, outs)):
        if i == 4:  # a plain stream-ordered call in the middle of the stream
            hx.apply_host(op, q, o, chunk_el=chunk, work=work)
        elif i == 5:  # another chunking: the pipeline drains first
            hx.apply_host(op, q, o, chunk_el=3, work=work, overlap=True)
        elif i == 6:  # the staged (pageable) path on the same plan
            torch.cuda.synchronize()
            o[:] = hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, np.array(q))).data
        else:
            hx.apply_host(op, q, o, chunk_el=chunk, work=work, overlap=True)
    torch.cuda.synchronize()
    for q, o in zip(qs, outs):
        np.testing.assert_array_equal(o, dev_apply(op, q))


def test_apply_host_ex_rejects_unknown_flags(mesh3):
    op = hx.make_operator(hx.BP35, 3, mesh3, lam=1.0)
    q = pinned((op.n_el, op.n_p))
    q[:] = 1.0
    o = pinned(q.shape)
    work = operators._device_work(op, op.n_el)
    st = _native.lib().hx_apply_host_ex(
        op.plan.handle, _native.ptr(q), _native.ptr(op.device_factors), _native.ptr(o),
        op.n_el, op.n_el, _native.ptr(work), None, 2, None)
    assert st != 0


@pytest.mark.parametrize("bp", BPS)
def test_staged_pageable_path_bitwise(bp, mesh3):
    """apply_operator on plain numpy (pageable) arrays, forced through many
    chunks of the pinned ring, in every combination of pageable / pinned
    input and output."""
    op = hx.make_operator(bp, 7, mesh3, lam=0.7)
    q = np.random.default_rng(9).standard_normal((op.n_el, op.n_p))
    ref = dev_apply(op, q)
    res = hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, q))
    assert isinstance(res.data, np.ndarray) and res.data.shape == q.shape
    np.testing.assert_array_equal(res.data, ref)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    q_pin = pinned(q.shape)
    q_pin[:] = q
    for src in (q, q_pin):
        for dst in (np.full_like(q, np.nan), pinned(q.shape)):
            dst[:] = np.nan
            for chunk in (1, 2, 5, 27):
                operators._apply_numpy(op, src, dst, flag, stream, chunk_el=chunk)
                np.testing.assert_array_equal(dst, ref)
    assert int(flag.item()) == 0


def test_staged_path_flags_nonfinite(mesh3):
    op = hx.make_operator(hx.BP1, 3, mesh3)
    q = np.random.default_rng(1).standard_normal((op.n_el, op.n_p))
    q[17, 5] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, q))


@pytest.mark.parametrize("on_device", [False, True])
def test_out_untouched_on_nonfinite_input(on_device, mesh3):
    op = hx.make_operator(hx.BP35, 4, mesh3, lam=1.0)
    q = np.random.default_rng(4).standard_normal((op.n_el, op.n_p))
    q[-1, -1] = np.nan
    if on_device:
        fv = hx.FieldVector(op.n_el, op.n_p, torch.from_numpy(q).cuda())
        out = torch.full((op.n_el, op.n_p), 3.0, dtype=torch.float64, device="cuda")
    else:
        fv = hx.FieldVector(op.n_el, op.n_p, q)
        out = np.full((op.n_el, op.n_p), 3.0)
    with pytest.raises(ValueError, match="non-finite"):
        hx.apply_operator(op, fv, out=out)
    vals = out.cpu().numpy() if on_device else out
    assert np.all(vals == 3.0)
    # and with finite input `out` receives the result
    q[-1, -1] = 0.0
    fv = hx.FieldVector(op.n_el, op.n_p, torch.from_numpy(q).cuda() if on_device else q)
    res = hx.apply_operator(op, fv, out=out)
    assert np.shares_memory(res.data, out) if not on_device else res.data.data_ptr() == out.data_ptr()
    vals = out.cpu().numpy() if on_device else out
    np.testing.assert_array_equal(vals, dev_apply(op, q))


def test_out_validation(mesh3):
    op = hx.make_operator(hx.BP35, 2, mesh3)
    shape = (op.n_el, op.n_p)
    qh = hx.FieldVector(op.n_el, op.n_p, np.ones(shape))
    qd = hx.FieldVector(op.n_el, op.n_p, torch.ones(shape, dtype=torch.float64, device="cuda"))
    bad_host = [np.empty(shape, dtype=np.float32), np.empty((op.n_el, op.n_p + 1)),
                np.empty((op.n_p, op.n_el)).T, np.empty(op.n_el * op.n_p),
                torch.empty(shape, dtype=torch.float64, device="cuda")]
    for out in bad_host:
        with pytest.raises(ValueError):
            hx.apply_operator(op, qh, out=out)
    ro = np.empty(shape)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        hx.apply_operator(op, qh, out=ro)
    with pytest.raises(ValueError, match="alias"):
        hx.apply_operator(op, qh, out=qh.data)
    bad_dev = [torch.empty(shape, dtype=torch.float32, device="cuda"),
               torch.empty((op.n_p, op.n_el), dtype=torch.float64, device="cuda").T,
               torch.empty(op.n_el * op.n_p + 1, dtype=torch.float64, device="cuda")[1:],
               np.empty(shape)]
    for out in bad_dev:
        with pytest.raises(ValueError):
            hx.apply_operator(op, qd, out=out)
    with pytest.raises(ValueError, match="alias"):
        hx.apply_operator(op, qd, out=qd.data)


def test_dense_interp_for_non_centro_matrix():
    """interpolate_to_gl / project_to_gll accept any (N+2) x (N+1) matrix,
    like the reference's contract_dim: a perturbed matrix takes
    the dense passes and matches the oracle."""
    rng = np.random.default_rng(3)
    for deg in (1, 4, 7, 15):
        n, m = deg + 1, deg + 2
        mat = hx.interp_matrix(deg).entries + 1e-3 * rng.standard_normal((m, n))
        q = rng.standard_normal((5, n, n, n))
        t = rng.standard_normal((5, m, m, m))
        assert orc.rel_l2(hx.interpolate_to_gl(q, mat), orc.interp_passes(mat, q)) <= 1e-13
        assert orc.rel_l2(hx.project_to_gll(t, mat), orc.project_passes(mat, t)) <= 1e-13
        q[2, 0, 1, 1] = np.nan
        with pytest.raises(ValueError, match="non-finite"):
            hx.interpolate_to_gl(q, mat)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs")
def test_two_devices_one_process(mesh3):
    """Operators on cuda:0 and cuda:1 in one process: the per-device launch
    setup (dynamic shared-memory opt-in above 48 KB) and the host pipeline's
    streams follow the device."""
    q = np.random.default_rng(0).standard_normal((mesh3.n_el, 512))
    res = {}
    for dev in ("cuda:0", "cuda:1", "cuda:0"):
        for bp in BPS:
            op = hx.make_operator(bp, 7, mesh3, lam=1.0, device=dev)
            fv = hx.FieldVector(op.n_el, op.n_p, torch.from_numpy(q).to(dev))
            got = hx.apply_operator(op, fv).data.cpu().numpy()
            host = hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, q)).data
            np.testing.assert_array_equal(host, got)
            res.setdefault(bp, got)
            np.testing.assert_array_equal(got, res[bp])
    op = hx.make_operator(hx.BP35, 7, mesh3, device="cuda:1")
    with pytest.raises(ValueError, match="cuda:0"):
        hx.apply_operator(op, hx.FieldVector(op.n_el, op.n_p, torch.from_numpy(q).cuda(0)))
