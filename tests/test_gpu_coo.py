"""GPU parity of the sparse (COO) compression (csrc/coo.cu) through the C-ABI
against the CPU oracle: compress(to_dense(batch)) (compression.cpp:108-130 on
tensor.cpp:118-122) and the SparseTensor errors (tensor.cpp:87-102).

Tolerance: 1e-5 relative Frobenius (BASELINE north star: <= 1e-4 in fp32).
The slice products accumulate in fp32 from fp32-rounded projections; the
mode-3 accumulation into the summaries is fp64."""
import numpy as np
import pytest

from oracle import octen_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    import paper_1807_01350_b200 as m
    return m


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300))


def zipf_coo(shape, nnz, seed, s=1.2, heavy_slice=None):
    """Zipf(s) rows/columns, uniform slices, U(0,1) values, duplicates dropped."""
    r = np.random.default_rng(seed)
    I, J, t = shape

    def zipf(n, m):
        p = 1.0 / np.arange(1, n + 1) ** s
        return r.choice(n, m, p=p / p.sum())

    i, j, k = zipf(I, nnz), zipf(J, nnz), r.integers(0, t, nnz)
    if heavy_slice is not None:
        k[: nnz // 2] = heavy_slice
    key = (k.astype(np.int64) * I + i) * J + j
    _, first = np.unique(key, return_index=True)
    first = np.sort(first)
    perm = r.permutation(first.size)  # arbitrary input order
    sel = first[perm]
    return np.stack([i[sel], j[sel], k[sel]], 1), r.random(sel.size).astype(np.float32)


def projections(p, dims, q, seed):
    r = np.random.default_rng(seed)
    return [[r.random((d, q)) for _ in range(p)] for d in dims]


def oracle_z(shape, idx, vals, u, v, w):
    return [O.compress_coo_direct(idx[:, 0], idx[:, 1], idx[:, 2], vals.astype(np.float64), u[r], v[r], w[r])
            for r in range(len(u))]


@pytest.mark.parametrize("q,p", [(5, 3), (20, 4), (32, 5), (50, 7), (64, 6), (100, 2), (128, 3)])
def test_coo_compress_matches_oracle(ob, q, p):
    shape = (70, 60, 9)
    idx, vals = zipf_coo(shape, 3000, q + p)
    u, v, w = projections(p, shape, q, q)
    z = ob.compress_coo(ob.SparseTensor(shape, idx, vals), u, v, w)
    ref = oracle_z(shape, idx, vals, u, v, w)
    for a, b in zip(z, ref):
        assert rel(a, b) < TOL


def test_coo_matches_dense_definition_and_dense_device_path(ob):
    shape = (30, 25, 7)
    idx, vals = zipf_coo(shape, 700, 5)
    u, v, w = projections(4, shape, 12, 6)
    dense = O.sparse_to_dense(shape, idx, vals.astype(np.float64))
    zc = ob.compress_coo(ob.SparseTensor(shape, idx, vals), u, v, w)
    zd = ob.compress(dense.astype(np.float32), u, v, w, 0)
    for r in range(4):
        zr = dense
        for m, mat in enumerate((u[r], v[r], w[r])):
            zr = O.mode_n_product(zr, mat.T, m)
        assert rel(zc[r], zr) < TOL
        assert rel(zc[r], zd[r]) < TOL


def test_coo_heavy_slice_and_rows_span_many_rounds(ob):
    # one row of one slice with 1500 entries (a group longer than several
    # 256-entry staging rounds) and slices with more than 32 distinct rows
    shape = (40, 3000, 5)
    idx, vals = zipf_coo(shape, 8000, 9, heavy_slice=2)
    keep = ~((idx[:, 0] == 0) & (idx[:, 2] == 2))
    heavy = np.stack([np.zeros(1500, int), np.arange(1500) * 2, np.full(1500, 2)], 1)
    idx = np.concatenate([idx[keep], heavy])
    vals = np.concatenate([vals[keep], np.random.default_rng(1).random(1500).astype(np.float32)])
    perm = np.random.default_rng(2).permutation(len(vals))
    idx, vals = idx[perm], vals[perm]
    assert len(np.unique(idx[idx[:, 2] == 2, 0])) > 32
    u, v, w = projections(5, shape, 24, 3)
    z = ob.compress_coo(ob.SparseTensor(shape, idx, vals), u, v, w)
    for a, b in zip(z, oracle_z(shape, idx, vals, u, v, w)):
        assert rel(a, b) < TOL
    # run-to-run determinism (no unordered atomics)
    z2 = ob.compress_coo(ob.SparseTensor(shape, idx, vals), u, v, w)
    assert all(np.array_equal(a, b) for a, b in zip(z, z2))


def test_coo_empty_batch_and_empty_slices(ob):
    shape = (20, 20, 6)
    u, v, w = projections(3, shape, 8, 1)
    z = ob.compress_coo(ob.SparseTensor(shape, [], []), u, v, w)
    assert all(np.count_nonzero(x) == 0 for x in z)
    idx = np.array([[0, 0, 0], [19, 19, 5], [3, 4, 5]])
    vals = np.array([1.0, 2.0, -3.0], np.float32)
    z = ob.compress_coo(ob.SparseTensor(shape, idx, vals), u, v, w)
    for a, b in zip(z, oracle_z(shape, idx, vals, u, v, w)):
        assert rel(a, b) < TOL


def test_coo_summaries_accumulate_and_errors_leave_them_unchanged(ob):
    shape = (50, 40, 8)
    u, v, w1 = projections(4, shape, 16, 2)
    w2 = projections(4, shape, 16, 12)[2]
    b1 = zipf_coo(shape, 900, 1)
    b2 = zipf_coo(shape, 1100, 2)
    s = ob.CooSummaries(u, v)
    s.compress(ob.SparseTensor(shape, *b1), w1)
    s.compress(ob.SparseTensor(shape, *b2), w2)
    y = s.summaries()
    ref = [a + b for a, b in zip(oracle_z(shape, *b1, u, v, w1), oracle_z(shape, *b2, u, v, w2))]
    for a, b in zip(y, ref):
        assert rel(a, b) < TOL
    bad = [
        (np.array([[0, 0, 0], [50, 0, 0]]), [1.0, 1.0], ob.ConfigError, "SparseTensor: index out of bounds"),
        (np.array([[0, 0, 0], [0, 0, -1]]), [1.0, 1.0], ob.ConfigError, "SparseTensor: index out of bounds"),
        (np.array([[0, 0, 0], [1, 0, 8]]), [1.0, 1.0], ob.ConfigError, "SparseTensor: index out of bounds"),
        (np.array([[0, 0, 0], [1, 1, 1]]), [1.0, np.nan], ob.NumericError, "SparseTensor: non-finite value"),
        (np.array([[0, 0, 0], [1, 1, 1]]), [np.inf, 1.0], ob.NumericError, "SparseTensor: non-finite value"),
        (np.array([[3, 2, 1], [0, 0, 0], [3, 2, 1]]), [1.0, 1.0, 1.0], ob.ConfigError,
         "SparseTensor: duplicate index"),
        # the first offending entry (input order) decides
        (np.array([[3, 2, 1], [3, 2, 1], [1, 1, 1], [99, 0, 0]]), [1.0, 1.0, np.nan, 1.0], ob.ConfigError,
         "SparseTensor: duplicate index"),
        (np.array([[3, 2, 1], [1, 1, 1], [3, 2, 1], [99, 0, 0]]), [1.0, np.nan, 1.0, 1.0], ob.NumericError,
         "SparseTensor: non-finite value"),
        (np.array([[3, 2, 1], [99, 1, 1], [3, 2, 1]]), [1.0, np.nan, 1.0], ob.ConfigError,
         "SparseTensor: index out of bounds"),
    ]
    for idx, vals, exc, msg in bad:
        with pytest.raises(exc) as ei:
            s.compress(ob.SparseTensor(shape, idx, np.array(vals, np.float32)), w1)
        assert str(ei.value) == msg
    for a, b in zip(s.summaries(), y):
        assert np.array_equal(a, b)
    s.reset()
    assert all(np.count_nonzero(x) == 0 for x in s.summaries())


def test_coo_cp_als_on_resident_summaries_equals_batched_als(ob):
    shape = (60, 60, 10)
    u, v, w = projections(3, shape, 12, 4)
    s = ob.CooSummaries(u, v)
    s.compress(ob.SparseTensor(shape, *zipf_coo(shape, 2500, 7)), w)
    cfg = ob.AlsConfig(rank=3, max_iters=40, rel_tol=1e-8, n_restarts=2)
    seeds = [11, 12, 13]
    m1, f1, it1 = s.cp_als(cfg, seeds)
    m2, f2, it2 = ob.cp_als_batched(s.summaries(), cfg, seeds)
    assert np.array_equal(it1, it2)
    assert np.allclose(f1, f2, rtol=0, atol=1e-12)
    for a, b in zip(m1, m2):
        for fa, fb in zip(a.factors, b.factors):
            assert np.allclose(fa, fb, rtol=0, atol=1e-10)
    st = s.stage_times()
    assert st["batches"] == 1 and st["als_runs"] == 1 and st["nnz"] > 0


def test_coo_full_scale_probe_property(ob):
    """c4 extents (1e5 x 1e5, 1000 slices per batch, Q=64, Zipf(1.2)) at 2e6
    nnz and P=3: <Y_p, a (x) b (x) c> against the exact O(nnz) probe."""
    import torch
    shape = (100000, 100000, 1000)
    idx, vals = zipf_coo(shape, 2_000_000, 21)
    p, q = 3, 64
    r = np.random.default_rng(5)
    u = [r.random((shape[0], q)) for _ in range(p)]
    v = [r.random((shape[1], q)) for _ in range(p)]
    w = [r.standard_normal((shape[2], q)) for _ in range(p)]
    s = ob.CooSummaries(u, v)
    dev = torch.device("cuda")
    W = torch.tensor(np.stack([x.T for x in w]), dtype=torch.float64, device=dev).contiguous()  # (p, Q, t)
    ti = torch.tensor(idx[:, 0], dtype=torch.int32, device=dev)
    tj = torch.tensor(idx[:, 1], dtype=torch.int32, device=dev)
    tk = torch.tensor(idx[:, 2], dtype=torch.int32, device=dev)
    tv = torch.tensor(vals, device=dev)
    torch.cuda.synchronize()
    s.compress_device(shape[2], W, ti, tj, tk, tv)
    y = s.summaries()
    for rr in range(p):
        for _ in range(3):
            a, b, c = r.random(q), r.random(q), r.standard_normal(q)
            got = float(np.einsum("abc,a,b,c", y[rr], a, b, c))
            want = O.coo_probe(idx[:, 0], idx[:, 1], idx[:, 2], vals, u[rr], v[rr], w[rr], a, b, c)
            scale = O.coo_probe(idx[:, 0], idx[:, 1], idx[:, 2], vals, u[rr], v[rr], np.abs(w[rr]), a, b, np.abs(c))
            assert abs(got - want) <= TOL * scale
