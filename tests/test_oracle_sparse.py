"""CPU: the sparse (COO) oracle against the reference's own SparseTensor
tests (proj/tests/test_tensor.cpp:302-318) and against the dense compress
(compression.cpp:108-130) it restates; the host side of the Python
SparseTensor mirror (no GPU)."""
import numpy as np
import pytest

from oracle import octen_oracle as O


def random_coo(shape, nnz, seed):
    r = np.random.default_rng(seed)
    flat = r.choice(int(np.prod(shape)), nnz, replace=False)
    idx = np.stack(np.unravel_index(flat, shape), axis=1)
    return idx, r.random(nnz)


def test_sparse_round_trip_preserves_nonzeros_exactly():
    # test_tensor.cpp:302-313
    r = np.random.default_rng(3)
    t = np.where(r.random((4, 3, 5)) < 0.3, r.standard_normal((4, 3, 5)), 0.0)
    import paper_1807_01350_b200 as ob
    sp = ob.SparseTensor.from_dense(t)
    back = O.sparse_to_dense(t.shape, np.stack([sp.i, sp.j, sp.k], 1), sp.values.astype(np.float64))
    assert np.array_equal(back, t.astype(np.float32).astype(np.float64))
    assert sp.nnz == int(np.count_nonzero(t))
    # first-index-fastest order (tensor.cpp:104-116)
    flat = sp.i + 4 * sp.j + 12 * sp.k
    assert np.all(np.diff(flat) > 0)


def test_sparse_rejects_bad_entries():
    # test_tensor.cpp:315-318
    with pytest.raises(O.ConfigError, match="index out of bounds"):
        O.sparse_to_dense((2, 2), [[2, 0]], [1.0])
    with pytest.raises(O.ConfigError, match="duplicate index"):
        O.sparse_to_dense((2, 2), [[0, 0], [0, 0]], [1.0, 2.0])
    with pytest.raises(O.NumericError, match="non-finite value"):
        O.sparse_to_dense((2, 2), [[0, 1]], [np.nan])
    # entries are checked in input order: the first bad entry decides
    with pytest.raises(O.NumericError):
        O.sparse_to_dense((2, 2), [[0, 1], [0, 1], [5, 5]], [np.inf, 1.0, 1.0])


@pytest.mark.parametrize("q", [3, 8])
def test_direct_coo_compress_equals_dense_compress(q):
    shape = (17, 13, 6)
    idx, v = random_coo(shape, 150, q)
    r = np.random.default_rng(10 + q)
    u, vv, w = r.random((shape[0], q)), r.random((shape[1], q)), r.random((shape[2], q))
    dense = O.sparse_to_dense(shape, idx, v)
    z = dense
    for m, mat in enumerate((u, vv, w)):
        z = O.mode_n_product(z, mat.T, m)
    zd = O.compress_coo_direct(idx[:, 0], idx[:, 1], idx[:, 2], v, u, vv, w, chunk=37)
    assert np.abs(zd - z).max() <= 1e-13 * np.abs(z).max()
    a, b, c = r.random(q), r.random(q), r.random(q)
    probe = O.coo_probe(idx[:, 0], idx[:, 1], idx[:, 2], v, u, vv, w, a, b, c)
    assert abs(probe - np.einsum("abc,a,b,c", z, a, b, c)) <= 1e-12 * abs(probe)


def test_python_sparse_tensor_host_checks():
    import paper_1807_01350_b200 as ob
    with pytest.raises(ob.ConfigError, match="arity"):
        ob.SparseTensor((2, 2, 2), [[0, 0]], [1.0])
    with pytest.raises(ob.ConfigError):
        ob.SparseTensor((2, 2, 2), [[0, 0, 0]], [1.0, 2.0])
    sp = ob.SparseTensor((2, 2, 2), [], [])
    assert sp.nnz == 0 and sp.i.dtype == np.int32


@pytest.mark.parametrize("rank", [3, 6, 9])
def test_congruence_host_abi_matches_oracle(rank):
    # eval.cpp:22-46 through the C-ABI's host evaluation (no GPU needed)
    import paper_1807_01350_b200 as ob
    r = np.random.default_rng(rank)
    dims = (20, 15, 12)
    g = O.KruskalModel([r.random((d, rank)) for d in dims], np.ones(rank))
    perm = r.permutation(rank)
    e = O.KruskalModel([f[:, perm] * (1 + 0.05 * r.standard_normal(f[:, perm].shape)) for f in g.factors],
                       np.ones(rank))
    got = ob.congruence(g, e)
    want = O.congruence(g, e)
    assert np.allclose(got, want, rtol=0, atol=1e-12)
