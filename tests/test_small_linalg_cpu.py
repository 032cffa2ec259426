"""The device small-linear-algebra routines (paper_1807_01350_b200/csrc/
small_linalg.cuh) compiled for the host with g++ and checked against numpy /
the oracle.  CPU only; the same source is instantiated inside the kernels."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cpu_harness", "small_linalg_host.cpp")
LIB = os.path.join(HERE, "cpu_harness", "_build", "libsmall_linalg_host.so")

dp = ctypes.POINTER(ctypes.c_double)
ip = ctypes.POINTER(ctypes.c_int)


@pytest.fixture(scope="module")
def lib():
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    deps = [SRC, os.path.join(HERE, "..", "paper_1807_01350_b200", "csrc", "small_linalg.cuh")]
    if not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in deps):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", LIB, SRC])
    return ctypes.CDLL(LIB)


def P(a):
    return a.ctypes.data_as(dp)


def test_mt64_matches_oracle_engine(lib):
    out = np.zeros(1000)
    lib.h_mt64(ctypes.c_ulonglong(rng.derive(77, [7])), 1000, P(out))
    ref = rng.Substream(rng.derive(77, [7])).uniform01_array(1000)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("n", [1, 2, 5, 20, 33, 64])
def test_jacobi_eig_sym(lib, n):
    s = rng.Substream(n)
    x = s.fill_uniform(n, n + 7)
    a = np.asfortranarray(x @ x.T)
    w = np.zeros(n)
    v = np.zeros((n, n), order="F")
    lib.h_jacobi_eig(n, P(a), P(w), P(v))
    ref = np.linalg.eigvalsh(a)
    assert np.allclose(np.sort(w), ref, rtol=1e-12, atol=1e-12 * ref.max())
    assert np.allclose(v.T @ v, np.eye(n), atol=1e-12)
    assert np.allclose(a @ v, v * w[None, :], atol=1e-10 * ref.max())


@pytest.mark.parametrize("fn", ["h_eig_real", "h_eig_real_team"])
@pytest.mark.parametrize("n,seed", [(3, 1), (5, 2), (20, 3), (32, 4), (17, 5)])
def test_eig_real_matches_lapack(lib, n, seed, fn):
    s = rng.Substream(seed)
    a = np.asfortranarray(s.fill_uniform(n, n) * 2 - 1)
    wr, wi = np.zeros(n), np.zeros(n)
    v = np.zeros((n, n), order="F")
    assert getattr(lib, fn)(n, P(a), P(wr), P(wi), P(v)) == 1
    lam = wr + 1j * wi
    ref = np.linalg.eigvals(a)
    assert np.allclose(np.sort_complex(lam), np.sort_complex(ref), atol=1e-10)
    # eigenvectors: real columns and [Re|Im] pairs
    c = 0
    while c < n:
        if wi[c] != 0.0:
            vec = v[:, c] + 1j * v[:, c + 1]
            assert wi[c] > 0 and abs(wi[c + 1] + wi[c]) < 1e-14
            assert np.linalg.norm(a @ vec - lam[c] * vec) <= 1e-9 * np.linalg.norm(vec)
            c += 2
        else:
            vec = v[:, c]
            assert np.linalg.norm(a @ vec - wr[c] * vec) <= 1e-9 * np.linalg.norm(vec)
            c += 1


@pytest.mark.parametrize("fn", ["h_eig_real", "h_eig_real_team"])
def test_eig_real_gevd_pencil(lib, fn):
    # a pencil built the way GevdInit builds it (cp_als.cpp:117-126)
    truth = O.KruskalModel([rng.Substream(9 + k).fill_uniform(12, 4) for k in range(3)], np.ones(4))
    t = O.reconstruct(truth)
    g = O.GevdInit(t, [O.matricize(t, n) for n in range(3)], 4)
    w1, w2 = g.mixture(123, 0)
    s1 = (g.flat @ w1).reshape((12, 12), order="F")
    s2 = (g.flat @ w2).reshape((12, 12), order="F")
    p1 = g.u_r.T @ s1 @ g.v_r
    p2 = g.u_r.T @ s2 @ g.v_r
    pencil = np.asfortranarray(p1 @ np.linalg.inv(p2))
    wr, wi = np.zeros(4), np.zeros(4)
    v = np.zeros((4, 4), order="F")
    assert getattr(lib, fn)(4, P(pencil), P(wr), P(wi), P(v)) == 1
    assert np.allclose(wi, 0)
    ev, evec = np.linalg.eig(pencil)
    # same eigen-pairs up to order/scale
    for c in range(4):
        k = np.argmin(np.abs(ev - wr[c]))
        x = v[:, c] / np.linalg.norm(v[:, c])
        y = evec[:, k].real / np.linalg.norm(evec[:, k].real)
        assert abs(abs(x @ y) - 1) < 1e-9


@pytest.mark.parametrize("fn", ["h_lu_inverse", "h_lu_inverse_team"])
def test_lu_fullpiv(lib, fn):
    s = rng.Substream(4)
    a = np.asfortranarray(s.fill_uniform(6, 6))
    inv = np.zeros((6, 6), order="F")
    assert getattr(lib, fn)(6, P(a), P(inv)) == 1
    assert np.allclose(inv @ a, np.eye(6), atol=1e-10)
    sing = np.asfortranarray(np.outer(np.arange(1.0, 5), np.arange(2.0, 6)))
    inv = np.zeros((4, 4), order="F")
    assert getattr(lib, fn)(4, P(sing), P(inv)) == 0
    assert O.fullpiv_lu_invertible(sing) is False


def test_chol_semidef_rank(lib):
    rs = O.gen_replicas([4, 4], 2, 3, 2, 8)  # fully shared: rank 2 of 4
    proj = O.stack_projections(rs, 0)
    g = np.asfortranarray(proj.T @ proj)
    assert lib.h_chol_semidef(4, P(g), ctypes.c_double(1e-14)) == 2
    s = rng.Substream(5)
    x = s.fill_uniform(30, 12)
    g = np.asfortranarray(x.T @ x)
    g0 = g.copy()
    assert lib.h_chol_semidef(12, P(g), ctypes.c_double(1e-14)) == 12
    l = np.tril(g)
    assert np.allclose(l @ l.T, g0, rtol=1e-12)


def test_greedy_match_vs_oracle(lib):
    s = rng.Substream(11)
    for _ in range(40):
        r = 2 + int(s.uniform01() * 9)
        sim = np.asfortranarray(s.fill_uniform(r, r))
        perm = np.zeros(r, dtype=np.int32)
        lib.h_greedy(r, P(sim), ctypes.c_double(1e-9), perm.ctypes.data_as(ip))
        assert perm.tolist() == O.greedy_match(sim)
    sim = np.asfortranarray(np.full((3, 3), 0.5))
    perm = np.zeros(3, dtype=np.int32)
    assert lib.h_greedy(3, P(sim), ctypes.c_double(1e-9), perm.ctypes.data_as(ip)) > 0
    assert perm.tolist() == [0, 1, 2]


@pytest.mark.parametrize("m,n", [(10, 10), (20, 15), (100, 100)])
def test_top_singular_pair(lib, m, n):
    s = rng.Substream(m * 1000 + n)
    a = np.asfortranarray(np.outer(s.uniform01_array(m), s.uniform01_array(n)) + 0.01 * s.fill_uniform(m, n))
    u, v = np.zeros(m), np.zeros(n)
    sig = lib.h_top_sv
    sig.restype = ctypes.c_double
    sigma = sig(m, n, P(a), P(u), P(v))
    uu, ss, vt = np.linalg.svd(a)
    assert abs(sigma - ss[0]) <= 1e-12 * ss[0]
    sgn = np.sign(u @ uu[:, 0])
    assert np.allclose(u, sgn * uu[:, 0], atol=1e-10)
    assert np.allclose(v, sgn * vt[0], atol=1e-10)


def test_team_chol_and_triangular_inverse(lib):
    s = rng.Substream(77)
    x = s.fill_uniform(40, 16)
    g = np.asfortranarray(x.T @ x)
    g0 = g.copy()
    inv = np.zeros((16, 16), order="F")
    assert lib.h_team_chol_inv(16, P(g), P(inv), ctypes.c_double(1e-14)) == 16
    l = np.tril(g)
    assert np.allclose(l @ l.T, g0, rtol=1e-12)
    assert np.allclose(inv @ l, np.eye(16), atol=1e-10)
    rs = O.gen_replicas([4, 4], 2, 3, 2, 8)
    proj = O.stack_projections(rs, 0)
    g = np.asfortranarray(proj.T @ proj)
    inv = np.zeros((4, 4), order="F")
    assert lib.h_team_chol_inv(4, P(g), P(inv), ctypes.c_double(1e-11)) == 2


def _gram_with_gap(n, k, seed, gap):
    s = rng.Substream(seed)
    q, _ = np.linalg.qr(s.fill_uniform(n, n) - 0.5)
    lam = np.concatenate([np.logspace(0, -10, k), gap * 1e-10 * s.uniform01_array(n - k)])
    return np.asfortranarray((q * lam) @ q.T), q[:, :k]


@pytest.mark.parametrize("n,k,m", [(100, 20, 28), (64, 8, 16), (120, 20, 28)])
def test_subspace_eig_top(lib, n, k, m):
    a, _ = _gram_with_gap(n, k, n + k, 1e-4)
    u = np.zeros((n, k), order="F")
    theta = np.zeros(m)
    assert lib.h_subspace_eig_top(n, P(a), k, m, P(u), P(theta)) == 1
    w, v = np.linalg.eigh(a)
    w, v = w[::-1], v[:, ::-1]
    assert np.allclose(u.T @ u, np.eye(k), atol=1e-12)
    # Ritz values and the top-k subspace agree with LAPACK (to the Gram floor)
    assert np.allclose(theta[:k], w[:k], rtol=1e-6, atol=1e-14 * w[0])
    sv = np.linalg.svd(v[:, :k].T @ u, compute_uv=False)
    assert sv.min() > 1 - 1e-8
    # leading (well separated) eigenvectors individually
    for c in range(3):
        assert abs(abs(u[:, c] @ v[:, c]) - 1) < 1e-10


def test_subspace_eig_top_gives_up_without_gap(lib):
    s = rng.Substream(3)
    x = s.fill_uniform(60, 60)
    a = np.asfortranarray(x @ x.T)  # slowly decaying spectrum: no gap at k
    u = np.zeros((60, 10), order="F")
    theta = np.zeros(16)
    assert lib.h_subspace_eig_top(60, P(a), 10, 16, P(u), P(theta)) == 0
    z = np.zeros((40, 40), order="F")
    assert lib.h_subspace_eig_top(40, P(z), 4, 8, P(np.zeros((40, 4), order="F")), P(np.zeros(8))) == 0


def test_eig_real_team_matches_the_serial_routine(lib):
    # one-thread team instantiation vs the serial routine: the team version
    # replaces a/b chains by one reciprocal, so agreement is to rounding
    for n, seed in [(7, 11), (20, 12), (25, 13)]:
        s = rng.Substream(seed)
        a = np.asfortranarray(s.fill_uniform(n, n) * 2 - 1)
        outs = []
        for fn in ("h_eig_real", "h_eig_real_team"):
            wr, wi = np.zeros(n), np.zeros(n)
            v = np.zeros((n, n), order="F")
            assert getattr(lib, fn)(n, P(a), P(wr), P(wi), P(v)) == 1
            outs.append((wr, wi, v))
        (wr0, wi0, v0), (wr1, wi1, v1) = outs
        assert np.allclose(wr0, wr1, rtol=1e-10, atol=1e-10) and np.allclose(wi0, wi1, rtol=1e-10, atol=1e-10)
        # eigenvectors of a non-normal matrix move with ulp-level changes;
        # the residual test above (vs LAPACK) pins both versions


@pytest.mark.parametrize("n,k,kb,kind", [(64, 16, 15, "gapless"), (100, 20, 25, "gapless"), (128, 32, 32, "lowrank"),
                                         (40, 40, 7, "gapless"), (30, 5, 5, "cluster")])
def test_sym_eig_top_tridiag(lib, n, k, kb, kind):
    # the dense fallback of the GEVD eigenbasis: Householder + bisection +
    # inverse iteration, against LAPACK (numpy.linalg.eigh)
    r = np.random.default_rng(n + k)
    if kind == "gapless":
        x = r.random((n, 3 * n))
        a = x @ x.T
    elif kind == "lowrank":
        x = r.random((n, k)) @ r.random((k, 4 * n)) + 1e-4 * r.standard_normal((n, 4 * n))
        a = x @ x.T
    else:  # clustered: eigenvalues 1 +- 1e-9 in the top block
        qm, _ = np.linalg.qr(r.standard_normal((n, n)))
        ev = np.concatenate([1.0 + 1e-9 * np.arange(8), np.linspace(0.1, 0.5, n - 8)])
        a = (qm * ev) @ qm.T
        a = 0.5 * (a + a.T)
    a = np.asfortranarray(a)
    u = np.zeros((n, k), order="F")
    th = np.zeros(k)
    lib.h_sym_eig_top_tridiag.restype = ctypes.c_int
    assert lib.h_sym_eig_top_tridiag(n, P(a), k, P(u), P(th), kb) == 1
    w, v = np.linalg.eigh(a)
    w, v = w[::-1], v[:, ::-1]
    scale = abs(w[0])
    assert np.max(np.abs(th - w[:k])) <= 1e-12 * scale
    assert np.max(np.abs(u.T @ u - np.eye(k))) < 1e-12
    # residuals |A u - theta u| at rounding level
    res = np.linalg.norm(a @ u - u * th, axis=0)
    assert np.max(res) <= 1e-11 * scale
    if kind != "cluster":
        # the same subspace as LAPACK's top-k eigenvectors
        s = np.linalg.svd(v[:, :k].T @ u, compute_uv=False)
        assert s.min() > 1 - 1e-9
