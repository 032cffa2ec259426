"""ORACLE (test infrastructure only) -- CPU restatement of the reference's
per-batch OCTen hot path.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it; the product path never
does.

Every function restates the reference file:line it cites (paths relative to
/root/reference/proj).  The reference library cannot be built here (Eigen3,
doctest and CLI11 are absent and it needs cmake), so the
Eigen decompositions it calls are restated with LAPACK (numpy/scipy):

  Eigen (unpinned, >=3.3)              -> restated as
  ColPivHouseholderQR (+setThreshold)  -> scipy.linalg.qr(pivoting=True);
                                          rank = #|r_ii| > thr*|r_00|
  CompleteOrthogonalDecomposition      -> scipy.linalg.lstsq(gelsy, cond=thr)
  LLT                                  -> numpy.linalg.cholesky (lower)
  BDCSVD / JacobiSVD (thin)            -> numpy.linalg.svd
  EigenSolver                          -> numpy.linalg.eig (LAPACK dgeev)
  FullPivLU::isInvertible              -> rank test on the LU pivots

Parity is pinned by the reference's own known-answer and property tests
restated in tests/test_oracle_kat.py (frozen unfolding / Khatri-Rao examples,
replica_bound=25, mode-product oracle, normal-equations ALS oracle, the
std::mt19937_64 known answer, ...).

Layout conventions follow tensor.hpp:32-34: a DenseTensor is an ndarray whose
Fortran-order ravel is the reference's flat vector (first index fastest).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.linalg as sla

from . import rng

EPS = np.finfo(np.float64).eps


class ConfigError(Exception):
    """errors.hpp:14-17."""


class NumericError(Exception):
    """errors.hpp:19-22."""


class IoError(Exception):
    """errors.hpp: file and serialization failures (checkpoint corruption)."""


# ---------------------------------------------------------------------------
# tensor.cpp
# ---------------------------------------------------------------------------

def matricize(t: np.ndarray, mode: int) -> np.ndarray:
    """tensor.cpp:124-142 -- rows index `mode`, remaining modes ascending with
    the lowest fastest."""
    if mode < 0 or mode >= t.ndim:
        raise ConfigError(f"matricize: mode {mode + 1} out of range for order-{t.ndim} tensor")
    return np.moveaxis(t, mode, 0).reshape((t.shape[mode], -1), order="F")


def dematricize(m: np.ndarray, dims, mode: int) -> np.ndarray:
    """tensor.cpp:144-166."""
    dims = list(dims)
    rest = [d for k, d in enumerate(dims) if k != mode]
    out = m.reshape([dims[mode]] + rest, order="F")
    return np.moveaxis(out, 0, mode)


def mode_n_product(t: np.ndarray, m: np.ndarray, mode: int) -> np.ndarray:
    """tensor.cpp:168-178."""
    if m.shape[1] != t.shape[mode]:
        raise ConfigError("mode_n_product: matrix columns (%d) != tensor extent (%d) on mode %d"
                          % (m.shape[1], t.shape[mode], mode + 1))
    dims = list(t.shape)
    dims[mode] = m.shape[0]
    return dematricize(m @ matricize(t, mode), dims, mode)


def khatri_rao(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """tensor.cpp:188-197 -- out.col(r).segment(i*|y|,|y|) = x(i,r)*y.col(r)."""
    if x.shape[1] != y.shape[1]:
        raise ConfigError("khatri_rao: column counts differ (%d vs %d)" % (x.shape[1], y.shape[1]))
    return np.einsum("ir,jr->ijr", x, y).reshape(x.shape[0] * y.shape[0], x.shape[1])


def khatri_rao_chain(factors, skip_mode: int) -> np.ndarray:
    """tensor.cpp:199-216 -- folded from the highest mode down."""
    acc = None
    for mode in range(len(factors) - 1, -1, -1):
        if mode == skip_mode:
            continue
        acc = factors[mode] if acc is None else khatri_rao(acc, factors[mode])
    if acc is None:
        raise ConfigError("khatri_rao_chain: no factors left after skip")
    return acc


def frobenius_norm(t: np.ndarray) -> float:
    """tensor.cpp:237-241 (sequential sum of squares)."""
    v = np.asarray(t, dtype=np.float64).ravel(order="F")
    return math.sqrt(float(np.dot(v, v)))


def slice_mode(t: np.ndarray, mode: int, start: int, count: int) -> np.ndarray:
    """tensor.cpp:275-293."""
    idx = [slice(None)] * t.ndim
    idx[mode] = slice(start, start + count)
    return np.array(t[tuple(idx)], order="F")


def rank1_outer(vectors) -> np.ndarray:
    """tensor.cpp:218-235."""
    out = np.asarray(vectors[0], dtype=np.float64)
    for v in vectors[1:]:
        out = np.multiply.outer(out, np.asarray(v, dtype=np.float64))
    return out


# ---------------------------------------------------------------------------
# compression.cpp
# ---------------------------------------------------------------------------

@dataclass
class CompressionReplica:
    """compression.hpp:20-33."""
    replica_id: int
    nontemporal: List[np.ndarray]
    temporal: np.ndarray
    temporal_window_start: int = 0
    temporal_rows_total: int = 0

    def temporal_rows(self, begin: int, end: int) -> np.ndarray:
        """compression.cpp:8-14."""
        if begin < self.temporal_window_start or end > self.temporal_rows_total or begin > end:
            raise ConfigError("temporal_rows: range [%d,%d) outside materialized window" % (begin, end))
        o = begin - self.temporal_window_start
        return self.temporal[o:o + end - begin, :]


@dataclass
class ReplicaSet:
    """compression.hpp:35-51."""
    replicas: List[CompressionReplica]
    seed: int
    q: int
    shared: int
    temporal_mode: int
    nontemporal_dims: List[int]
    batches_drawn: int = 0
    temporal_shared_gram: Optional[np.ndarray] = None

    def p(self) -> int:
        return len(self.replicas)

    def order(self) -> int:
        return len(self.nontemporal_dims) + 1

    def nontemporal_slot(self, mode: int) -> int:
        """compression.cpp:16-20."""
        if mode == self.temporal_mode or mode < 0 or mode >= self.order():
            raise ConfigError("nontemporal_slot: bad mode")
        return mode if mode < self.temporal_mode else mode - 1


def gen_replicas(nontemporal_dims, q: int, p: int, shared: int, seed: int,
                 temporal_mode: int = -1) -> ReplicaSet:
    """compression.cpp:22-70."""
    if q < 1:
        raise ConfigError("gen_replicas: Q must be >= 1")
    if p < 1:
        raise ConfigError("gen_replicas: p must be >= 1")
    if shared < 0 or shared > q:
        raise ConfigError("gen_replicas: shared must lie in [0, Q]")
    if len(nontemporal_dims) == 0:
        raise ConfigError("gen_replicas: no non-temporal modes")
    for d in nontemporal_dims:
        if d < 1:
            raise ConfigError("gen_replicas: non-temporal extents must be >= 1")
    order = len(nontemporal_dims) + 1
    tm = order - 1 if temporal_mode < 0 else temporal_mode
    if tm < 0 or tm >= order:
        raise ConfigError("gen_replicas: temporal mode out of range")
    shared_blocks = []
    for m, d in enumerate(nontemporal_dims):
        s = rng.Substream(rng.derive(seed, [rng.K_NONTEMPORAL_SHARED, m]))
        shared_blocks.append(s.fill_uniform(d, shared))
    reps = []
    for r in range(p):
        mats = []
        for m, d in enumerate(nontemporal_dims):
            mat = np.empty((d, q), order="F")
            mat[:, :shared] = shared_blocks[m]
            if q > shared:
                s = rng.Substream(rng.derive(seed, [rng.K_NONTEMPORAL_PRIVATE, m, r]))
                mat[:, shared:] = s.fill_uniform(d, q - shared)
            mats.append(mat)
        reps.append(CompressionReplica(r, mats, np.zeros((0, q))))
    return ReplicaSet(reps, seed, q, shared, tm, list(nontemporal_dims), 0,
                      np.zeros((shared, shared)))


def extend_temporal(rs: ReplicaSet, t_new: int, batch_key: Optional[int] = None) -> None:
    """compression.cpp:72-99."""
    if t_new < 1:
        raise ConfigError("extend_temporal: t_new must be >= 1")
    key = rs.batches_drawn if batch_key is None else batch_key
    q, shared = rs.q, rs.shared
    s = rng.Substream(rng.derive(rs.seed, [rng.K_TEMPORAL_SHARED, key]))
    shared_rows = s.fill_uniform(t_new, shared)
    rs.temporal_shared_gram = rs.temporal_shared_gram + shared_rows.T @ shared_rows
    for rep in rs.replicas:
        fresh = np.empty((t_new, q), order="F")
        fresh[:, :shared] = shared_rows
        if q > shared:
            s2 = rng.Substream(rng.derive(rs.seed, [rng.K_TEMPORAL_PRIVATE, key, rep.replica_id]))
            fresh[:, shared:] = s2.fill_uniform(t_new, q - shared)
        rep.temporal = np.vstack([rep.temporal, fresh])
        rep.temporal_rows_total += t_new
    rs.batches_drawn += 1


def drop_temporal_history(rs: ReplicaSet) -> None:
    """compression.cpp:101-106."""
    for rep in rs.replicas:
        rep.temporal = np.zeros((0, rs.q))
        rep.temporal_window_start = rep.temporal_rows_total


def compress(t: np.ndarray, rs: ReplicaSet, replica: int, row_begin: int, row_end: int) -> np.ndarray:
    """compression.cpp:108-130 -- mode products, mode 0 first."""
    if replica < 0 or replica >= rs.p():
        raise ConfigError("compress: replica out of range")
    if t.ndim != rs.order():
        raise ConfigError("compress: tensor order mismatch")
    rep = rs.replicas[replica]
    if t.shape[rs.temporal_mode] != row_end - row_begin:
        raise ConfigError("compress: temporal extent does not match row range")
    out = np.asarray(t, dtype=np.float64)
    for mode in range(rs.order()):
        if mode == rs.temporal_mode:
            proj = rep.temporal_rows(row_begin, row_end).T
        else:
            u = rep.nontemporal[rs.nontemporal_slot(mode)]
            if u.shape[0] != t.shape[mode]:
                raise ConfigError("compress: extent mismatch on mode %d" % (mode + 1))
            proj = u.T
        out = mode_n_product(out, proj, mode)
    return out


def sparse_to_dense(shape, indices, values) -> np.ndarray:
    """SparseTensor validation (tensor.cpp:87-102) then to_dense
    (tensor.cpp:118-122).  indices: nnz x order (0-based), values: nnz.
    Entries are checked in input order; per entry arity, then bounds, then
    finiteness, then duplicates, as the constructor does."""
    shape = tuple(int(d) for d in shape)
    if any(d < 1 for d in shape):
        raise ConfigError("Shape: dimensions must be positive")
    idx = np.asarray(indices, dtype=np.int64).reshape(-1, len(shape)) if len(indices) else np.zeros((0, len(shape)), np.int64)
    vals = np.asarray(values, dtype=np.float64)
    seen = set()
    for e in range(idx.shape[0]):
        ix = tuple(int(x) for x in idx[e])
        for m in range(len(shape)):
            if ix[m] < 0 or ix[m] >= shape[m]:
                raise ConfigError("SparseTensor: index out of bounds")
        if not math.isfinite(vals[e]):
            raise NumericError("SparseTensor: non-finite value")
        if ix in seen:
            raise ConfigError("SparseTensor: duplicate index")
        seen.add(ix)
    out = np.zeros(shape, order="F")
    if idx.shape[0]:
        out[tuple(idx.T)] = vals
    return out


def compress_coo_direct(i, j, k, vals, u: np.ndarray, v: np.ndarray, w: np.ndarray, chunk: int = 1 << 14) -> np.ndarray:
    """compress(to_dense(batch)) (compression.cpp:108-130 on tensor.cpp:118-122)
    for one replica, evaluated entry-wise without densifying:
    Z(a,b,c) = sum_e v_e U(i_e,a) V(j_e,b) W(k_e,c).  Equal to the dense
    compress by linearity of the mode products (checked against it in
    tests/test_oracle_kat.py)."""
    q = u.shape[1]
    z = np.zeros((q, q * q))
    for s in range(0, len(vals), chunk):
        e = slice(s, s + chunk)
        a = u[i[e]] * np.asarray(vals[e], dtype=np.float64)[:, None]
        kr = (v[j[e]][:, :, None] * w[k[e]][:, None, :]).reshape(-1, q * q)  # column b + Q c
        z += a.T @ kr
    return z.reshape(q, q, q)  # [a, b, c]


def coo_probe(i, j, k, vals, u, v, w, a, b, c) -> float:
    """<compress(to_dense(batch)), a (x) b (x) c> = sum_e v_e (U a)_i (V b)_j (W c)_k,
    exact in O(nnz): the size-independent check of a full-scale compression."""
    return float(np.sum(np.asarray(vals, np.float64) * (u @ a)[i] * (v @ b)[j] * (w @ c)[k]))


@dataclass
class SummaryState:
    """compression.hpp:56-60."""
    y: List[np.ndarray]
    history: List[np.ndarray]
    batches_seen: int = 0


def init_summaries(rs: ReplicaSet) -> SummaryState:
    """compression.cpp:132-139."""
    shape = tuple([rs.q] * rs.order())
    return SummaryState([np.zeros(shape) for _ in range(rs.p())],
                        [np.zeros((rs.q, 0)) for _ in range(rs.p())], 0)


def update_summaries(state: SummaryState, z) -> None:
    """compression.cpp:141-153."""
    if len(z) != len(state.y):
        raise ConfigError("update_summaries: replica count mismatch")
    for i, zi in enumerate(z):
        if zi.shape != state.y[i].shape:
            raise ConfigError("update_summaries: summary shape mismatch for replica %d" % (i + 1))
        state.y[i] = state.y[i] + zi
    state.batches_seen += 1


# ---------------------------------------------------------------------------
# Eigen decompositions restated with LAPACK
# ---------------------------------------------------------------------------

def colpiv_qr_rank(a: np.ndarray, threshold: float) -> int:
    """Eigen ColPivHouseholderQR::rank(): #|r_ii| > threshold * |maxpivot|."""
    if a.size == 0:
        return 0
    r = sla.qr(a, mode="r", pivoting=True)[0]
    d = np.abs(np.diag(r))
    if d.size == 0 or d[0] == 0.0:
        return 0
    return int(np.sum(d > threshold * d.max()))


def ls_solve(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Least-squares solve of a full-column-rank system (ColPivQR.solve)."""
    return np.linalg.lstsq(a, b, rcond=None)[0]


def colpiv_qr_solve(a: np.ndarray, b: np.ndarray, threshold: float):
    """One ColPivHouseholderQR (Eigen) with setThreshold(threshold): returns
    (rank, x) with rank = #|r_ii| > threshold * max|r_jj| and, when the rank
    is full, x = P R^-1 (Q^T b) (else x = None) -- the rank test and the
    solve of recovery.cpp:26-38 / 396-401 from the same factorization."""
    if a.size == 0:
        return 0, None
    qm, rm, piv = sla.qr(a, mode="economic", pivoting=True, check_finite=False)
    d = np.abs(np.diag(rm))
    if d.size == 0 or d.max() == 0.0:
        return 0, None
    rank = int(np.sum(d > threshold * d.max()))
    if rank < a.shape[1]:
        return rank, None
    z = sla.solve_triangular(rm, qm.T @ b, lower=False, check_finite=False)
    x = np.empty_like(z)
    x[piv] = z
    return rank, x


def cod_solve(a: np.ndarray, b: np.ndarray, threshold: Optional[float] = None) -> np.ndarray:
    """Eigen CompleteOrthogonalDecomposition(a).solve(b): minimum-norm LS with
    a rank-revealing pivoted QR (LAPACK gelsy).  Default threshold is Eigen's
    epsilon * diagSize."""
    if threshold is None:
        threshold = EPS * min(a.shape)
    return sla.lstsq(a, b, cond=threshold, lapack_driver="gelsy")[0]


def fullpiv_lu_invertible(a: np.ndarray) -> bool:
    """Eigen FullPivLU::isInvertible: square and rank == n, rank counting
    pivots > epsilon*n*|maxpivot| under full pivoting."""
    n = a.shape[0]
    m = np.array(a, dtype=np.float64)
    piv = []
    for k in range(n):
        sub = np.abs(m[k:, k:])
        i, j = np.unravel_index(np.argmax(sub), sub.shape)
        i += k
        j += k
        m[[k, i], :] = m[[i, k], :]
        m[:, [k, j]] = m[:, [j, k]]
        p = m[k, k]
        piv.append(abs(p))
        if p != 0.0:
            m[k + 1:, k] /= p
            m[k + 1:, k + 1:] -= np.outer(m[k + 1:, k], m[k, k + 1:])
    maxp = max(piv) if piv else 0.0
    thr = EPS * n
    rank = sum(1 for p in piv if p > thr * maxp)
    return rank == n


# ---------------------------------------------------------------------------
# cp_als.cpp
# ---------------------------------------------------------------------------

K_DEGENERATE_NORM = 1e-14  # cp_als.cpp:17


@dataclass
class KruskalModel:
    """cp_als.hpp:12-23."""
    factors: List[np.ndarray]
    lambda_: np.ndarray

    def rank(self) -> int:
        return len(self.lambda_)

    def order(self) -> int:
        return len(self.factors)

    def normalize(self) -> None:
        """cp_als.cpp:216-228."""
        r = self.rank()
        if len(self.lambda_) == 0:
            self.lambda_ = np.ones(r)
        for f in self.factors:
            for c in range(r):
                nrm = np.linalg.norm(f[:, c])
                if nrm > 0.0:
                    f[:, c] /= nrm
                    self.lambda_[c] *= nrm


@dataclass
class AlsConfig:
    """cp_als.hpp:25-31."""
    rank: int = 1
    max_iters: int = 100
    rel_tol: float = 1e-8
    n_restarts: int = 3
    seed: int = 0


@dataclass
class AlsResult:
    """cp_als.hpp:33-40."""
    model: KruskalModel
    fit: float
    iterations: int
    fit_history: List[float] = field(default_factory=list)
    residual_history: List[float] = field(default_factory=list)
    rescued_degenerate: bool = False
    restart: int = 0        # oracle-only diagnostic: winning restart
    gevd_attempt: int = -1  # oracle-only diagnostic: GEVD attempt used (-1 random)


def peel_rank1(v: np.ndarray, dims):
    """cp_als.cpp:24-36 -- successive rank-1 SVD splits."""
    out = [None] * len(dims)
    carry = np.array(v, dtype=np.float64)
    for k in range(len(dims) - 1):
        rows = dims[k]
        cols = carry.size // rows
        m = carry.reshape((rows, cols), order="F")
        u, s, vt = np.linalg.svd(m, full_matrices=False)
        out[k] = u[:, 0].copy()
        carry = s[0] * vt[0, :]
    out[len(dims) - 1] = carry
    return out


class GevdInit:
    """cp_als.cpp:46-190 -- direct slice-eigendecomposition warm start."""

    def __init__(self, t: np.ndarray, unfoldings, rank: int):
        self.t = t
        self.unf = unfoldings
        self.rank = rank
        self.usable = False
        order = t.ndim
        if order < 3:
            return
        dims = t.shape
        m1 = 0
        for n in range(1, order):
            if dims[n] > dims[m1]:
                m1 = n
        m2 = 1 if m1 == 0 else 0
        for n in range(order):
            if n != m1 and dims[n] > dims[m2]:
                m2 = n
        if m1 > m2:
            m1, m2 = m2, m1
        self.m1, self.m2 = m1, m2
        self.d1, self.d2 = dims[m1], dims[m2]
        self.l_total = t.size // (self.d1 * self.d2)
        if self.d1 < rank or self.d2 < rank or self.l_total < 2:
            return
        rest = [n for n in range(order) if n != m1 and n != m2]
        # three-mode view (d1, d2, L), remaining modes ascending lowest fastest
        v = np.transpose(t, [m1, m2] + rest)
        self.flat = v.reshape((self.d1 * self.d2, self.l_total), order="F")
        u1, s1, _ = np.linalg.svd(unfoldings[m1], full_matrices=False)
        u2, s2, _ = np.linalg.svd(unfoldings[m2], full_matrices=False)
        if np.count_nonzero(s1) < rank or np.count_nonzero(s2) < rank:
            return
        self.u_r = u1[:, :rank]
        self.v_r = u2[:, :rank]
        self.usable = True

    def mixture(self, mixture_seed: int, attempt: int):
        ws = rng.Substream(rng.derive(mixture_seed, [rng.K_ALS_GEVD, attempt]))
        w1 = ws.uniform01_array(self.l_total) * 2 - 1
        w2 = ws.uniform01_array(self.l_total) * 2 - 1
        return w1, w2

    def factors(self, mixture_seed: int):
        if not self.usable:
            return None
        order = self.t.ndim
        rank = self.rank
        for attempt in range(3):
            w1, w2 = self.mixture(mixture_seed, attempt)
            s1m = (self.flat @ w1).reshape((self.d1, self.d2), order="F")
            s2m = (self.flat @ w2).reshape((self.d1, self.d2), order="F")
            p1 = self.u_r.T @ s1m @ self.v_r
            p2 = self.u_r.T @ s2m @ self.v_r
            if not fullpiv_lu_invertible(p2):
                continue
            pencil = p1 @ np.linalg.inv(p2)
            try:
                ev, evec = np.linalg.eig(pencil)
            except np.linalg.LinAlgError:
                continue
            # Eigen normalizes eigenvectors (complex) to unit norm
            a_sub = np.zeros((rank, rank))
            c = 0
            while c < rank:
                if abs(ev[c].imag) > 1e-9 * abs(ev[c].real) and c + 1 < rank:
                    a_sub[:, c] = evec[:, c].real
                    a_sub[:, c + 1] = evec[:, c].imag
                    c += 2
                else:
                    a_sub[:, c] = evec[:, c].real
                    c += 1
            a1 = self.u_r @ a_sub
            ok = True
            for c in range(rank):
                nrm = np.linalg.norm(a1[:, c])
                if nrm < K_DEGENERATE_NORM:
                    ok = False
                    break
                a1[:, c] /= nrm
            if not ok:
                continue
            h = cod_solve(a1, self.unf[self.m1])
            chain_modes = [n for n in range(order) if n != self.m1]
            chain_dims = [self.t.shape[n] for n in chain_modes]
            factors = [None] * order
            factors[self.m1] = a1
            for n in chain_modes:
                factors[n] = np.zeros((self.t.shape[n], rank))
            for r in range(rank):
                parts = peel_rank1(h[r, :], chain_dims)
                for k, n in enumerate(chain_modes):
                    factors[n][:, r] = parts[k]
            if not all(np.all(np.isfinite(f)) for f in factors):
                continue
            return factors, attempt
        return None


def gram_product(grams, skip: int) -> np.ndarray:
    """cp_als.cpp:193-206."""
    v = None
    for n, g in enumerate(grams):
        if n == skip:
            continue
        v = g.copy() if v is None else v * g
    return v


def als_solve_mode(unfolding: np.ndarray, factors, mode: int) -> np.ndarray:
    """cp_als.cpp:230-238."""
    chain = khatri_rao_chain(factors, mode)
    grams = [f.T @ f for f in factors]
    v = gram_product(grams, mode)
    mttkrp = unfolding @ chain
    return cod_solve(v, mttkrp.T).T


def cp_als(t: np.ndarray, cfg: AlsConfig) -> AlsResult:
    """cp_als.cpp:240-359."""
    if cfg.rank < 1:
        raise ConfigError("cp_als: rank must be >= 1")
    if cfg.max_iters < 1:
        raise ConfigError("cp_als: max_iters must be >= 1")
    if cfg.rel_tol <= 0.0:
        raise ConfigError("cp_als: rel_tol must be > 0")
    if cfg.n_restarts < 1:
        raise ConfigError("cp_als: n_restarts must be >= 1")
    order = t.ndim
    numel = t.size
    for n in range(order):
        others = 0 if t.shape[n] == 0 else numel // max(t.shape[n], 1)
        if cfg.rank > others:
            raise ConfigError("cp_als: rank %d exceeds solvability bound for mode %d" % (cfg.rank, n + 1))
    norm_x = frobenius_norm(t)
    if norm_x == 0.0:
        raise NumericError("cp_als: input tensor is identically zero")
    unf = [matricize(t, n) for n in range(order)]
    r = cfg.rank
    best = None
    best_fit = -math.inf
    gevd = GevdInit(t, unf, r)
    for restart in range(cfg.n_restarts):
        restart_seed = rng.derive(cfg.seed, [rng.K_ALS_RESTART, restart])
        init = gevd.factors(restart_seed)
        attempt = -1
        if init is not None:
            factors, attempt = init
        else:
            factors = []
            for n in range(order):
                s = rng.Substream(rng.derive(restart_seed, [rng.K_ALS_FACTOR, n]))
                factors.append(s.fill_uniform(t.shape[n], r))
        factors = [np.array(f, dtype=np.float64, order="F") for f in factors]
        grams = [f.T @ f for f in factors]
        lam = np.ones(r)
        prev_fit = 0.0
        rescued = False
        fits, residuals = [], []
        rescue = rng.Substream(rng.derive(restart_seed, [rng.K_ALS_RESCUE]))
        sweep = 0
        while sweep < cfg.max_iters:
            last_mttkrp = None
            for n in range(order):
                chain = khatri_rao_chain(factors, n)
                v = gram_product(grams, n)
                mttkrp = unf[n] @ chain
                raw = cod_solve(v, mttkrp.T).T
                if not np.all(np.isfinite(raw)):
                    raise NumericError("cp_als: non-finite factor at sweep %d, mode %d" % (sweep + 1, n + 1))
                raw = np.array(raw, order="F")
                for c in range(r):
                    nrm = np.linalg.norm(raw[:, c])
                    if nrm < K_DEGENERATE_NORM:
                        raw[:, c] = rescue.uniform01_array(raw.shape[0])
                        nrm = np.linalg.norm(raw[:, c])
                        rescued = True
                    lam[c] = nrm
                    raw[:, c] /= nrm
                factors[n] = raw
                grams[n] = raw.T @ raw
                if n == order - 1:
                    last_mttkrp = mttkrp
            inner = float(np.sum((last_mttkrp * factors[order - 1]) * lam[None, :]))
            full_gram = gram_product(grams, -1)
            norm_m_sq = float(lam @ (full_gram @ lam))
            res_sq = max(0.0, norm_x * norm_x - 2.0 * inner + norm_m_sq)
            residual = math.sqrt(res_sq)
            fit = 1.0 - residual / norm_x
            if not math.isfinite(fit):
                raise NumericError("cp_als: non-finite fit at sweep %d" % (sweep + 1))
            fits.append(fit)
            residuals.append(residual)
            if sweep > 0 and abs(fit - prev_fit) < cfg.rel_tol:
                sweep += 1
                break
            prev_fit = fit
            sweep += 1
        final_fit = fits[-1] if fits else -math.inf
        if final_fit > best_fit:
            best_fit = final_fit
            best = AlsResult(KruskalModel([f.copy() for f in factors], lam.copy()), final_fit,
                             sweep, fits, residuals, rescued, restart, attempt)
    return best


def reconstruct(m: KruskalModel) -> np.ndarray:
    """cp_als.cpp:361-367."""
    lam = m.lambda_ if len(m.lambda_) else np.ones(m.rank())
    out = None
    for r in range(m.rank()):
        term = rank1_outer([f[:, r] for f in m.factors]) * lam[r]
        out = term if out is None else out + term
    return out


def model_fit(t: np.ndarray, m: KruskalModel) -> float:
    """cp_als.cpp:369-380."""
    norm_x = frobenius_norm(t)
    if norm_x == 0.0:
        raise NumericError("model_fit: zero-norm tensor")
    rec = reconstruct(m)
    return 1.0 - math.sqrt(float(np.sum((t - rec) ** 2))) / norm_x


# ---------------------------------------------------------------------------
# recovery.cpp
# ---------------------------------------------------------------------------

K_RANK_TOL = 1e-10       # recovery.cpp:12
K_DEGENERATE_ROW = 1e-12  # recovery.cpp:13


def column_normalized(m: np.ndarray) -> np.ndarray:
    """recovery.cpp:15-22."""
    out = np.array(m, dtype=np.float64)
    for c in range(out.shape[1]):
        nrm = np.linalg.norm(out[:, c])
        if nrm > 0.0:
            out[:, c] /= nrm
    return out


def checked_solve(proj: np.ndarray, rhs: np.ndarray, mode: int) -> np.ndarray:
    """recovery.cpp:26-38."""
    if proj.shape[0] < proj.shape[1]:
        raise NumericError("recover: mode %d projection is %dx%d; p*Q must reach the mode extent "
                           "(raise p per the replica bound)" % (mode + 1, proj.shape[0], proj.shape[1]))
    rank, x = colpiv_qr_solve(proj, rhs, K_RANK_TOL)
    if rank < proj.shape[1]:
        raise NumericError("recover: rank-deficient projection on mode %d (rank %d of %d)"
                           % (mode + 1, rank, proj.shape[1]))
    return x


def greedy_match(sim: np.ndarray, tie_tol: float = 1e-9, log=None):
    """recovery.cpp:42-85."""
    r = sim.shape[0]
    if sim.shape[1] != r:
        raise ConfigError("greedy_match: similarity must be square")
    perm = [-1] * r
    ref_used = [False] * r
    cand_used = [False] * r
    for _ in range(r):
        best = -math.inf
        for i in range(r):
            if ref_used[i]:
                continue
            for j in range(r):
                if cand_used[j]:
                    continue
                best = max(best, sim[i, j])
        bi = bj = -1
        for i in range(r):
            if bi >= 0:
                break
            if ref_used[i]:
                continue
            for j in range(r):
                if cand_used[j]:
                    continue
                if sim[i, j] >= best - tie_tol:
                    bi, bj = i, j
                    break
        ties = 0
        for i in range(r):
            if ref_used[i]:
                continue
            for j in range(r):
                if not cand_used[j] and sim[i, j] >= best - tie_tol:
                    ties += 1
        if ties > 1 and log is not None:
            log.append("ambiguous match at similarity %f (%d candidates), resolved to lowest index"
                       % (best, ties))
        perm[bi] = bj
        ref_used[bi] = True
        cand_used[bj] = True
    return perm


def exhaustive_match(sim: np.ndarray):
    """recovery.cpp:87-104."""
    import itertools
    r = sim.shape[0]
    if r > 8:
        raise ConfigError("exhaustive_match: rank too large for enumeration")
    best, best_perm = -math.inf, list(range(r))
    for cand in itertools.permutations(range(r)):
        total = sum(sim[i, cand[i]] for i in range(r))
        if total > best:
            best, best_perm = total, list(cand)
    return best_perm


@dataclass
class AlignedStack:
    """recovery.hpp:26-37."""
    stacks: List[np.ndarray]
    perms: List[List[int]]
    scales: List[List[np.ndarray]]
    reference: int = 0
    min_match_similarity: float = 1.0
    max_offdiag_similarity: float = 0.0
    notes: List[str] = field(default_factory=list)


def align_replicas(models: List[KruskalModel], rs: ReplicaSet) -> AlignedStack:
    """recovery.cpp:106-291."""
    p = rs.p()
    if len(models) != p:
        raise ConfigError("align_replicas: expected %d models" % p)
    order = rs.order()
    rank = models[0].rank()
    for m in models:
        if m.rank() != rank or m.order() != order:
            raise ConfigError("align_replicas: models disagree on rank or order")
    if p >= 2 and rs.shared < 1:
        raise ConfigError("align_replicas: shared columns required to align multiple replicas")
    inv_order = 1.0 / order
    q = rs.q

    def redistributed(rep):
        lam = models[rep].lambda_
        root = np.array([max(l, 0.0) ** inv_order for l in lam])
        return [f * root[None, :] for f in models[rep].factors]

    out = AlignedStack([np.zeros((p * q, rank)) for _ in range(order)], [None] * p, [None] * p)
    ref = redistributed(0)
    for n in range(order):
        out.stacks[n][:q, :] = ref[n]
    out.perms[0] = list(range(rank))
    out.scales[0] = [np.ones(rank) for _ in range(order)]

    whiten = [None] * order
    if p >= 2:
        for n in range(order):
            if n == rs.temporal_mode:
                gram = rs.temporal_shared_gram
            else:
                u = rs.replicas[0].nontemporal[rs.nontemporal_slot(n)]
                us = u[:, :rs.shared]
                gram = us.T @ us
            if gram.shape == (rs.shared, rs.shared) and rs.shared > 0:
                try:
                    whiten[n] = np.linalg.cholesky(gram)
                except np.linalg.LinAlgError:
                    whiten[n] = None

    def shared_coords(factor, n):
        rows = factor[:rs.shared, :]
        if whiten[n] is not None:
            rows = sla.solve_triangular(whiten[n], rows, lower=True)
        return rows

    ref_shared = []
    for n in range(order):
        rsn = shared_coords(ref[n], n)
        ref_shared.append(rsn)
        for c in range(rank):
            if p >= 2 and np.linalg.norm(rsn[:, c]) < K_DEGENERATE_ROW:
                raise NumericError("align_replicas: degenerate shared rows in reference, mode %d" % (n + 1))

    pair_solve = p >= 2
    for d in rs.nontemporal_dims:
        if 2 * q < d + 1:
            pair_solve = False

    for rep in range(1, p):
        cand = redistributed(rep)
        cand_shared = [shared_coords(cand[n], n) for n in range(order)]
        if pair_solve:
            rms = np.zeros((rank, rank))
            modes_used = 0
            for n in range(order):
                if n == rs.temporal_mode:
                    continue
                slot = rs.nontemporal_slot(n)
                u_ref = rs.replicas[0].nontemporal[slot]
                u_rep = rs.replicas[rep].nontemporal[slot]
                joint = np.vstack([u_ref.T, u_rep.T])
                rb, cb = ref[n], cand[n]
                for i in range(rank):
                    for j in range(rank):
                        zr = ref_shared[n][:, i]
                        zc = cand_shared[n][:, j]
                        denom = float(zc @ zc)
                        s = float(zr @ zc) / denom if denom > 0.0 else 0.0
                        rhs = np.concatenate([rb[:, i], s * cb[:, j]])
                        x = np.linalg.lstsq(joint, rhs, rcond=None)[0]
                        rel = np.linalg.norm(joint @ x - rhs) / max(np.linalg.norm(rhs), 1e-300)
                        rms[i, j] += rel * rel
                modes_used += 1
            sim = 1.0 - np.minimum(1.0, np.sqrt(rms / max(modes_used, 1)))
        else:
            sim = np.ones((rank, rank))
            for n in range(order):
                r_n = column_normalized(ref_shared[n])
                c_n = cand_shared[n]
                for c in range(rank):
                    if np.linalg.norm(c_n[:, c]) < K_DEGENERATE_ROW:
                        raise NumericError("align_replicas: degenerate shared rows in replica %d, mode %d"
                                           % (rep + 1, n + 1))
                c_n = column_normalized(c_n)
                sim = sim * np.abs(r_n.T @ c_n)
        perm = greedy_match(sim, 1e-9, out.notes)
        for i in range(rank):
            out.min_match_similarity = min(out.min_match_similarity, sim[i, perm[i]])
            for j in range(rank):
                if j != perm[i]:
                    out.max_offdiag_similarity = max(out.max_offdiag_similarity, sim[i, j])
        mode_scales = [np.ones(rank) for _ in range(order)]
        for n in range(order):
            block = np.zeros((q, rank))
            for i in range(rank):
                j = perm[i]
                cr = cand_shared[n][:, j]
                rr = ref_shared[n][:, i]
                denom = float(cr @ cr)
                scale = float(rr @ cr) / denom if denom > 0.0 else 0.0
                if not math.isfinite(scale) or scale == 0.0:
                    raise NumericError("align_replicas: degenerate scale for replica %d, mode %d"
                                       % (rep + 1, n + 1))
                mode_scales[n][i] = scale
                block[:, i] = scale * cand[n][:, j]
            out.stacks[n][rep * q:(rep + 1) * q, :] = block
        out.perms[rep] = perm
        out.scales[rep] = mode_scales
    return out


def stack_projections(rs: ReplicaSet, mode: int, row_begin: int = 0, row_end: int = 0) -> np.ndarray:
    """recovery.cpp:293-313."""
    blocks = []
    for rep in rs.replicas:
        if mode == rs.temporal_mode:
            blocks.append(rep.temporal_rows(row_begin, row_end).T)
        else:
            blocks.append(rep.nontemporal[rs.nontemporal_slot(mode)].T)
    return np.vstack(blocks)


def recover_nontemporal(stacked_factor, stacked_projection, mode: int) -> np.ndarray:
    """recovery.cpp:315-319."""
    if stacked_factor.shape[0] != stacked_projection.shape[0]:
        raise ConfigError("recover_nontemporal: stack and projection row counts differ")
    return checked_solve(stacked_projection, stacked_factor, mode)


def recover_nontemporal_weighted(stacked_factor, stacked_projection, mode: int, q: int,
                                 col_weights) -> np.ndarray:
    """recovery.cpp:321-339."""
    if stacked_factor.shape[0] != stacked_projection.shape[0]:
        raise ConfigError("recover_nontemporal: stack and projection row counts differ")
    rank = stacked_factor.shape[1]
    out = np.zeros((stacked_projection.shape[1], rank))

    def one(r):
        w = np.repeat(col_weights[:, r], q)
        return checked_solve(stacked_projection * w[:, None], stacked_factor[:, r] * w, mode)

    # the R column solves are independent (the reference runs them in a
    # loop); the port spreads them over the host cores, lowest column's
    # error first
    for r, x in enumerate(parallel_columns(rank, one)):
        out[:, r] = x
    return out


@dataclass
class TemporalAppendResult:
    """recovery.hpp:71-74."""
    new_rows: np.ndarray
    solve_residual: float


def recover_temporal_append(temporal_stack, rs: ReplicaSet, summaries: SummaryState, c_old,
                            t_new: int, col_weights=None) -> TemporalAppendResult:
    """recovery.cpp:341-427."""
    p, q = rs.p(), rs.q
    rank = temporal_stack.shape[1]
    if temporal_stack.shape[0] != p * q:
        raise ConfigError("recover_temporal_append: stack rows != p*Q")
    if t_new < 1:
        raise ConfigError("recover_temporal_append: t_new must be >= 1")
    k_old = c_old.shape[0]
    history = np.zeros((p * q, rank))
    for rep in range(p):
        if summaries.history[rep].shape[1] == 0:
            summaries.history[rep] = np.zeros((q, rank))
        if summaries.history[rep].shape != (q, rank):
            raise ConfigError("recover_temporal_append: history accumulator shape mismatch")
        history[rep * q:(rep + 1) * q, :] = summaries.history[rep]
    proj = stack_projections(rs, rs.temporal_mode, k_old, k_old + t_new)
    if proj.shape[0] < proj.shape[1] + 1:
        raise NumericError("recover_temporal_append: p*Q too small for the batch extent")
    new_rows = np.zeros((t_new, rank))
    res_sq = rhs_sq = 0.0

    def one(r):
        rhs = temporal_stack[:, r].copy()
        hist_col = history[:, r].copy()
        wproj = proj.copy()
        if col_weights is not None:
            w = np.repeat(col_weights[:, r], q)
            rhs *= w
            hist_col *= w
            wproj *= w[:, None]
        if np.linalg.norm(hist_col) <= K_RANK_TOL * max(1.0, np.linalg.norm(rhs)):
            solved = checked_solve(wproj, rhs, rs.temporal_mode)
            fitted = rhs - wproj @ solved
        else:
            system = np.hstack([wproj, hist_col[:, None]])
            qrank, sol = colpiv_qr_solve(system, rhs, K_RANK_TOL)
            if qrank < system.shape[1]:
                raise NumericError("recover_temporal_append: rank-deficient joint system")
            gauge = float(sol[t_new])
            if not math.isfinite(gauge):
                raise NumericError("recover_temporal_append: non-finite history gauge")
            if abs(gauge - 1.0) > 0.5:
                solved = checked_solve(wproj, rhs - hist_col, rs.temporal_mode)
                gauge = 1.0
            else:
                solved = sol[:t_new] / gauge
            fitted = rhs - gauge * (hist_col + wproj @ solved)
        return solved, float(fitted @ fitted), float(rhs @ rhs)

    # independent per-column solves (a loop in the reference), spread over
    # the host cores; sums in column order
    for r, (solved, f2, r2) in enumerate(parallel_columns(rank, one)):
        new_rows[:, r] = solved
        res_sq += f2
        rhs_sq += r2
    rel = math.sqrt(res_sq / rhs_sq) if rhs_sq > 0.0 else 0.0
    for rep in range(p):
        w_new = rs.replicas[rep].temporal_rows(k_old, k_old + t_new)
        summaries.history[rep] = summaries.history[rep] + w_new.T @ new_rows
    return TemporalAppendResult(new_rows, rel)


def temporal_stack_from_summaries(rs: ReplicaSet, summaries: SummaryState, nontemporal_final) -> np.ndarray:
    """recovery.cpp:429-462."""
    p, q, order, tmode = rs.p(), rs.q, rs.order(), rs.temporal_mode
    if len(nontemporal_final) != order - 1:
        raise ConfigError("temporal_stack_from_summaries: need one factor per non-temporal mode")
    rank = nontemporal_final[0].shape[1]
    stack = np.zeros((p * q, rank))
    for rep in range(p):
        compressed = [None] * order
        slot = 0
        for n in range(order):
            if n == tmode:
                compressed[n] = np.zeros((q, rank))
                continue
            u = rs.replicas[rep].nontemporal[rs.nontemporal_slot(n)]
            compressed[n] = u.T @ nontemporal_final[slot]
            slot += 1
        chain = khatri_rao_chain(compressed, tmode)
        unfolding = matricize(summaries.y[rep], tmode)
        stack[rep * q:(rep + 1) * q, :] = cod_solve(chain, unfolding.T, 1e-8).T
    return stack


def refine_stack(aligned: AlignedStack, rs: ReplicaSet, nontemporal_solved) -> np.ndarray:
    """recovery.cpp:464-529."""
    p, q, tmode, order = rs.p(), rs.q, rs.temporal_mode, rs.order()
    rank = aligned.stacks[0].shape[1]
    weights = np.ones((p, rank))
    if len(nontemporal_solved) == 0:
        return weights
    for rep in range(p):
        temporal_scale = np.ones(rank)
        agreement = np.ones(rank)
        slot = 0
        for n in range(order):
            if n == tmode:
                continue
            u = rs.replicas[rep].nontemporal[rs.nontemporal_slot(n)]
            try:
                l = np.linalg.cholesky(u.T @ u)
                white = True
            except np.linalg.LinAlgError:
                white = False
            target = u.T @ nontemporal_solved[slot]
            block = aligned.stacks[n][rep * q:(rep + 1) * q, :]
            zt = sla.solve_triangular(l, target, lower=True) if white else target
            zb = sla.solve_triangular(l, block, lower=True) if white else block.copy()
            for r in range(rank):
                bb = float(zb[:, r] @ zb[:, r])
                bt = float(zb[:, r] @ zt[:, r])
                tt = float(zt[:, r] @ zt[:, r])
                scale = bt / bb if bb > 0.0 else 0.0
                cosine = bt / math.sqrt(bb * tt) if (bb > 0.0 and tt > 0.0) else 0.0
                if not math.isfinite(scale) or abs(scale) < 1e-3 or abs(scale) > 1e3:
                    agreement[r] = 0.0
                    continue
                block[:, r] *= scale
                temporal_scale[r] /= scale
                agreement[r] *= abs(cosine)
            slot += 1
        tblock = aligned.stacks[tmode][rep * q:(rep + 1) * q, :]
        for r in range(rank):
            if math.isfinite(temporal_scale[r]) and agreement[r] > 0.0:
                tblock[:, r] *= temporal_scale[r]
            a = agreement[r]
            weights[rep, r] = 0.0 if a <= 0.5 else ((a - 0.5) / 0.5) * ((a - 0.5) / 0.5)
    max_dim = max(rs.nontemporal_dims)
    for r in range(rank):
        mass = sum(q if weights[rep, r] > 0.0 else 0 for rep in range(p))
        if mass < max_dim + 1:
            weights[:, r] = 1.0
    return weights


def kruskal_check(q: int, k_ranks, rank: int) -> bool:
    """recovery.cpp:531-541."""
    if q < 1 or rank < 1:
        raise ConfigError("kruskal_check: Q and R must be >= 1")
    if len(k_ranks) < 2:
        raise ConfigError("kruskal_check: need k-ranks for >= 3 modes")
    s = 0
    for r in k_ranks:
        if r < 1:
            raise ConfigError("kruskal_check: k-ranks must be >= 1")
        s += min(q, r)
    return s >= 2 * rank + len(k_ranks) - 1


def replica_bound_nmode(nontemporal_dims, k_batch: int, q: int, shared: int) -> int:
    """recovery.cpp:548-557."""
    if q <= shared:
        raise ConfigError("replica_bound: requires Q > shared")
    if len(nontemporal_dims) == 0:
        raise ConfigError("replica_bound: no non-temporal dims")
    worst = (nontemporal_dims[0] - shared) / (q - shared)
    for d in nontemporal_dims[1:]:
        worst = max(worst, d / q)
    worst = max(worst, k_batch / q)
    return int(math.ceil(worst))


def replica_bound(i_dim, j_dim, k_batch, q, shared) -> int:
    """recovery.cpp:543-546."""
    return replica_bound_nmode([i_dim, j_dim], k_batch, q, shared)


@dataclass
class GaugeMatch:
    """recovery.hpp:117-123."""
    perm: List[int]
    signs: List[np.ndarray]
    norms: List[np.ndarray]


def match_columns(current, stored) -> GaugeMatch:
    """recovery.cpp:559-588."""
    if len(current) != len(stored) or len(current) == 0:
        raise ConfigError("match_columns: mode count mismatch")
    order = len(current)
    rank = current[0].shape[1]
    sim = np.ones((rank, rank))
    cur_unit = [column_normalized(c) for c in current]
    sto_unit = [column_normalized(s) for s in stored]
    for n in range(order):
        sim = sim * np.abs(sto_unit[n].T @ cur_unit[n])
    perm = greedy_match(sim)
    signs = [np.ones(rank) for _ in range(order)]
    norms = [np.ones(rank) for _ in range(order)]
    for n in range(order):
        for i in range(rank):
            j = perm[i]
            cosine = float(sto_unit[n][:, i] @ cur_unit[n][:, j])
            signs[n][i] = -1.0 if cosine < 0.0 else 1.0
            norms[n][i] = np.linalg.norm(current[n][:, j])
    return GaugeMatch(perm, signs, norms)


# ---------------------------------------------------------------------------
# streaming.cpp
# ---------------------------------------------------------------------------

@dataclass
class StreamConfig:
    """streaming.hpp:15-27."""
    rank: int = 1
    p: int = 1
    q: int = 1
    shared: int = 0
    temporal_mode: int = -1
    als: AlsConfig = field(default_factory=AlsConfig)
    seed: int = 0
    enforce_bounds: bool = False
    workers: int = 0
    strict: bool = False
    residual_warning: float = 1e-3


@dataclass
class BatchRecord:
    """streaming.hpp:31-42."""
    batch_index: int = 0
    t_new: int = 0
    temporal_residual: float = 0.0
    min_match_similarity: float = 1.0
    max_offdiag_similarity: float = 0.0
    warned: bool = False
    compress_seconds: float = 0.0
    als_seconds: float = 0.0
    recover_seconds: float = 0.0
    total_seconds: float = 0.0


@dataclass
class StreamState:
    """streaming.hpp:48-59."""
    config: StreamConfig
    replicas: ReplicaSet
    summaries: SummaryState
    model: Optional[KruskalModel] = None
    slices_seen: int = 0
    log: List[BatchRecord] = field(default_factory=list)
    replica_models: List[KruskalModel] = field(default_factory=list)  # oracle-only diagnostic


def validate_config(cfg: StreamConfig, order: int) -> None:
    """streaming.cpp:23-34."""
    if order < 3:
        raise ConfigError("stream: tensor order must be >= 3")
    if cfg.rank < 1:
        raise ConfigError("stream: rank must be >= 1")
    if cfg.p < 1:
        raise ConfigError("stream: p must be >= 1")
    if cfg.q < 1:
        raise ConfigError("stream: Q must be >= 1")
    if cfg.shared < 0 or cfg.shared >= cfg.q:
        raise ConfigError("stream: shared must lie in [0, Q)")
    if cfg.temporal_mode >= order:
        raise ConfigError("stream: temporal mode out of range")
    if cfg.p >= 2 and cfg.shared < 1:
        raise ConfigError("stream: alignment across replicas needs shared >= 1")


def _recover_batch(aligned: AlignedStack, rs: ReplicaSet, summaries: SummaryState,
                   stored_nontemporal, c_old_raw, t_new: int):
    """streaming.cpp:89-160."""
    final, weights = _recover_nontemporal_final(aligned, rs, stored_nontemporal)
    tstack = temporal_stack_from_summaries(rs, summaries, final)
    temporal = recover_temporal_append(tstack, rs, summaries, c_old_raw, t_new)
    return final, temporal, weights


def _recover_nontemporal_final(aligned: AlignedStack, rs: ReplicaSet, stored_nontemporal):
    """streaming.cpp:89-148: solves, two refinement passes, gauge match."""
    order = rs.order()
    rank = aligned.stacks[0].shape[1]
    tmode = rs.temporal_mode
    projs, solved = [], []
    for n in range(order):
        if n == tmode:
            continue
        projs.append(stack_projections(rs, n))
        solved.append(recover_nontemporal(aligned.stacks[n], projs[-1], n))
    weights = np.ones((rs.p(), rank))
    for _ in range(2):
        weights = refine_stack(aligned, rs, solved)
        slot = 0
        for n in range(order):
            if n == tmode:
                continue
            solved[slot] = recover_nontemporal_weighted(aligned.stacks[n], projs[slot], n, rs.q, weights)
            slot += 1
    if len(stored_nontemporal) == 0:
        perm = list(range(rank))
        signs = [np.ones(rank) for _ in solved]
    else:
        gm = match_columns(solved, stored_nontemporal)
        perm, signs = gm.perm, gm.signs
    final = []
    for m, s in enumerate(solved):
        fin = np.zeros((s.shape[0], rank))
        for i in range(rank):
            j = perm[i]
            nrm = np.linalg.norm(s[:, j])
            if nrm <= 0.0:
                raise NumericError("recover: zero column in recovered factor")
            fin[:, i] = s[:, j] * (signs[m][i] / nrm)
        final.append(fin)
    return final, weights


def _assemble_model(nontemporal, temporal_raw, tmode: int) -> KruskalModel:
    """streaming.cpp:162-177."""
    order = len(nontemporal) + 1
    factors = []
    slot = 0
    for n in range(order):
        if n == tmode:
            factors.append(np.array(temporal_raw, dtype=np.float64))
        else:
            factors.append(np.array(nontemporal[slot], dtype=np.float64))
            slot += 1
    m = KruskalModel(factors, np.ones(temporal_raw.shape[1]))
    m.normalize()
    return m


def _nontemporal_dims_of(t, tmode):
    return [t.shape[n] for n in range(t.ndim) if n != tmode]


def resolve_workers(cfg) -> int:
    """streaming.cpp:36-41: workers = cfg.workers, or min(hardware
    concurrency, p) when 0."""
    import os
    w = cfg.workers if cfg.workers > 0 else min(os.cpu_count() or 1, cfg.p)
    return max(1, min(w, cfg.p))


def parallel_replicas(n: int, workers: int, fn):
    """streaming.cpp:45-69: fn(i) for i in [0, n) on `workers` threads; slot
    i is written only by iteration i (deterministic for any worker count);
    the first exception (lowest index) is rethrown after the join.  BLAS runs
    single-threaded inside each worker (the reference's Eigen is)."""
    if workers <= 1 or n <= 1:
        return [fn(i) for i in range(n)]
    from concurrent.futures import ThreadPoolExecutor
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    out = [None] * n
    errs = [None] * n

    def run(i):
        try:
            out[i] = fn(i)
        except Exception as e:  # noqa: BLE001
            errs[i] = e

    if threadpool_limits is not None:
        with threadpool_limits(limits=1):
            with ThreadPoolExecutor(max_workers=workers) as ex:
                list(ex.map(run, range(n)))
    else:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(run, range(n)))
    for e in errs:
        if e is not None:
            raise e
    return out


# scipy's LAPACK wrappers hold the GIL, so threads do not overlap the merge's
# pivoted QRs; the CPU-baseline legs of bench.py set this to run those
# independent column solves in forked worker processes instead (tests keep
# the default: forking a process that drives a GPU is not worth the risk).
MERGE_PROCESSES = False
_FORK_FN = None


def _fork_call(i):
    return _FORK_FN(i)


def parallel_columns(n: int, fn):
    """fn(i) for the independent per-column solves of the merge, in column
    order, over the host cores (processes when MERGE_PROCESSES, else threads)."""
    import os
    workers = min(n, os.cpu_count() or 1)
    if not MERGE_PROCESSES or workers <= 1 or n <= 1:
        return parallel_replicas(n, workers, fn)
    global _FORK_FN
    import multiprocessing as mp
    _FORK_FN = fn
    try:
        with mp.get_context("fork").Pool(workers) as pool:
            return pool.map(_fork_call, range(n), chunksize=1)
    finally:
        _FORK_FN = None


def _run_replica_als(st: StreamState, batch_index: int):
    cfg = st.config

    def one(r):
        als = AlsConfig(cfg.rank, cfg.als.max_iters, cfg.als.rel_tol, cfg.als.n_restarts,
                        rng.derive(cfg.seed, [rng.K_STREAM_ALS, r, batch_index]))
        return cp_als(st.summaries.y[r], als).model

    return parallel_replicas(cfg.p, resolve_workers(cfg), one)


def init_stream(first_batch: np.ndarray, cfg_in: StreamConfig) -> StreamState:
    """streaming.cpp:181-256."""
    import copy
    cfg = copy.deepcopy(cfg_in)
    order = first_batch.ndim
    if cfg.temporal_mode < 0:
        cfg.temporal_mode = order - 1
    validate_config(cfg, order)
    cfg.als.rank = cfg.rank
    tmode = cfg.temporal_mode
    t0 = first_batch.shape[tmode]
    if t0 < 1:
        raise ConfigError("init_stream: first batch has no temporal extent")
    nt = _nontemporal_dims_of(first_batch, tmode)
    if cfg.enforce_bounds:
        need = replica_bound_nmode(nt, t0, cfg.q, cfg.shared)
        if cfg.p < need:
            raise ConfigError("init_stream: p=%d below the replica bound; need p >= %d" % (cfg.p, need))
        kranks = [min(first_batch.shape[n], cfg.rank) for n in range(order)]
        if not kruskal_check(cfg.q, kranks, cfg.rank):
            raise ConfigError("init_stream: compressed decomposition fails the identifiability bound")
    rs = gen_replicas(nt, cfg.q, cfg.p, cfg.shared, cfg.seed, tmode)
    st = StreamState(cfg, rs, init_summaries(rs))
    rec = BatchRecord(0, t0)
    import time as _time
    t_begin = _time.perf_counter()
    extend_temporal(st.replicas, t0)
    z = parallel_replicas(cfg.p, resolve_workers(cfg), lambda r: compress(first_batch, st.replicas, r, 0, t0))
    update_summaries(st.summaries, z)
    t_c = _time.perf_counter()
    rec.compress_seconds = t_c - t_begin
    models = _run_replica_als(st, 0)
    st.replica_models = models
    t_a = _time.perf_counter()
    rec.als_seconds = t_a - t_c
    aligned = align_replicas(models, st.replicas)
    rec.min_match_similarity = aligned.min_match_similarity
    rec.max_offdiag_similarity = aligned.max_offdiag_similarity
    final, temporal, _ = _recover_batch(aligned, st.replicas, st.summaries, [], np.zeros((0, cfg.rank)), t0)
    rec.temporal_residual = temporal.solve_residual
    rec.warned = temporal.solve_residual > cfg.residual_warning
    if rec.warned and cfg.strict:
        raise NumericError("init_stream: temporal solve residual %f exceeds strict threshold"
                           % temporal.solve_residual)
    st.model = _assemble_model(final, temporal.new_rows, tmode)
    drop_temporal_history(st.replicas)
    st.slices_seen = t0
    rec.recover_seconds = _time.perf_counter() - t_a
    rec.total_seconds = _time.perf_counter() - t_begin
    st.log.append(rec)
    return st


def ingest_batch(st: StreamState, batch: np.ndarray) -> None:
    """streaming.cpp:258-346 (strict rollback restated with a deep copy)."""
    import copy
    order = st.replicas.order()
    tmode = st.replicas.temporal_mode
    if batch.ndim != order:
        raise ConfigError("ingest_batch: batch order mismatch at batch %d" % st.summaries.batches_seen)
    for n in range(order):
        if n != tmode and batch.shape[n] != st.model.factors[n].shape[0]:
            raise ConfigError("ingest_batch: extent mismatch on mode %d at batch %d"
                              % (n + 1, st.summaries.batches_seen))
    t_new = batch.shape[tmode]
    if t_new < 1:
        raise ConfigError("ingest_batch: batch has no temporal extent")
    backup = copy.deepcopy(st) if st.config.strict else None
    context = "batch %d: " % st.summaries.batches_seen
    try:
        import time as _time
        t_begin = _time.perf_counter()
        rec = BatchRecord(st.summaries.batches_seen, t_new)
        k_old = st.slices_seen
        extend_temporal(st.replicas, t_new)
        z = parallel_replicas(st.config.p, resolve_workers(st.config),
                              lambda r: compress(batch, st.replicas, r, k_old, k_old + t_new))
        update_summaries(st.summaries, z)
        t_c = _time.perf_counter()
        rec.compress_seconds = t_c - t_begin
        models = _run_replica_als(st, rec.batch_index)
        st.replica_models = models
        t_a = _time.perf_counter()
        rec.als_seconds = t_a - t_c
        aligned = align_replicas(models, st.replicas)
        rec.min_match_similarity = aligned.min_match_similarity
        rec.max_offdiag_similarity = aligned.max_offdiag_similarity
        stored = [st.model.factors[n] for n in range(order) if n != tmode]
        c_old_raw = st.model.factors[tmode] * st.model.lambda_[None, :]
        final, temporal, _ = _recover_batch(aligned, st.replicas, st.summaries, stored, c_old_raw, t_new)
        rec.temporal_residual = temporal.solve_residual
        rec.warned = temporal.solve_residual > st.config.residual_warning
        if rec.warned and st.config.strict:
            raise NumericError("temporal solve residual %f exceeds strict threshold" % temporal.solve_residual)
        temporal_raw = np.vstack([c_old_raw, temporal.new_rows])
        st.model = _assemble_model(final, temporal_raw, tmode)
        drop_temporal_history(st.replicas)
        st.slices_seen += t_new
        rec.recover_seconds = _time.perf_counter() - t_a
        rec.total_seconds = _time.perf_counter() - t_begin
        st.log.append(rec)
    except ConfigError as e:
        if backup is not None:
            st.__dict__.update(backup.__dict__)
        raise ConfigError(context + str(e)) from None
    except NumericError as e:
        if backup is not None:
            st.__dict__.update(backup.__dict__)
        raise NumericError(context + str(e)) from None


# ---------------------------------------------------------------------------
# eval.cpp / commands.cpp (parity harness helpers)
# ---------------------------------------------------------------------------

def fitness(x: np.ndarray, x_hat: np.ndarray) -> float:
    """eval.cpp:10-20."""
    norm_x = frobenius_norm(x)
    if norm_x == 0.0:
        raise NumericError("fitness: zero-norm reference tensor")
    d = (x - x_hat).ravel()
    return 100.0 * (1.0 - math.sqrt(float(d @ d)) / norm_x)


def congruence(ground: KruskalModel, est: KruskalModel):
    """eval.cpp:22-46 (factor match score per component)."""
    rank = ground.rank()
    sim = np.ones((rank, rank))
    for g, e in zip(ground.factors, est.factors):
        sim = sim * np.abs(column_normalized(g).T @ column_normalized(e))
    perm = exhaustive_match(sim) if rank <= 6 else greedy_match(sim)
    return [float(sim[i, perm[i]]) for i in range(rank)]


# ---------------------------------------------------------------------------
# checkpoint.cpp -- the OCTS container (format only; test infrastructure)
# ---------------------------------------------------------------------------

def _crc64(data: bytes) -> int:
    """checkpoint.cpp:17-31 -- CRC-64/ECMA-182, bit-reflected."""
    table = _crc64.table if hasattr(_crc64, "table") else None
    if table is None:
        poly = 0xC96C5795D7870F42
        table = []
        for i in range(256):
            c = i
            for _ in range(8):
                c = (c >> 1) ^ (poly if c & 1 else 0)
            table.append(c)
        _crc64.table = table
    c = 0xFFFFFFFFFFFFFFFF
    for b in data:
        c = table[(c ^ b) & 0xFF] ^ (c >> 8)
    return c ^ 0xFFFFFFFFFFFFFFFF


def checkpoint_save(st: StreamState) -> bytes:
    """checkpoint.cpp:168-219 (native little-endian)."""
    import struct
    out = bytearray()

    def u8(v): out.extend(struct.pack("<B", v))
    def u32(v): out.extend(struct.pack("<I", v & 0xFFFFFFFF))
    def u64(v): out.extend(struct.pack("<Q", v & 0xFFFFFFFFFFFFFFFF))
    def i64(v): out.extend(struct.pack("<q", v))
    def f64(v): out.extend(struct.pack("<d", v))

    def matrix(m):
        m = np.asarray(m, dtype=np.float64)
        i64(m.shape[0])
        i64(m.shape[1])
        out.extend(np.asfortranarray(m).tobytes(order="F"))

    c = st.config
    for v in (c.rank, c.p, c.q, c.shared, c.temporal_mode):
        u32(v)
    u64(c.seed)
    u8(1 if c.enforce_bounds else 0)
    u32(0)
    u8(1 if c.strict else 0)
    f64(c.residual_warning)
    u32(c.als.rank)
    u32(c.als.max_iters)
    f64(c.als.rel_tol)
    u32(c.als.n_restarts)
    u64(c.als.seed)
    rs = st.replicas
    u64(rs.seed)
    u32(rs.q)
    u32(rs.shared)
    u32(rs.temporal_mode)
    i64(rs.batches_drawn)
    u64(len(rs.nontemporal_dims))
    for d in rs.nontemporal_dims:
        i64(d)
    matrix(rs.temporal_shared_gram if rs.temporal_shared_gram is not None else np.zeros((rs.shared, rs.shared)))
    u32(rs.p())
    for rep in rs.replicas:
        u32(rep.replica_id)
        u64(len(rep.nontemporal))
        for m in rep.nontemporal:
            matrix(m)
        i64(rep.temporal_window_start)
        i64(rep.temporal_rows_total)
        matrix(rep.temporal)
    sm = st.summaries
    i64(sm.batches_seen)
    u64(len(sm.y))
    for y, h in zip(sm.y, sm.history):
        u64(y.ndim)
        for d in y.shape:
            i64(d)
        u64(y.size)
        out.extend(np.asfortranarray(y).tobytes(order="F"))
        matrix(h)
    u32(len(st.model.factors))
    for f in st.model.factors:
        matrix(f)
    i64(len(st.model.lambda_))
    out.extend(np.asarray(st.model.lambda_, dtype=np.float64).tobytes())
    i64(st.slices_seen)
    u64(len(st.log))
    for r in st.log:
        i64(r.batch_index)
        i64(r.t_new)
        f64(r.temporal_residual)
        f64(r.min_match_similarity)
        f64(r.max_offdiag_similarity)
        u8(1 if r.warned else 0)
    payload = bytes(out)
    return b"OCTS" + struct.pack("<IQQ", 1, len(payload), _crc64(payload)) + payload


def checkpoint_load(data: bytes) -> StreamState:
    """checkpoint.cpp:222-295 (header checks in the reference's order)."""
    import struct
    if len(data) < 24 or data[:4] != b"OCTS":
        raise IoError("checkpoint: bad magic")
    version, plen, crc = struct.unpack("<IQQ", data[4:24])
    if version != 1:
        raise IoError("checkpoint: unsupported format version %d" % version)
    if len(data) != 24 + plen:
        raise IoError("checkpoint: payload length mismatch (corrupt or truncated)")
    payload = data[24:]
    if _crc64(payload) != crc:
        raise IoError("checkpoint: checksum mismatch")
    pos = [0]

    def take(fmt):
        n = struct.calcsize(fmt)
        if pos[0] + n > len(payload):
            raise IoError("checkpoint: truncated payload")
        v = struct.unpack(fmt, payload[pos[0]:pos[0] + n])
        pos[0] += n
        return v[0] if len(v) == 1 else v

    def doubles(n):
        if pos[0] + 8 * n > len(payload):
            raise IoError("checkpoint: truncated payload")
        v = np.frombuffer(payload, dtype="<f8", count=n, offset=pos[0]).copy()
        pos[0] += 8 * n
        return v

    def matrix():
        r, c_ = take("<q"), take("<q")
        if r < 0 or c_ < 0:
            raise IoError("checkpoint: negative matrix extent")
        return doubles(r * c_).reshape((r, c_), order="F")

    cfg = StreamConfig()
    cfg.rank, cfg.p, cfg.q, cfg.shared, cfg.temporal_mode = (take("<I") for _ in range(5))
    cfg.seed = take("<Q")
    cfg.enforce_bounds = take("<B") != 0
    cfg.workers = take("<I")
    cfg.strict = take("<B") != 0
    cfg.residual_warning = take("<d")
    cfg.als = AlsConfig(take("<I"), take("<I"), take("<d"), take("<I"), take("<Q"))
    rseed = take("<Q")
    q, shared, tmode = take("<I"), take("<I"), take("<I")
    drawn = take("<q")
    nd = take("<Q")
    dims = [take("<q") for _ in range(nd)]
    tg = matrix()
    p = take("<I")
    reps = []
    for _ in range(p):
        rid = take("<I")
        nm = take("<Q")
        mats = [matrix() for _ in range(nm)]
        ws, tot = take("<q"), take("<q")
        reps.append(CompressionReplica(rid, mats, matrix(), ws, tot))
    rs = ReplicaSet(reps, rseed, q, shared, tmode, dims, drawn, tg)
    seen = take("<q")
    ns = take("<Q")
    ys, hs = [], []
    for _ in range(ns):
        nd2 = take("<Q")
        shape = [take("<q") for _ in range(nd2)]
        n = take("<Q")
        ys.append(doubles(n).reshape(shape, order="F"))
        hs.append(matrix())
    order = take("<I")
    factors = [matrix() for _ in range(order)]
    lam = doubles(take("<q"))
    st = StreamState(cfg, rs, SummaryState(ys, hs, seen), KruskalModel(factors, lam))
    st.slices_seen = take("<q")
    nlog = take("<Q")
    for _ in range(nlog):
        rec = BatchRecord(take("<q"), take("<q"))
        rec.temporal_residual, rec.min_match_similarity, rec.max_offdiag_similarity = take("<d"), take("<d"), take("<d")
        rec.warned = take("<B") != 0
        st.log.append(rec)
    if pos[0] != len(payload):
        raise IoError("checkpoint: trailing bytes after payload")
    return st


def memory_account(cfg, nontemporal_dims, t_old: int, t_new: int) -> dict:
    """eval.cpp:62-86 -- element counts of the streaming state against the
    paper's space formula."""
    if cfg.q < 1 or cfg.p < 1 or cfg.rank < 1:
        raise ConfigError("memory_account: invalid configuration")
    order = len(nontemporal_dims) + 1
    t_sum = int(sum(nontemporal_dims))
    q_pow = cfg.q ** order
    sm = {
        "predicted_replica_elements": cfg.p * cfg.q * t_sum,
        "predicted_summary_elements": cfg.p * q_pow,
        "predicted_factor_elements": (t_sum + t_old + t_new) * cfg.rank + cfg.rank,
        "predicted_accumulator_elements": cfg.p * cfg.q * cfg.rank,
    }
    sm["predicted_elements"] = sum(sm.values())
    sm["formula_elements"] = cfg.p * cfg.q * (cfg.p * t_sum + t_new + cfg.rank) + (t_sum + t_old) * cfg.rank + q_pow
    sm["ratio"] = sm["predicted_elements"] / sm["formula_elements"]
    return sm


def measure_footprint(st) -> dict:
    """eval.cpp:48-60 -- bytes of the state as stored (8 per double); the
    temporal window is empty between batches (drop_temporal_history)."""
    fp = {"replica_bytes": 0, "summary_bytes": 0, "factor_bytes": 0, "accumulator_bytes": 0}
    for rep in st.replicas.replicas:
        fp["replica_bytes"] += sum(8 * m.size for m in rep.nontemporal) + 8 * rep.temporal.size
    fp["summary_bytes"] = sum(8 * y.size for y in st.summaries.y)
    fp["factor_bytes"] = sum(8 * f.size for f in st.model.factors) + 8 * len(st.model.lambda_)
    fp["accumulator_bytes"] = sum(8 * h.size for h in st.summaries.history)
    return fp


def generate_synthetic(dims, rank: int, seed: int, noise_mu: float = 0.0, noise_sigma: float = 0.0,
                       exact_noise: bool = True):
    """commands.cpp:110-134 -- U(0,1) factors from {9,n}, lambda = 1,
    X = reconstruct + N(mu, sigma) in flat order from {10}."""
    factors = []
    for n, d in enumerate(dims):
        s = rng.Substream(rng.derive(seed, [rng.K_SYNTH_FACTOR, n]))
        factors.append(s.fill_uniform(d, rank))
    model = KruskalModel(factors, np.ones(rank))
    t = reconstruct_fast(model)
    if noise_sigma > 0.0 or noise_mu != 0.0:
        s = rng.Substream(rng.derive(seed, [rng.K_SYNTH_NOISE]))
        n = t.size
        if exact_noise:
            noise = np.array([s.normal(noise_mu, noise_sigma) for _ in range(n)])
        else:
            noise = s.normal_array(n, noise_mu, noise_sigma)
        flat = t.ravel(order="F") + noise
        t = flat.reshape(t.shape, order="F")
    model.normalize()
    return t, model


def reconstruct_fast(m: KruskalModel) -> np.ndarray:
    """reconstruct (cp_als.cpp:361-367) via the unfolding identity
    X_(0) = A diag(lambda) KR(...)^T."""
    chain = khatri_rao_chain(m.factors, 0)
    lam = m.lambda_ if len(m.lambda_) else np.ones(m.rank())
    unf = (m.factors[0] * lam[None, :]) @ chain.T
    return dematricize(unf, [f.shape[0] for f in m.factors], 0)
