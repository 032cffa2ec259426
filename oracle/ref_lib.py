"""TEST INFRASTRUCTURE ONLY: ctypes binding of the reference library compiled
from its own sources (oracle/Makefile -> oracle/_ref/libcpstream_ref.so).

Only tests/, the golden-fixture scripts and bench.py's CPU reference arm use
this; the product never does.  The library is built here (where
/root/reference exists) and travels to the GPU box with the repo snapshot.
Errors come back as the oracle's exception classes (ConfigError,
NumericError, IoError) carrying the reference's own messages.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

from . import octen_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libcpstream_ref.so")
REF_SRC = "/root/reference/proj"

_lib = None


def build(quiet: bool = True) -> bool:
    """Compile the reference + stand-ins (only where the sources exist)."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(LIB_PATH)
    r = subprocess.run(["make", "-C", HERE, "-j16", "all"], capture_output=quiet, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle/_ref build failed:\n" + (r.stderr or "")[-4000:])
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(LIB_PATH + " (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        P, I, I64, D, U64 = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64
        pd, pi, pi64, pv = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_void_p)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_set_blas_threads": (None, [I]),
            "ref_generate_synthetic": (I, [I, pi64, I, D, D, U64, pd, pd, pd]),
            "ref_cp_als": (I, [I, pi64, pd, I, I, D, I, U64, pd, pd, pd, pi, pd, pi]),
            "ref_stream_init": (I, [I, pi64, pd, I, I, I, I, I, I, D, I, U64, I, I, I, D, pv]),
            "ref_stream_ingest": (I, [P, I, pi64, pd]),
            "ref_stream_free": (None, [P]),
            "ref_stream_info": (I, [P, pi64]),
            "ref_stream_model": (I, [P, pd, pd]),
            "ref_stream_summaries": (I, [P, pd, pd]),
            "ref_stream_log": (I, [P, pd]),
            "ref_stream_timers": (I, [P, pd]),
            "ref_stream_checkpoint_size": (I, [P, pi64]),
            "ref_stream_checkpoint": (I, [P, C.POINTER(C.c_uint8), I64]),
            "ref_stream_load": (I, [C.POINTER(C.c_uint8), I64, pv]),
            "ref_fitness": (I, [I64, pd, pd, pd]),
            "ref_congruence": (I, [I, pi64, I, pd, pd, pd, pd, pd]),
            "ref_reconstruct": (I, [I, pi64, I, pd, pd, pd]),
            "ref_run_stream_synth": (I, [I, pi64, I, D, D, U64, I, I, I, U64, I, I, D, I, I64, I, pd]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        L.ref_set_blas_threads(1)
        _lib = L
    return _lib


_ERR = {1: O.ConfigError, 2: O.NumericError, 3: O.IoError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().ref_last_error().decode()
        raise _ERR.get(rc, RuntimeError)(msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64(v: Sequence[int]):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.int64))
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


def _flat(t: np.ndarray) -> np.ndarray:
    """First-index-fastest (Fortran-order) flat copy."""
    return np.ascontiguousarray(np.asarray(t, dtype=np.float64).ravel(order="F"))


def _split_factors(flat: np.ndarray, dims: Sequence[int], rank: int) -> List[np.ndarray]:
    out, off = [], 0
    for d in dims:
        out.append(flat[off:off + d * rank].reshape((d, rank), order="F").copy())
        off += d * rank
    return out


def _model(factors, lam) -> O.KruskalModel:
    return O.KruskalModel([np.asarray(f, dtype=np.float64) for f in factors], np.asarray(lam, dtype=np.float64))


def generate_synthetic(dims, rank: int, seed: int, noise_mu: float = 0.0, noise_sigma: float = 0.0):
    """-> (tensor, truth KruskalModel); proj/src/commands.cpp:110-134."""
    dims = [int(d) for d in dims]
    n = int(np.prod(dims))
    t = np.empty(n)
    f = np.empty(sum(dims) * rank)
    lam = np.empty(rank)
    da, dp = _i64(dims)
    _check(lib().ref_generate_synthetic(len(dims), dp, rank, noise_mu, noise_sigma, seed, _dptr(t), _dptr(f),
                                        _dptr(lam)))
    return t.reshape(dims, order="F"), _model(_split_factors(f, dims, rank), lam)


class AlsOut:
    def __init__(self, model, fit, iterations, fit_history, rescued):
        self.model, self.fit, self.iterations = model, fit, iterations
        self.fit_history, self.rescued_degenerate = fit_history, rescued


def cp_als(t: np.ndarray, rank: int, max_iters: int = 100, rel_tol: float = 1e-8, n_restarts: int = 3,
           seed: int = 0) -> AlsOut:
    """proj/src/cp_als.cpp:240-359 on a dense tensor."""
    dims = list(t.shape)
    x = _flat(t)
    f = np.empty(sum(dims) * rank)
    lam = np.empty(rank)
    fit = C.c_double()
    iters = C.c_int()
    resc = C.c_int()
    hist = np.empty(max_iters)
    da, dp = _i64(dims)
    _check(lib().ref_cp_als(len(dims), dp, _dptr(x), rank, max_iters, rel_tol, n_restarts, seed, _dptr(f),
                            _dptr(lam), C.byref(fit), C.byref(iters), _dptr(hist), C.byref(resc)))
    k = iters.value
    return AlsOut(_model(_split_factors(f, dims, rank), lam), fit.value, k, list(hist[:k]), bool(resc.value))


class RefStream:
    """init_stream / ingest_batch of the reference (proj/src/streaming.cpp)."""

    def __init__(self, first_batch: np.ndarray, cfg: O.StreamConfig):
        dims = list(first_batch.shape)
        x = _flat(first_batch)
        da, dp = _i64(dims)
        h = C.c_void_p()
        tm = cfg.temporal_mode if cfg.temporal_mode is not None else -1
        _check(lib().ref_stream_init(len(dims), dp, _dptr(x), cfg.rank, cfg.p, cfg.q, cfg.shared, int(tm),
                                     cfg.als.max_iters, cfg.als.rel_tol, cfg.als.n_restarts, cfg.seed,
                                     int(bool(cfg.enforce_bounds)), int(cfg.workers), int(bool(cfg.strict)),
                                     float(cfg.residual_warning), C.byref(h)))
        self.h = h

    @classmethod
    def _from_handle(cls, h):
        s = cls.__new__(cls)
        s.h = h
        return s

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ref_stream_free(h)
            self.h = None

    def ingest(self, batch: np.ndarray) -> None:
        dims = list(batch.shape)
        x = _flat(batch)
        da, dp = _i64(dims)
        _check(lib().ref_stream_ingest(self.h, len(dims), dp, _dptr(x)))

    def info(self) -> dict:
        out = np.zeros(9 + 16, dtype=np.int64)
        _check(lib().ref_stream_info(self.h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        order = int(out[0])
        return dict(order=order, rank=int(out[1]), p=int(out[2]), q=int(out[3]), shared=int(out[4]),
                    temporal_mode=int(out[5]), slices_seen=int(out[6]), batches_seen=int(out[7]),
                    log_size=int(out[8]), dims=[int(v) for v in out[9:9 + order]])

    def model(self) -> O.KruskalModel:
        i = self.info()
        f = np.empty(sum(i["dims"]) * i["rank"])
        lam = np.empty(i["rank"])
        _check(lib().ref_stream_model(self.h, _dptr(f), _dptr(lam)))
        return _model(_split_factors(f, i["dims"], i["rank"]), lam)

    def summaries(self) -> np.ndarray:
        """(p, Q, ..., Q) replica summaries y_p."""
        i = self.info()
        n = i["q"] ** i["order"]
        y = np.empty(i["p"] * n)
        _check(lib().ref_stream_summaries(self.h, _dptr(y), None))
        return np.stack([y[k * n:(k + 1) * n].reshape([i["q"]] * i["order"], order="F") for k in range(i["p"])])

    def history(self) -> np.ndarray:
        i = self.info()
        h = np.empty(i["p"] * i["q"] * i["rank"])
        _check(lib().ref_stream_summaries(self.h, None, _dptr(h)))
        return h.reshape((i["p"], i["rank"], i["q"])).transpose(0, 2, 1).copy()

    def log(self) -> List[dict]:
        n = self.info()["log_size"]
        out = np.empty(max(1, n * 6))
        _check(lib().ref_stream_log(self.h, _dptr(out)))
        keys = ("batch_index", "t_new", "temporal_residual", "min_match_similarity", "max_offdiag_similarity",
                "warned")
        return [dict(zip(keys, out[6 * b:6 * b + 6])) for b in range(n)]

    def timers(self) -> np.ndarray:
        n = self.info()["log_size"]
        out = np.empty(max(1, n * 4))
        _check(lib().ref_stream_timers(self.h, _dptr(out)))
        return out[:n * 4].reshape(n, 4)

    def checkpoint(self) -> bytes:
        n = C.c_int64()
        _check(lib().ref_stream_checkpoint_size(self.h, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _check(lib().ref_stream_checkpoint(self.h, buf, n.value))
        return bytes(buf)

    @classmethod
    def load(cls, data: bytes) -> "RefStream":
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        h = C.c_void_p()
        _check(lib().ref_stream_load(buf, len(data), C.byref(h)))
        return cls._from_handle(h)


def congruence(ground: O.KruskalModel, est: O.KruskalModel) -> np.ndarray:
    dims = [f.shape[0] for f in ground.factors]
    rank = ground.factors[0].shape[1]
    gf = np.concatenate([np.asarray(f, dtype=np.float64).ravel(order="F") for f in ground.factors])
    ef = np.concatenate([np.asarray(f, dtype=np.float64).ravel(order="F") for f in est.factors])
    gl = np.ascontiguousarray(np.asarray(ground.lambda_, dtype=np.float64))
    el = np.ascontiguousarray(np.asarray(est.lambda_, dtype=np.float64))
    out = np.empty(rank)
    da, dp = _i64(dims)
    _check(lib().ref_congruence(len(dims), dp, rank, _dptr(gf), _dptr(gl), _dptr(ef), _dptr(el), _dptr(out)))
    return out


def reconstruct(m: O.KruskalModel) -> np.ndarray:
    dims = [f.shape[0] for f in m.factors]
    rank = m.factors[0].shape[1]
    f = np.concatenate([np.asarray(x, dtype=np.float64).ravel(order="F") for x in m.factors])
    lam = np.ascontiguousarray(np.asarray(m.lambda_, dtype=np.float64))
    out = np.empty(int(np.prod(dims)))
    da, dp = _i64(dims)
    _check(lib().ref_reconstruct(len(dims), dp, rank, _dptr(f), _dptr(lam), _dptr(out)))
    return out.reshape(dims, order="F")


def run_stream_synth(dims, rank, mu, sigma, synth_seed, p, q, shared, seed, enforce_bounds, als_max_iters,
                     als_rel_tol, als_restarts, batch_size, with_oracle=True):
    """-> (stream_fitness_pct, full CP-ALS fitness_pct); proj/src/commands.cpp run_stream."""
    out = np.empty(2)
    da, dp = _i64(dims)
    _check(lib().ref_run_stream_synth(len(dims), dp, rank, mu, sigma, synth_seed, p, q, shared, seed,
                                      int(enforce_bounds), als_max_iters, als_rel_tol, als_restarts, batch_size,
                                      int(with_oracle), _dptr(out)))
    return float(out[0]), float(out[1])
