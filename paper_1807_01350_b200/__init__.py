"""B200-native OCTen per-batch pipeline (arXiv 1807.01350) -- Python mirror of
the reference library's hot-path API (cpstream: init_stream / ingest_batch /
compress / cp_als / align_replicas / recover_*), calling the sm_100a kernels
through the C-ABI in include/octen_b200.h.

Tensors follow the reference layout (first index fastest,
proj/include/cpstream/tensor.hpp:32-34): a numpy array of shape (I, J, t) is
read in Fortran order; a torch CUDA tensor must be Fortran-contiguous
(strides (1, I, I*J)), e.g. ``torch.empty(t, J, I).permute(2, 1, 0)``.
Matrices are column-major float64.  Errors raise ConfigError / NumericError
with the reference's message text.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as C
from . import sharding as _sharding

__all__ = ["ConfigError", "NumericError", "IoError", "CudaError", "AlsConfig", "StreamConfig", "BatchRecord",
           "KruskalModel", "StreamState", "init_stream", "ingest_batch", "compress", "cp_als_batched",
           "align_replicas", "recover_nontemporal", "temporal_stack_from_summaries", "recover_temporal_append",
           "SparseTensor", "CooSummaries", "compress_coo", "congruence", "version"]


class Error(RuntimeError):
    """errors.hpp:9-12."""


class ConfigError(Error):
    """errors.hpp:14-17."""


class NumericError(Error):
    """errors.hpp:19-22."""


class IoError(Error):
    """errors.hpp:24-27."""


class CudaError(Error):
    """Device failure (no reference counterpart)."""


def _check(status: int) -> None:
    if status == C.OCTEN_OK:
        return
    msg = C.LIB.octen_last_error().decode()
    if status == C.OCTEN_ERR_CONFIG:
        raise ConfigError(msg)
    if status == C.OCTEN_ERR_NUMERIC:
        raise NumericError(msg)
    if status == C.OCTEN_ERR_IO:
        raise IoError(msg)
    if status == C.OCTEN_ERR_CUDA:
        raise CudaError(msg)
    raise Error(msg)


def version() -> str:
    return C.LIB.octen_version().decode()


def kernel_counts() -> dict:
    """Process-wide kernel path counters (octen_kernel_counts): every launch,
    tcgen05 launches of the fp32 dense compression, fp32 chunks that fell
    back to the SIMT GEMM (shape outside the tcgen05 kernels' limits), DMMA
    launches of the fp64 compression, tcgen05 (kind::i8 digit-split fp64)
    launches of the CP-ALS T-GEMM."""
    out = (C.c_i64 * 5)()
    C.LIB.octen_kernel_counts(out)
    return {"launches": out[0], "tcgen05": out[1], "simt_fallbacks": out[2], "dmma_compress": out[3],
            "tcgen05_als": out[4]}


@dataclass
class AlsConfig:
    """cp_als.hpp:25-31."""
    rank: int = 1
    max_iters: int = 100
    rel_tol: float = 1e-8
    n_restarts: int = 3
    seed: int = 0

    def _c(self) -> C.AlsConfigC:
        return C.AlsConfigC(self.rank, self.max_iters, self.rel_tol, self.n_restarts, self.seed)


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
    device: int = 0

    def _c(self) -> C.StreamConfigC:
        return C.StreamConfigC(self.rank, self.p, self.q, self.shared, self.temporal_mode, self.als._c(), self.seed,
                               int(self.enforce_bounds), self.workers, int(self.strict), self.residual_warning,
                               self.device)


@dataclass
class BatchRecord:
    """streaming.hpp:31-42."""
    batch_index: int
    t_new: int
    temporal_residual: float
    min_match_similarity: float
    max_offdiag_similarity: float
    warned: bool
    compress_seconds: float
    als_seconds: float
    recover_seconds: float
    total_seconds: float


@dataclass
class KruskalModel:
    """cp_als.hpp:12-23."""
    factors: List[np.ndarray]
    lambda_: np.ndarray


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.P_dbl)


def _f64(a) -> np.ndarray:
    """Column-major contiguous float64 copy/view."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _batch_args(batch):
    """-> (keepalive, void*, dtype, location, dims)."""
    try:
        import torch
    except Exception:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(batch, torch.Tensor):
        if batch.dim() < 1:
            raise ConfigError("octen: batch must be a tensor")
        dims = list(batch.shape)
        expect = []
        s = 1
        for d in dims:
            expect.append(s)
            s *= d
        if [st for st, d in zip(batch.stride(), dims) if d > 1] != [e for e, d in zip(expect, dims) if d > 1]:
            raise ConfigError("octen: torch batch must be first-index-fastest (Fortran-contiguous)")
        if batch.dtype == torch.float32:
            dt = C.OCTEN_F32
        elif batch.dtype == torch.float64:
            dt = C.OCTEN_F64
        else:
            raise ConfigError("octen: batch dtype must be float32 or float64")
        loc = C.OCTEN_DEVICE if batch.is_cuda else C.OCTEN_HOST
        if batch.is_cuda:
            # the library works on its own CUDA streams: work queued on
            # torch's current stream (e.g. the kernels producing this batch)
            # must be complete before the batch is read
            torch.cuda.current_stream(batch.device).synchronize()
        return batch, ctypes.c_void_p(batch.data_ptr()), dt, loc, dims
    a = np.asarray(batch)
    if a.dtype == np.float32:
        dt = C.OCTEN_F32
    else:
        a = a.astype(np.float64, copy=False)
        dt = C.OCTEN_F64
    a = np.asfortranarray(a)
    return a, ctypes.c_void_p(a.ctypes.data), dt, C.OCTEN_HOST, list(a.shape)


class StreamState:
    """streaming.hpp:48-59, device resident.  Use init_stream()."""

    def __init__(self, handle, config: StreamConfig):
        self._h = handle
        self.config = config

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(C, "LIB", None) if C is not None else None  # None at interpreter shutdown
        if h and lib is not None:
            lib.octen_stream_destroy(h)
            self._h = None

    def _info(self):
        info = (C.c_i64 * 8)()
        _check(C.LIB.octen_stream_info(self._h, info))
        return list(info)

    @property
    def slices_seen(self) -> int:
        return self._info()[3]

    @property
    def batches_seen(self) -> int:
        return self._info()[7]

    @property
    def model(self) -> KruskalModel:
        info = self._info()
        dims, rank = info[1:4], info[4]
        factors = [np.zeros((dims[m], rank), order="F") for m in range(3)]
        lam = np.zeros(rank)
        _check(C.LIB.octen_stream_get_model(self._h, _dptr(factors[0]), _dptr(factors[1]), _dptr(factors[2]),
                                            _dptr(lam)))
        return KruskalModel(factors, lam)

    @property
    def log(self) -> List[BatchRecord]:
        out = []
        nn = C.c_i64()
        _check(C.LIB.octen_stream_log_size(self._h, ctypes.byref(nn)))
        for i in range(nn.value):
            r = C.BatchRecordC()
            _check(C.LIB.octen_stream_get_record(self._h, i, ctypes.byref(r)))
            out.append(BatchRecord(r.batch_index, r.t_new, r.temporal_residual, r.min_match_similarity,
                                   r.max_offdiag_similarity, bool(r.warned), r.compress_seconds, r.als_seconds,
                                   r.recover_seconds, r.total_seconds))
        return out

    def summaries(self):
        """SummaryState.y as a list of Q^3 tensors and history (p x Q x R)."""
        info = self._info()
        rank, p, q = info[4], info[5], info[6]
        y = np.zeros(p * q * q * q)
        _check(C.LIB.octen_stream_get_summaries(self._h, _dptr(y)))
        h = np.zeros(p * q * rank)
        _check(C.LIB.octen_stream_get_history(self._h, _dptr(h)))
        ys = [y[i * q ** 3:(i + 1) * q ** 3].reshape((q, q, q), order="F") for i in range(p)]
        hs = [h[i * q * rank:(i + 1) * q * rank].reshape((q, rank), order="F") for i in range(p)]
        return ys, hs

    def prefetch(self, batch) -> None:
        """Start the host->device copy of a later batch (host array; pin it,
        e.g. a pinned torch CPU tensor, for the copy to overlap the device work
        of the batches before it).  The next ingest of the same array consumes
        the copy.  At most two may be pending; the array must not change until
        it is ingested (octen_stream_prefetch)."""
        keep, ptr, dt, loc, dims = _batch_args(batch)
        if loc != C.OCTEN_HOST:
            raise ConfigError("octen: prefetch takes a host batch")
        d = (C.c_i64 * len(dims))(*dims)
        _check(C.LIB.octen_stream_prefetch(self._h, ptr, dt, len(dims), d))
        ka = getattr(self, "_pf_keep", [])
        self._pf_keep = (ka + [keep])[-3:]  # the copies read these buffers until ingested

    def ingest_async(self, batch) -> None:
        """Pipelined ingest_batch (octen_stream_ingest_async): compression and
        CP-ALS of `batch` run now, its merge overlaps the next call's work.
        Results equal ingest_batch's bit for bit; a merge error is raised by
        the next ingest_async / sync / state read."""
        keep, ptr, dt, loc, dims = _batch_args(batch)
        d = (C.c_i64 * len(dims))(*dims)
        _check(C.LIB.octen_stream_ingest_async(self._h, ptr, dt, loc, len(dims), d))
        del keep

    def sync(self) -> None:
        """Wait for the merge of the last ingest_async (raises its error)."""
        _check(C.LIB.octen_stream_sync(self._h))

    def set_publish(self, on: bool = True) -> None:
        """Every finished batch copies its model to host memory (for
        pipelined callers: last_model() reads it without waiting)."""
        _check(C.LIB.octen_stream_set_publish(self._h, 1 if on else 0))

    def last_model(self):
        """(KruskalModel, batches finished) of the last published model, or
        (None, 0) before the first publication."""
        info = (C.c_i64 * 2)()
        tm = self.config.temporal_mode if self.config.temporal_mode >= 0 else 2
        if getattr(self, "_dims", None) is None:  # (waits for the merge in flight once)
            self._dims = tuple(d for n, d in enumerate(self._info()[1:4]) if n != tm)
        dims, rank = self._dims, self.config.rank
        cap = getattr(self, "_last_cap", 0)
        while True:
            a = np.zeros((dims[0], rank), order="F")
            b = np.zeros((dims[1], rank), order="F")
            c = np.zeros((max(cap, 1), rank), order="F")
            lam = np.zeros(rank)
            rc = C.LIB.octen_stream_last_model(self._h, info, _dptr(a), _dptr(b), _dptr(c), max(cap, 1), _dptr(lam))
            if rc == C.OCTEN_OK or info[0] <= cap:
                _check(rc)
                break
            cap = self._last_cap = int(info[0]) * 2
        if info[1] == 0:
            return None, 0
        fs = [a, b]  # the non-temporal factors in mode order, the temporal one at its mode
        fs.insert(tm, c[:info[0]].copy(order="F"))
        return KruskalModel(fs, lam), int(info[1])

    def kernel_stats(self) -> dict:
        """Live CP-ALS kernel timing (octen_stream_get_kernel_stats)."""
        out = (ctypes.c_double * 8)()
        _check(C.LIB.octen_stream_get_kernel_stats(self._h, out))
        keys = ["gemm_ms", "gemm_launches", "gemm_flops", "mttkrp_ms", "mttkrp_launches", "mttkrp_bytes", "sweeps"]
        return dict(zip(keys, list(out)[:7]))

    def checkpoint_save(self) -> bytes:
        """checkpoint_save (checkpoint.cpp:168-219): the OCTS bytes."""
        n = C.c_i64()
        _check(C.LIB.octen_stream_checkpoint_save(self._h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_uint8 * n.value)()
        _check(C.LIB.octen_stream_checkpoint_save(self._h, buf, n.value, ctypes.byref(n)))
        return bytes(buf)

    def footprint(self) -> dict:
        """measure_footprint (eval.cpp:48-60) of the device-resident state."""
        out = (C.c_i64 * 4)()
        _check(C.LIB.octen_stream_footprint(self._h, out))
        fp = {"replica_bytes": out[0], "summary_bytes": out[1], "factor_bytes": out[2],
              "accumulator_bytes": out[3]}
        fp["total"] = sum(fp.values())
        return fp

    def batch_fitness(self, batch, k0: int) -> float:
        """eval.cpp:10-20 fitness of the current model on slices [k0, k0 + t)
        of the stream, given as a batch (computed on the device)."""
        keep, ptr, dt, loc, dims = _batch_args(batch)
        d = (C.c_i64 * len(dims))(*dims)
        out = ctypes.c_double()
        _check(C.LIB.octen_stream_batch_fitness(self._h, ptr, dt, loc, len(dims), d, int(k0), ctypes.byref(out)))
        del keep
        return out.value

    def replica_models(self) -> List[KruskalModel]:
        info = self._info()
        rank, p, q = info[4], info[5], info[6]
        f = np.zeros(p * 3 * q * rank)
        lam = np.zeros(p * rank)
        _check(C.LIB.octen_stream_get_replica_models(self._h, _dptr(f), _dptr(lam)))
        out = []
        for i in range(p):
            fs = [f[(i * 3 + n) * q * rank:(i * 3 + n + 1) * q * rank].reshape((q, rank), order="F").copy()
                  for n in range(3)]
            out.append(KruskalModel(fs, lam[i * rank:(i + 1) * rank].copy()))
        return out


def init_stream(first_batch, cfg: StreamConfig) -> StreamState:
    """streaming.hpp:64 / streaming.cpp:181-256."""
    keep, ptr, dt, loc, dims = _batch_args(first_batch)
    d = (C.c_i64 * len(dims))(*dims)
    h = ctypes.c_void_p()
    c = cfg._c()
    _check(C.LIB.octen_stream_init(ctypes.byref(c), ptr, dt, loc, len(dims), d, ctypes.byref(h)))
    del keep
    st = StreamState(h, cfg)
    tm = cfg.temporal_mode if cfg.temporal_mode >= 0 else len(dims) - 1
    st._dims = tuple(d for n, d in enumerate(dims) if n != tm)  # the non-temporal extents
    return st


def checkpoint_load(data: bytes, device: int = 0) -> StreamState:
    """checkpoint_load (checkpoint.cpp:222-295): a device stream from OCTS
    bytes (the reference's, the oracle's or this library's)."""
    h = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * len(data)).from_buffer_copy(data)
    _check(C.LIB.octen_stream_checkpoint_load(buf, len(data), device, ctypes.byref(h)))
    # the StreamConfig the container holds
    import struct
    rank, p, q, shared, tmode = struct.unpack("<IIIII", data[24:44])
    seed = struct.unpack("<Q", data[44:52])[0]
    cfg = StreamConfig(rank=rank, p=p, q=q, shared=shared, seed=seed, temporal_mode=tmode, device=device)
    st = StreamState(h, cfg)
    return st


def ingest_batch(state: StreamState, batch) -> None:
    """streaming.hpp:70 / streaming.cpp:258-346."""
    keep, ptr, dt, loc, dims = _batch_args(batch)
    d = (C.c_i64 * len(dims))(*dims)
    _check(C.LIB.octen_stream_ingest(state._h, ptr, dt, loc, len(dims), d))
    del keep


def shard_range(p: int, world: int, rank: int):
    """Replicas owned by `rank` of a `world`-way sharded stream: (p0, p_local)."""
    try:
        return _sharding.shard_range(p, world, rank)
    except ValueError as e:
        raise ConfigError("octen: " + str(e)) from None


exchange_sizes = _sharding.exchange_sizes


class ShardedStream(StreamState):
    """One rank of a replica-sharded stream (include/octen_b200.h,
    octen_stream_begin/merge/finish).  `allgather(send, recv)` is the
    caller's collective on CUDA float64 tensors (recv = world x send, rank
    order), e.g. torch.distributed.all_gather_into_tensor over NCCL."""

    def __init__(self, cfg: StreamConfig, shard_rank: int, shard_world: int, allgather):
        import torch
        h = ctypes.c_void_p()
        c = cfg._c()
        _check(C.LIB.octen_stream_create(ctypes.byref(c), shard_rank, shard_world, ctypes.byref(h)))
        super().__init__(h, cfg)
        sz = (C.c_i64 * 6)()
        _check(C.LIB.octen_stream_exchange_sizes(h, sz))
        self.models_count, self.rows_count, self.p0, self.p_local = sz[0], sz[1], sz[2], sz[3]
        self.shard_rank, self.shard_world = shard_rank, shard_world
        dev = torch.device("cuda", cfg.device)
        self._mo = torch.zeros(self.models_count, dtype=torch.float64, device=dev)
        self._ma = torch.zeros(self.models_count * shard_world, dtype=torch.float64, device=dev)
        self._ro = torch.zeros(self.rows_count, dtype=torch.float64, device=dev)
        self._ra = torch.zeros(self.rows_count * shard_world, dtype=torch.float64, device=dev)
        self._allgather = allgather
        # the zero fills run on torch's stream; the library writes these
        # buffers on its own stream
        torch.cuda.current_stream(dev).synchronize()

    @staticmethod
    def _torch_ready(t) -> None:
        """A torch CUDA tensor handed to the library (e.g. a fresh NCCL
        all_gather / reduce_scatter output) was produced on torch's current
        stream: wait for it before the library's own stream reads it."""
        import torch
        if getattr(t, "is_cuda", False):
            torch.cuda.current_stream(t.device).synchronize()

    def summaries(self):
        """The owned replicas' summaries (p_local Q^3 tensors) and the full
        history (p x Q x R, kept on every rank)."""
        ys, hs = super().summaries()
        return ys[:self.p_local], hs

    # the three phases, exposed for callers that drive the exchange themselves
    def begin(self, batch):
        keep, ptr, dt, loc, dims = _batch_args(batch)
        d = (C.c_i64 * len(dims))(*dims)
        _check(C.LIB.octen_stream_begin(self._h, ptr, dt, loc, len(dims), d, ctypes.c_void_p(self._mo.data_ptr())))
        del keep
        return self._mo

    def merge(self, models_all):
        self._torch_ready(models_all)
        _check(C.LIB.octen_stream_merge(self._h, ctypes.c_void_p(models_all.data_ptr()),
                                        ctypes.c_void_p(self._ro.data_ptr())))
        return self._ro

    def finish(self, rows_all):
        self._torch_ready(rows_all)
        _check(C.LIB.octen_stream_finish(self._h, ctypes.c_void_p(rows_all.data_ptr())))

    # temporal sharding of the compression (octen_stream_begin_temporal /
    # octen_stream_begin_reduced): this rank's slices of the batch
    def begin_temporal(self, local_slices, k_off: int, t_total: int):
        """Partial summaries of every replica from this rank's slices
        [k_off, k_off + local t) of a batch of t_total slices; returns the
        world x B partial buffer for the caller's reduce-scatter (sum)."""
        import torch
        if not hasattr(self, "_pp"):
            n = C.c_i64()
            _check(C.LIB.octen_stream_partial_block_size(self._h, ctypes.byref(n)))
            dev = torch.device("cuda", self.config.device)
            self.partial_count = n.value
            self._pp = torch.zeros(n.value * self.shard_world, dtype=torch.float64, device=dev)
            self._po = torch.zeros(n.value, dtype=torch.float64, device=dev)
            torch.cuda.current_stream(dev).synchronize()
        keep, ptr, dt, loc, dims = _batch_args(local_slices)
        d = (C.c_i64 * len(dims))(*dims)
        _check(C.LIB.octen_stream_begin_temporal(self._h, ptr, dt, loc, len(dims), d, int(k_off), int(t_total),
                                                 ctypes.c_void_p(self._pp.data_ptr())))
        del keep
        return self._pp

    def begin_reduced(self, owned):
        self._torch_ready(owned)
        _check(C.LIB.octen_stream_begin_reduced(self._h, ctypes.c_void_p(owned.data_ptr()),
                                                ctypes.c_void_p(self._mo.data_ptr())))
        return self._mo

    def ingest_temporal(self, local_slices, k_off: int, t_total: int, reduce_scatter) -> None:
        """One batch with the compression sharded over the temporal mode:
        `reduce_scatter(send, recv)` sums the world x B partials into this
        rank's B (e.g. torch.distributed.reduce_scatter_tensor over NCCL)."""
        import torch
        self.begin_temporal(local_slices, k_off, t_total)
        reduce_scatter(self._pp, self._po)
        torch.cuda.synchronize()
        self.begin_reduced(self._po)
        self._exchange()

    def ingest(self, batch) -> None:
        """init_stream on the first call, ingest_batch afterwards."""
        self.begin(batch)
        self._exchange()

    def _exchange(self) -> None:
        import torch
        self._allgather(self._mo, self._ma)
        torch.cuda.synchronize()
        self.merge(self._ma)
        self._allgather(self._ro, self._ra)
        torch.cuda.synchronize()
        self.finish(self._ra)


class SynthStream:
    """On-device generate_synthetic (commands.cpp:110-134; octen_synth_*):
    U(0,1) factors from derive(seed, {9, n}), X = reconstruct + N(mu, sigma)
    noise in flat order from derive(seed, {10}).  next(t) returns the next t
    slices as a CUDA tensor viewed (I, J, t) first-index-fastest."""

    def __init__(self, dims, rank: int, seed: int, noise_mu: float = 0.0, noise_sigma: float = 0.0,
                 device: int = 0):
        self.dims = [int(d) for d in dims]
        self.rank = int(rank)
        self.device = device
        h = ctypes.c_void_p()
        d = (C.c_i64 * len(self.dims))(*self.dims)
        _check(C.LIB.octen_synth_create(len(self.dims), d, self.rank, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        float(noise_mu), float(noise_sigma), device, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(C, "LIB", None) if C is not None else None
        if h is not None and h.value and lib is not None:
            lib.octen_synth_destroy(h)
            self._h = None

    def next(self, t: int, dtype: str = "f32", out=None):
        import torch
        I, J = self.dims[0], self.dims[1]
        tdt = torch.float32 if dtype == "f32" else torch.float64
        if out is None:
            out = torch.empty((t, J, I), dtype=tdt, device=torch.device("cuda", self.device)).permute(2, 1, 0)
        _check(C.LIB.octen_synth_next(self._h, int(t), ctypes.c_void_p(out.data_ptr()),
                                      C.OCTEN_F32 if tdt == torch.float32 else C.OCTEN_F64))
        return out

    def truth(self) -> KruskalModel:
        fs = [np.zeros((d, self.rank), order="F") for d in self.dims]
        arr = (C.P_dbl * len(fs))(*[_dptr(f) for f in fs])
        lam = np.zeros(self.rank)
        _check(C.LIB.octen_synth_truth(self._h, arr, _dptr(lam)))
        return KruskalModel(fs, lam)


def nccl_unique_id() -> bytes:
    """A 128-byte ncclUniqueId for octen_stream_create_nccl (one rank draws
    it, the caller distributes it, e.g. torch.distributed.broadcast)."""
    buf = (ctypes.c_uint8 * 128)()
    _check(C.LIB.octen_nccl_get_unique_id(buf))
    return bytes(buf)


class NcclStream(StreamState):
    """One rank of a sharded stream whose collectives the library runs over
    NCCL on its own CUDA stream (octen_stream_create_nccl /
    octen_stream_ingest_sharded / octen_stream_ingest_temporal): no caller
    collectives between the phases."""

    def __init__(self, cfg: StreamConfig, shard_rank: int, shard_world: int, uid: bytes = None, comm: int = None):
        h = ctypes.c_void_p()
        c = cfg._c()
        ubuf = (ctypes.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
        _check(C.LIB.octen_stream_create_nccl(ctypes.byref(c), shard_rank, shard_world, ubuf,
                                              ctypes.c_void_p(comm) if comm else None, ctypes.byref(h)))
        super().__init__(h, cfg)
        sz = (C.c_i64 * 6)()
        _check(C.LIB.octen_stream_exchange_sizes(h, sz))
        self.p0, self.p_local = sz[2], sz[3]
        self.shard_rank, self.shard_world = shard_rank, shard_world

    def summaries(self):
        ys, hs = super().summaries()
        return ys[:self.p_local], hs

    def ingest(self, batch) -> None:
        """init_stream on the first call, ingest_batch afterwards; replicas
        sharded over the ranks, models and rows all-gathered by the library."""
        keep, ptr, dt, loc, dims = _batch_args(batch)
        d = (C.c_i64 * len(dims))(*dims)
        _check(C.LIB.octen_stream_ingest_sharded(self._h, ptr, dt, loc, len(dims), d))
        del keep

    def ingest_temporal(self, local_slices, k_off: int, t_total: int) -> None:
        """One batch whose slices [k_off, k_off + local t) of t_total are this
        rank's; partial summaries reduce-scattered by the library."""
        keep, ptr, dt, loc, dims = _batch_args(local_slices)
        d = (C.c_i64 * len(dims))(*dims)
        _check(C.LIB.octen_stream_ingest_temporal(self._h, ptr, dt, loc, len(dims), d, int(k_off), int(t_total)))
        del keep


def compress(batch, u: List[np.ndarray], v: List[np.ndarray], w: List[np.ndarray], shared: int) -> List[np.ndarray]:
    """compression.cpp:108-130 for every replica: z_r = x x1 U_r^T x2 V_r^T x3 W_r^T.
    u[r]: I x Q, v[r]: J x Q, w[r]: t x Q (temporal rows of this batch)."""
    p = len(u)
    q = u[0].shape[1]
    x = np.asarray(batch)
    I, J, t = x.shape
    if x.dtype == np.float32:
        xa, dt = np.asfortranarray(x), C.OCTEN_F32
    else:
        xa, dt = np.asfortranarray(x, dtype=np.float64), C.OCTEN_F64
    U = np.concatenate([_f64(a).ravel(order="F") for a in u])
    V = np.concatenate([_f64(a).ravel(order="F") for a in v])
    W = np.concatenate([_f64(a).ravel(order="F") for a in w])
    z = np.zeros(p * q ** 3)
    _check(C.LIB.octen_compress(p, q, shared, I, J, t, _dptr(U), _dptr(V), _dptr(W),
                                ctypes.c_void_p(xa.ctypes.data), dt, _dptr(z)))
    return [z[r * q ** 3:(r + 1) * q ** 3].reshape((q, q, q), order="F") for r in range(p)]


def cp_als_batched(tensors: List[np.ndarray], cfg: AlsConfig, seeds: List[int]):
    """cp_als (cp_als.cpp:240-359) on several Q x Q x Q tensors, seeds per
    tensor.  Returns (models, fits, iterations)."""
    p = len(tensors)
    q = tensors[0].shape[0]
    y = np.concatenate([_f64(t).ravel(order="F") for t in tensors])
    f = np.zeros(p * 3 * q * cfg.rank)
    lam = np.zeros(p * cfg.rank)
    fit = np.zeros(p)
    it = np.zeros(p, dtype=np.int32)
    sd = (C.c_u64 * p)(*seeds)
    c = cfg._c()
    _check(C.LIB.octen_cp_als_batched(p, q, _dptr(y), ctypes.byref(c), sd, _dptr(f), _dptr(lam), _dptr(fit),
                                      it.ctypes.data_as(C.P_i32)))
    r = cfg.rank
    models = []
    for i in range(p):
        fs = [f[(i * 3 + n) * q * r:(i * 3 + n + 1) * q * r].reshape((q, r), order="F").copy() for n in range(3)]
        models.append(KruskalModel(fs, lam[i * r:(i + 1) * r].copy()))
    return models, fit, it


def als_tgemm(y: np.ndarray, factors: np.ndarray, mode: int, engine: int = 1) -> np.ndarray:
    """One partial MTTKRP contraction of the device CP-ALS (octen_als_tgemm):
    T = Y x_mode F for every restart.  y: p x Q x Q x Q; factors:
    p x s x 3 x Q x R (the mode's Q x R blocks).  Returns p x Q^2 x (s R)
    with row m = the two remaining indices (first fastest).  engine 1: the
    int8 tcgen05 digit-split GEMM the sweeps use, 0: the FP64 DMMA GEMM."""
    p, q = y.shape[0], y.shape[1]
    s, r = factors.shape[1], factors.shape[4]
    yf = np.concatenate([_f64(y[i]).ravel(order="F") for i in range(p)])
    ff = np.concatenate([_f64(factors[i, j, n]).ravel(order="F") for i in range(p) for j in range(s)
                         for n in range(3)])
    t = np.zeros(p * q * q * s * r)
    _check(C.LIB.octen_als_tgemm(p, q, s, r, mode, _dptr(yf), _dptr(ff), _dptr(t), engine))
    return t.reshape((p, s * r, q * q)).transpose(0, 2, 1).copy()


def align_replicas(models: List[KruskalModel], u: List[np.ndarray], v: List[np.ndarray], tgram: np.ndarray,
                   shared: int):
    """recovery.cpp:106-291.  Returns (stacks[3] (pQ x R), perms (p x R),
    scales (p x 3 x R), min_match, max_offdiag)."""
    p = len(models)
    q, rank = models[0].factors[0].shape
    I, J = u[0].shape[0], v[0].shape[0]
    U = np.concatenate([_f64(a).ravel(order="F") for a in u])
    V = np.concatenate([_f64(a).ravel(order="F") for a in v])
    F = np.concatenate([_f64(f).ravel(order="F") for m in models for f in m.factors])
    L = np.concatenate([np.asarray(m.lambda_, dtype=np.float64) for m in models])
    tg = _f64(tgram if shared > 0 else np.zeros((0, 0))).ravel(order="F")
    if tg.size == 0:
        tg = np.zeros(1)
    stacks = np.zeros(3 * p * q * rank)
    perms = np.zeros(p * rank, dtype=np.int32)
    scales = np.zeros(p * 3 * rank)
    sims = np.zeros(2)
    _check(C.LIB.octen_align_replicas(p, q, shared, rank, I, J, _dptr(U), _dptr(V), _dptr(tg), _dptr(F), _dptr(L),
                                      _dptr(stacks), perms.ctypes.data_as(C.P_i32), _dptr(scales), _dptr(sims)))
    st = [stacks[n * p * q * rank:(n + 1) * p * q * rank].reshape((p * q, rank), order="F") for n in range(3)]
    return st, perms.reshape((p, rank)), scales.reshape((p, 3, rank)), float(sims[0]), float(sims[1])


def recover_nontemporal(stack: np.ndarray, proj_blocks: List[np.ndarray], mode: int) -> np.ndarray:
    """recovery.cpp:315-319 with P~ = [B_1^T; ...; B_p^T], B_r = proj_blocks[r] (d x Q)."""
    p = len(proj_blocks)
    d, q = proj_blocks[0].shape
    rank = stack.shape[1]
    Bk = np.concatenate([_f64(a).ravel(order="F") for a in proj_blocks])
    S = _f64(stack)
    out = np.zeros((d, rank), order="F")
    _check(C.LIB.octen_recover_nontemporal(p, q, d, rank, mode, _dptr(Bk), _dptr(S), _dptr(out)))
    return out


def temporal_stack_from_summaries(ys: List[np.ndarray], u, v, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """recovery.cpp:429-462."""
    p = len(ys)
    q = ys[0].shape[0]
    rank = a.shape[1]
    Y = np.concatenate([_f64(y).ravel(order="F") for y in ys])
    U = np.concatenate([_f64(x).ravel(order="F") for x in u])
    V = np.concatenate([_f64(x).ravel(order="F") for x in v])
    A, B = _f64(a), _f64(b)
    out = np.zeros((p * q, rank), order="F")
    _check(C.LIB.octen_temporal_stack_from_summaries(p, q, rank, A.shape[0], B.shape[0], _dptr(Y), _dptr(U), _dptr(V),
                                                     _dptr(A), _dptr(B), _dptr(out)))
    return out


def recover_temporal_append(temporal_stack: np.ndarray, w: List[np.ndarray], history: List[np.ndarray]):
    """recovery.cpp:341-427 (no column weights).  history is updated in place
    (list of Q x R).  Returns (new_rows, residual)."""
    p = len(w)
    t, q = w[0].shape
    rank = temporal_stack.shape[1]
    W = np.concatenate([_f64(x).ravel(order="F") for x in w])
    H = np.concatenate([_f64(h if h.size else np.zeros((q, rank))).ravel(order="F") for h in history])
    S = _f64(temporal_stack)
    rows = np.zeros((t, rank), order="F")
    res = ctypes.c_double(0.0)
    _check(C.LIB.octen_recover_temporal_append(p, q, rank, t, _dptr(S), _dptr(W), _dptr(H), _dptr(rows),
                                               ctypes.byref(res)))
    for i in range(p):
        history[i] = H[i * q * rank:(i + 1) * q * rank].reshape((q, rank), order="F").copy()
    return rows, res.value


# ---------------------------------------------------------------------------
# Sparse (COO) temporal batches
# ---------------------------------------------------------------------------

class SparseTensor:
    """tensor.hpp:66-90 -- a COO temporal batch of shape (I, J, t): indices
    (nnz x 3, 0-based; the third is the slice within the batch) and values.
    Stored SoA (int32 i, j, k; float32 values) for the device.  Validation
    (tensor.cpp:87-102) happens on the device when the batch is compressed,
    with the reference's exceptions and messages."""

    def __init__(self, shape, indices, values):
        if len(shape) != 3:
            raise ConfigError("octen: sparse batches are order-3 (I, J, t)")
        self.shape = tuple(int(d) for d in shape)
        idx = np.asarray(indices)
        if idx.size == 0:
            idx = np.zeros((0, 3), dtype=np.int64)
        if idx.ndim != 2 or idx.shape[1] != 3:
            raise ConfigError("SparseTensor: index arity mismatch")
        if np.any(idx > np.iinfo(np.int32).max) or np.any(idx < np.iinfo(np.int32).min):
            raise ConfigError("SparseTensor: index out of bounds")
        self.i = np.ascontiguousarray(idx[:, 0], dtype=np.int32)
        self.j = np.ascontiguousarray(idx[:, 1], dtype=np.int32)
        self.k = np.ascontiguousarray(idx[:, 2], dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float32)
        if self.values.shape != (idx.shape[0],):
            raise ConfigError("SparseTensor: values do not match indices")

    @staticmethod
    def from_arrays(shape, i: np.ndarray, j: np.ndarray, k: np.ndarray, values: np.ndarray) -> "SparseTensor":
        """Wrap existing SoA arrays without copying (contiguous int32 i, j, k
        and float32 values; e.g. numpy views of pinned torch CPU tensors, so
        the device copy runs at full PCIe speed)."""
        sp = SparseTensor.__new__(SparseTensor)
        sp.shape = tuple(int(d) for d in shape)
        for a, dt in ((i, np.int32), (j, np.int32), (k, np.int32), (values, np.float32)):
            if a.dtype != dt or a.ndim != 1 or not a.flags.c_contiguous or a.shape[0] != values.shape[0]:
                raise ConfigError("SparseTensor.from_arrays: contiguous int32 i, j, k and float32 values of one length")
        sp.i, sp.j, sp.k, sp.values = i, j, k, values
        return sp

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @staticmethod
    def read(path: str) -> "SparseTensor":
        """read_tensor_coo (io.cpp:49-84) of an order-3 file (octen_read_coo):
        1-based text entries, the reference's IoError messages; duplicates
        are reported when the batch is compressed."""
        h = ctypes.c_void_p()
        _check(C.LIB.octen_read_coo(str(path).encode(), ctypes.byref(h)))
        try:
            order, nnz = C.c_i64(), C.c_i64()
            dims = (C.c_i64 * 16)()
            _check(C.LIB.octen_coo_file_info(h, ctypes.byref(order), dims, ctypes.byref(nnz)))
            if order.value != 3:
                raise ConfigError("octen: sparse batches are order-3 (I, J, t)")
            idx = np.zeros((nnz.value, 3), dtype=np.int64)
            val = np.zeros(nnz.value)
            if nnz.value:
                _check(C.LIB.octen_coo_file_entries(h, idx.ctypes.data_as(C.P_i64), _dptr(val)))
            return SparseTensor(tuple(dims[:3]), idx, val)
        finally:
            C.LIB.octen_coo_file_destroy(h)

    @staticmethod
    def from_dense(t) -> "SparseTensor":
        """tensor.cpp:104-116 (nonzeros in first-index-fastest order)."""
        a = np.asarray(t)
        flat = a.ravel(order="F")
        nz = np.nonzero(flat)[0]
        idx = np.stack(np.unravel_index(nz, a.shape, order="F"), axis=1)
        return SparseTensor(a.shape, idx, flat[nz])


def _stack_cols(mats, rows, q):
    return np.concatenate([_f64(m).reshape(rows, q, order="F").ravel(order="F") for m in mats])


class CooSummaries:
    """Device-resident SummaryState (compression.hpp:56-60) fed by COO
    batches: compress() is update_summaries(compress(to_dense(batch)))
    (compression.cpp:108-153, io.cpp:124-132) without densifying."""

    def __init__(self, u: List[np.ndarray], v: List[np.ndarray], device: int = 0):
        self.p = len(u)
        self.I, self.q = np.asarray(u[0]).shape
        self.J = np.asarray(v[0]).shape[0]
        U = _stack_cols(u, self.I, self.q)
        V = _stack_cols(v, self.J, self.q)
        h = ctypes.c_void_p()
        _check(C.LIB.octen_coo_create(self.p, self.q, self.I, self.J, _dptr(U), _dptr(V), device, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(C, "LIB", None) if C is not None else None
        if h is not None and h.value and lib is not None:
            lib.octen_coo_destroy(h)
            self._h = None

    def compress(self, batch: SparseTensor, w) -> None:
        """w: per-replica temporal rows of this batch (t x Q each) or a
        stacked (p, t, Q) array."""
        t = batch.shape[2]
        if (batch.shape[0], batch.shape[1]) != (self.I, self.J):
            raise ConfigError("compress: extent mismatch on mode 1")
        W = _stack_cols(list(w), t, self.q)
        _check(C.LIB.octen_coo_compress(self._h, t, W.ctypes.data, batch.nnz, batch.i.ctypes.data,
                                        batch.j.ctypes.data, batch.k.ctypes.data, batch.values.ctypes.data,
                                        C.OCTEN_HOST))

    def compress_device(self, t: int, w, i, j, k, values) -> None:
        """Device-resident inputs (torch CUDA tensors): w float64 (p, Q, t)
        contiguous = per replica t x Q column-major; i, j, k int32; values
        float32."""
        import torch
        torch.cuda.current_stream(values.device).synchronize()  # producers on torch's stream
        _check(C.LIB.octen_coo_compress(self._h, int(t), w.data_ptr(), int(values.numel()), i.data_ptr(),
                                        j.data_ptr(), k.data_ptr(), values.data_ptr(), C.OCTEN_DEVICE))

    def summaries(self) -> List[np.ndarray]:
        q3 = self.q ** 3
        y = np.zeros(self.p * q3)
        _check(C.LIB.octen_coo_get_summaries(self._h, _dptr(y)))
        return [y[r * q3:(r + 1) * q3].reshape((self.q,) * 3, order="F") for r in range(self.p)]

    def reset(self) -> None:
        _check(C.LIB.octen_coo_reset(self._h))

    def cp_als(self, cfg: AlsConfig, seeds: List[int], fetch: bool = True):
        """cp_als (cp_als.cpp:240-359) on every resident summary."""
        p, q, r = self.p, self.q, cfg.rank
        f = np.zeros(p * 3 * q * r)
        lam = np.zeros(p * r)
        fit = np.zeros(p)
        it = np.zeros(p, dtype=np.int32)
        sd = (C.c_u64 * p)(*seeds)
        c = cfg._c()
        _check(C.LIB.octen_coo_cp_als(self._h, ctypes.byref(c), sd, _dptr(f) if fetch else None,
                                      _dptr(lam) if fetch else None, _dptr(fit), it.ctypes.data_as(C.P_i32)))
        models = []
        for i in range(p):
            fs = [f[(i * 3 + n) * q * r:(i * 3 + n + 1) * q * r].reshape((q, r), order="F").copy() for n in range(3)]
            models.append(KruskalModel(fs, lam[i * r:(i + 1) * r].copy()))
        return models, fit, it

    def stage_times(self) -> dict:
        out = np.zeros(8)
        _check(C.LIB.octen_coo_stage_times(self._h, _dptr(out)))
        keys = ["prep_ms", "slice_ms", "accum_ms", "groups", "nnz", "batches", "als_ms", "als_runs"]
        return dict(zip(keys, out.tolist()))

    def cuda_stream(self) -> int:
        return int(C.LIB.octen_coo_cuda_stream(self._h) or 0)


def compress_coo(batch: SparseTensor, u: List[np.ndarray], v: List[np.ndarray], w: List[np.ndarray]) -> List[np.ndarray]:
    """compress (compression.cpp:108-130) of to_dense(batch) for every
    replica, computed from the COO entries on the device."""
    p = len(u)
    I, q = np.asarray(u[0]).shape
    J = np.asarray(v[0]).shape[0]
    t = batch.shape[2]
    if (batch.shape[0], batch.shape[1]) != (I, J):
        raise ConfigError("compress: extent mismatch on mode 1")
    U = _stack_cols(u, I, q)
    V = _stack_cols(v, J, q)
    W = _stack_cols(w, t, q)
    z = np.zeros(p * q ** 3)
    _check(C.LIB.octen_compress_coo(p, q, I, J, t, _dptr(U), _dptr(V), _dptr(W), batch.nnz, batch.i.ctypes.data,
                                    batch.j.ctypes.data, batch.k.ctypes.data, batch.values.ctypes.data, _dptr(z)))
    return [z[r * q ** 3:(r + 1) * q ** 3].reshape((q, q, q), order="F") for r in range(p)]


def congruence(ground: KruskalModel, est: KruskalModel) -> List[float]:
    """eval.cpp:22-46 per-component congruence (factor match score) after
    exhaustive (rank <= 6) or greedy matching (octen_congruence).  Checks
    and messages in the reference's order: rank, order, per-mode rows."""
    gf = [_f64(f) for f in ground.factors]
    ef = [_f64(f) for f in est.factors]
    r = len(np.asarray(ground.lambda_))  # KruskalModel::rank() (cp_als.hpp:17)
    if len(np.asarray(est.lambda_)) != r:
        raise ConfigError("congruence: rank mismatch")
    if len(gf) != len(ef):
        raise ConfigError("congruence: order mismatch")
    for n, (g, e) in enumerate(zip(gf, ef)):
        if g.shape[0] != e.shape[0]:
            raise ConfigError("congruence: factor shape mismatch on mode %d" % (n + 1))
    for n, f in enumerate(gf + ef):  # the C call reads d_n * r values per factor
        if f.ndim != 2 or f.shape[1] != r:
            raise ConfigError("congruence: factor shape mismatch on mode %d" % (n % max(len(gf), 1) + 1))
    dims = [g.shape[0] for g in gf]
    g = np.concatenate([f.ravel(order="F") for f in gf])
    e = np.concatenate([f.ravel(order="F") for f in ef])
    out = np.zeros(r)
    d = (C.c_i64 * len(dims))(*dims)
    _check(C.LIB.octen_congruence(len(dims), r, d, _dptr(g), _dptr(e), _dptr(out)))
    return out.tolist()
