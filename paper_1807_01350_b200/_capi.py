"""ctypes binding of include/octen_b200.h (the drop-in C-ABI).

The native library is mandatory: there is no CPU fallback.  Importing this
module when lib/libocten_b200.so is missing raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libocten_b200.so")

OCTEN_OK = 0
OCTEN_ERR_CONFIG = 2
OCTEN_ERR_NUMERIC = 3
OCTEN_ERR_IO = 4
OCTEN_ERR_CUDA = 5
OCTEN_ERR_INTERNAL = 6
OCTEN_F64 = 0
OCTEN_F32 = 1
OCTEN_HOST = 0
OCTEN_DEVICE = 1

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
P_dbl = ctypes.POINTER(ctypes.c_double)
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_u64 = ctypes.POINTER(ctypes.c_uint64)


class AlsConfigC(ctypes.Structure):
    _fields_ = [("rank", c_i32), ("max_iters", c_i32), ("rel_tol", c_dbl), ("n_restarts", c_i32), ("seed", c_u64)]


class StreamConfigC(ctypes.Structure):
    _fields_ = [("rank", c_i32), ("p", c_i32), ("q", c_i32), ("shared", c_i32), ("temporal_mode", c_i32),
                ("als", AlsConfigC), ("seed", c_u64), ("enforce_bounds", c_i32), ("workers", c_i32),
                ("strict", c_i32), ("residual_warning", c_dbl), ("device", c_i32)]


class BatchRecordC(ctypes.Structure):
    _fields_ = [("batch_index", c_i64), ("t_new", c_i64), ("temporal_residual", c_dbl),
                ("min_match_similarity", c_dbl), ("max_offdiag_similarity", c_dbl), ("warned", c_i32),
                ("compress_seconds", c_dbl), ("als_seconds", c_dbl), ("recover_seconds", c_dbl),
                ("total_seconds", c_dbl)]


# every symbol include/octen_b200.h declares, with its ctypes signature
SIGNATURES = {
    "octen_last_error": (ctypes.c_char_p, []),
    "octen_version": (ctypes.c_char_p, []),
    "octen_launch_count": (ctypes.c_int64, []),
    "octen_kernel_counts": (None, [P_i64]),
    "octen_stream_footprint": (ctypes.c_int, [ctypes.c_void_p, P_i64]),
    "octen_stream_get_stage_times": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_stream_init": (ctypes.c_int, [ctypes.POINTER(StreamConfigC), ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, P_i64, ctypes.POINTER(ctypes.c_void_p)]),
    "octen_stream_ingest": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, P_i64]),
    "octen_stream_destroy": (None, [ctypes.c_void_p]),
    "octen_synth_create": (ctypes.c_int, [ctypes.c_int, P_i64, ctypes.c_int, c_u64, c_dbl, c_dbl, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "octen_synth_next": (ctypes.c_int, [ctypes.c_void_p, c_i64, ctypes.c_void_p, ctypes.c_int]),
    "octen_synth_truth": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(P_dbl), P_dbl]),
    "octen_synth_destroy": (None, [ctypes.c_void_p]),
    "octen_stream_ingest_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, P_i64]),
    "octen_stream_sync": (ctypes.c_int, [ctypes.c_void_p]),
    "octen_read_coo": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "octen_coo_file_info": (ctypes.c_int, [ctypes.c_void_p, P_i64, P_i64, P_i64]),
    "octen_coo_file_entries": (ctypes.c_int, [ctypes.c_void_p, P_i64, P_dbl]),
    "octen_coo_file_destroy": (None, [ctypes.c_void_p]),
    "octen_nccl_get_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "octen_stream_create_nccl": (ctypes.c_int, [ctypes.POINTER(StreamConfigC), ctypes.c_int, ctypes.c_int,
                                                ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "octen_stream_ingest_sharded": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, P_i64]),
    "octen_stream_ingest_temporal": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                    ctypes.c_int, P_i64, c_i64, c_i64]),
    "octen_stream_checkpoint_save": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, c_i64, P_i64]),
    "octen_stream_checkpoint_load": (ctypes.c_int, [ctypes.c_void_p, c_i64, ctypes.c_int,
                                                    ctypes.POINTER(ctypes.c_void_p)]),
    "octen_stream_log_size": (ctypes.c_int, [ctypes.c_void_p, P_i64]),
    "octen_stream_get_kernel_stats": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_stream_set_publish": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "octen_stream_last_model": (ctypes.c_int, [ctypes.c_void_p, P_i64, P_dbl, P_dbl, P_dbl, c_i64, P_dbl]),
    "octen_congruence": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, P_i64, P_dbl, P_dbl, P_dbl]),
    "octen_stream_batch_fitness": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int, P_i64, c_i64, P_dbl]),
    "octen_stream_partial_block_size": (ctypes.c_int, [ctypes.c_void_p, P_i64]),
    "octen_stream_begin_temporal": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, P_i64, c_i64, c_i64, ctypes.c_void_p]),
    "octen_stream_begin_reduced": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "octen_stream_prefetch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, P_i64]),
    "octen_stream_create": (ctypes.c_int, [ctypes.POINTER(StreamConfigC), ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_void_p)]),
    "octen_stream_exchange_sizes": (ctypes.c_int, [ctypes.c_void_p, P_i64]),
    "octen_stream_begin": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          P_i64, ctypes.c_void_p]),
    "octen_stream_merge": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "octen_stream_finish": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "octen_stream_info": (ctypes.c_int, [ctypes.c_void_p, P_i64]),
    "octen_stream_get_factor": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, P_dbl]),
    "octen_stream_get_lambda": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_stream_get_model": (ctypes.c_int, [ctypes.c_void_p, P_dbl, P_dbl, P_dbl, P_dbl]),
    "octen_stream_get_record": (ctypes.c_int, [ctypes.c_void_p, c_i64, ctypes.POINTER(BatchRecordC)]),
    "octen_stream_get_summaries": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_stream_get_history": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_stream_get_replica_models": (ctypes.c_int, [ctypes.c_void_p, P_dbl, P_dbl]),
    "octen_compress": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64, c_i64, c_i64, P_dbl, P_dbl,
                                      P_dbl, ctypes.c_void_p, ctypes.c_int, P_dbl]),
    "octen_cp_als_batched": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, P_dbl, ctypes.POINTER(AlsConfigC), P_u64,
                                            P_dbl, P_dbl, P_dbl, P_i32]),
    "octen_als_tgemm": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P_dbl,
                                       P_dbl, P_dbl, ctypes.c_int]),
    "octen_align_replicas": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64, c_i64,
                                            P_dbl, P_dbl, P_dbl, P_dbl, P_dbl, P_dbl, P_i32, P_dbl, P_dbl]),
    "octen_recover_nontemporal": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int, ctypes.c_int,
                                                 P_dbl, P_dbl, P_dbl]),
    "octen_temporal_stack_from_summaries": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64, c_i64,
                                                           P_dbl, P_dbl, P_dbl, P_dbl, P_dbl, P_dbl]),
    "octen_recover_temporal_append": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, c_i64, P_dbl, P_dbl,
                                                     P_dbl, P_dbl, P_dbl]),
    "octen_coo_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_i64, c_i64, P_dbl, P_dbl, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "octen_coo_compress": (ctypes.c_int, [ctypes.c_void_p, c_i64, ctypes.c_void_p, c_i64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "octen_coo_get_summaries": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_coo_reset": (ctypes.c_int, [ctypes.c_void_p]),
    "octen_coo_cp_als": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(AlsConfigC), P_u64, P_dbl, P_dbl, P_dbl,
                                        P_i32]),
    "octen_coo_stage_times": (ctypes.c_int, [ctypes.c_void_p, P_dbl]),
    "octen_coo_cuda_stream": (ctypes.c_void_p, [ctypes.c_void_p]),
    "octen_coo_destroy": (None, [ctypes.c_void_p]),
    "octen_compress_coo": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_i64, c_i64, c_i64, P_dbl, P_dbl, P_dbl, c_i64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, P_dbl]),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError("octen_b200: native library %s not built; run `python -m paper_1807_01350_b200.build`"
                          % path)
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """Loads the native library on first use (so `python -m
    paper_1807_01350_b200.build` can run before it exists); any call without
    the library raises ImportError -- there is no fallback."""

    _lib = None

    def __getattr__(self, name):
        if _LazyLib._lib is None:
            _LazyLib._lib = load()
        return getattr(_LazyLib._lib, name)


LIB = _LazyLib()
