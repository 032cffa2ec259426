"""Host-side layout of the replica-sharded exchange (include/octen_b200.h,
octen_stream_begin/merge/finish), in numpy.

Rank g of `world` owns replicas [p0, p0 + p_local) with chunk = ceil(P / world)
(octen::Stream).  Its blocks in the two all-gathers are
  models: [status kind, a, b, 0] + chunk x (3 x Q x R) factors + chunk x R lambdas
  rows:   chunk x (Q x R) temporal-stack rows (replica-major, column-major Q x R)
and the gathered buffers are the world blocks in rank order.  The device
packs/unpacks these itself (stream.cu); these helpers are the same layout for
callers that carry the blocks over their own transport and for the CPU tests.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def shard_range(p: int, world: int, rank: int) -> Tuple[int, int]:
    """(p0, p_local) of `rank`; same rule as octen::Stream."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard rank/world out of range")
    if world > p:
        raise ValueError("more shards than replicas")
    chunk = -(-p // world)
    p0 = min(p, rank * chunk)
    return p0, max(0, min(p, p0 + chunk) - p0)


def exchange_sizes(p: int, q: int, rank: int, world: int) -> Tuple[int, int]:
    """Doubles per rank: (models block, rows block)."""
    chunk = -(-p // world)
    return 4 + chunk * (3 * q * rank + rank), chunk * q * rank


def pack_models(factors: Sequence[Sequence[np.ndarray]], lambdas: Sequence[np.ndarray], p: int, q: int, rank: int,
                world: int, status=(0, 0, 0)) -> np.ndarray:
    """One rank's models block from its p_local replica models (factors[r] =
    [A, B, C], each Q x R)."""
    chunk = -(-p // world)
    mc, _ = exchange_sizes(p, q, rank, world)
    out = np.zeros(mc)
    out[:3] = status
    qr = q * rank
    for r, (fs, lam) in enumerate(zip(factors, lambdas)):
        for n in range(3):
            out[4 + (r * 3 + n) * qr:4 + (r * 3 + n + 1) * qr] = np.asarray(fs[n]).ravel(order="F")
        out[4 + chunk * 3 * qr + r * rank:4 + chunk * 3 * qr + (r + 1) * rank] = lam
    return out


def unpack_models(gathered: np.ndarray, p: int, q: int, rank: int, world: int):
    """-> (status per rank, [factors per replica], [lambda per replica])."""
    chunk = -(-p // world)
    mc, _ = exchange_sizes(p, q, rank, world)
    qr = q * rank
    status, facs, lams = [], [], []
    for g in range(world):
        blk = gathered[g * mc:(g + 1) * mc]
        status.append(tuple(int(v) for v in blk[:3]))
        g0, gl = shard_range(p, world, g)
        for r in range(gl):
            facs.append([blk[4 + (r * 3 + n) * qr:4 + (r * 3 + n + 1) * qr].reshape((q, rank), order="F")
                         for n in range(3)])
            lams.append(blk[4 + chunk * 3 * qr + r * rank:4 + chunk * 3 * qr + (r + 1) * rank].copy())
    return status, facs, lams


def pack_rows(stack_rows: Sequence[np.ndarray], p: int, q: int, rank: int, world: int) -> np.ndarray:
    """One rank's rows block from its replicas' Q x R temporal-stack rows."""
    _, rc = exchange_sizes(p, q, rank, world)
    out = np.zeros(rc)
    for r, m in enumerate(stack_rows):
        out[r * q * rank:(r + 1) * q * rank] = np.asarray(m).ravel(order="F")
    return out


def unpack_rows(gathered: np.ndarray, p: int, q: int, rank: int, world: int) -> np.ndarray:
    """-> the P*Q x R stacked temporal system (recovery.cpp:429-462 layout)."""
    _, rc = exchange_sizes(p, q, rank, world)
    out = np.zeros((p * q, rank))
    for rep in range(p):
        g = rep // (-(-p // world))
        pi = rep - g * (-(-p // world))
        out[rep * q:(rep + 1) * q] = gathered[g * rc + pi * q * rank:g * rc + (pi + 1) * q * rank].reshape(
            (q, rank), order="F")
    return out
