"""Pipelined ingest (octen_stream_ingest_async): two batches in flight.
Batch b+1 is compressed and its CP-ALS started while batch b's sweeps (CP-ALS
worker) and batch b-1's merge (merge worker) run.  It must give the same bits
as the synchronous ingest_batch (streaming.cpp:258-346) and the reference's
error behaviour: a CP-ALS failure of batch b is reported (with the
reference's "batch N: " prefix) by the call of batch b+1, a merge failure by
the call of batch b+2 or sync(), and the later batches are rolled back, so
the state is the one the reference leaves after its failed ingest_batch."""
import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    import paper_1807_01350_b200 as m
    return m


def _data(dims, rank, seed, noise):
    x, _ = O.generate_synthetic(dims, rank, seed, 0.0, 0.0)
    if noise:
        x = x + noise * np.sqrt(np.mean(x ** 2)) * np.random.default_rng(seed).standard_normal(x.shape)
    return np.asfortranarray(x)


def _same_state(a, b):
    ma, mb = a.model, b.model
    for fa, fb in zip(ma.factors, mb.factors):
        assert np.array_equal(fa, fb)
    assert np.array_equal(ma.lambda_, mb.lambda_)
    ya, ha = a.summaries()
    yb, hb = b.summaries()
    for u, v in zip(ya, yb):
        assert np.array_equal(u, v)
    for u, v in zip(ha, hb):
        assert np.array_equal(u, v)
    la, lb = a.log, b.log
    assert len(la) == len(lb)
    for ra, rb in zip(la, lb):
        assert ra.batch_index == rb.batch_index and ra.t_new == rb.t_new
        assert ra.temporal_residual == rb.temporal_residual
        assert ra.min_match_similarity == rb.min_match_similarity


@pytest.mark.parametrize("dtype,noise", [(np.float64, 0.0), (np.float32, 0.02)])
def test_async_ingest_bit_identical(ob, dtype, noise):
    x = _data([64, 48, 90], 3, 11, noise).astype(dtype)
    cfg = ob.StreamConfig(rank=3, p=8, q=12, shared=3, seed=9, als=ob.AlsConfig(rank=3, max_iters=40, rel_tol=1e-9))
    a = ob.init_stream(np.asfortranarray(x[:, :, :30]), cfg)
    b = ob.init_stream(np.asfortranarray(x[:, :, :30]), cfg)
    b.set_publish(True)
    seen = []
    for k in range(30, 90, 10):
        ob.ingest_batch(a, np.asfortranarray(x[:, :, k:k + 10]))
        b.ingest_async(np.asfortranarray(x[:, :, k:k + 10]))
        m, nb = b.last_model()  # the model of the last batch whose merge completed (none at first)
        seen.append(nb)
    b.sync()
    _same_state(a, b)
    assert b.batches_seen == a.batches_seen == 7
    # the call of batch j returns once batch j-2's merge is done (batch j-1's
    # may be done too): batches merged so far, counting the initial block
    assert seen[0] == 0 and all(u <= v for u, v in zip(seen, seen[1:]))
    for j in range(3, 7):
        assert j - 1 <= seen[j - 1] <= j, seen
    m, nb = b.last_model()
    assert nb == 7
    ma = a.model
    for f, g in zip(m.factors, ma.factors):
        assert np.array_equal(f, g)
    assert np.array_equal(m.lambda_, ma.lambda_)


def test_async_ingest_device_batches_and_prefetch(ob):
    import torch
    x = _data([64, 64, 70], 3, 5, 0.01).astype(np.float32)
    cfg = ob.StreamConfig(rank=3, p=8, q=12, shared=3, seed=4, als=ob.AlsConfig(rank=3, max_iters=30))
    a = ob.init_stream(np.asfortranarray(x[:, :, :30]), cfg)
    b = ob.init_stream(np.asfortranarray(x[:, :, :30]), cfg)
    host = [torch.from_numpy(np.ascontiguousarray(x[:, :, k:k + 10].transpose(2, 1, 0))).pin_memory()
            .permute(2, 1, 0) for k in range(30, 70, 10)]
    for h in host:
        ob.ingest_batch(a, h)
    b.prefetch(host[0])
    for i in range(len(host)):
        if i + 1 < len(host):
            b.prefetch(host[i + 1])
        b.ingest_async(host[i])
    b.sync()
    _same_state(a, b)


def test_async_merge_error_reported_by_next_call(ob):
    # recover_temporal_append needs p*Q >= t_new + 1 (recovery.cpp:365-366):
    # a 40-slice batch at p*Q = 36 fails in the merge, after its compression
    # and CP-ALS -- exactly where the pipelined ingest defers it
    x = _data([20, 18, 90], 2, 3, 0.0)
    cfg = ob.StreamConfig(rank=2, p=6, q=6, shared=2, seed=2, als=ob.AlsConfig(rank=2, max_iters=40))
    a = ob.init_stream(np.asfortranarray(x[:, :, :10]), cfg)
    b = ob.init_stream(np.asfortranarray(x[:, :, :10]), cfg)
    ob.ingest_batch(a, np.asfortranarray(x[:, :, 10:20]))
    with pytest.raises(ob.NumericError, match=r"^batch 2: recover_temporal_append: p\*Q too small"):
        ob.ingest_batch(a, np.asfortranarray(x[:, :, 20:60]))
    ob.ingest_batch(a, np.asfortranarray(x[:, :, 60:70]))

    for via in ("sync", "next"):
        b = ob.init_stream(np.asfortranarray(x[:, :, :10]), cfg)
        b.ingest_async(np.asfortranarray(x[:, :, 10:20]))
        b.ingest_async(np.asfortranarray(x[:, :, 20:60]))  # compression + CP-ALS start succeed
        b.ingest_async(np.asfortranarray(x[:, :, 60:70]))  # batch 2's sweeps succeed, its merge is posted
        with pytest.raises(ob.NumericError, match=r"^batch 2: recover_temporal_append: p\*Q too small"):
            if via == "sync":
                b.sync()
            else:  # reports batch 2; batches 3 and this one are rolled back
                b.ingest_async(np.asfortranarray(x[:, :, 70:80]))
        assert b.batches_seen == 3
        b.ingest_async(np.asfortranarray(x[:, :, 60:70]))
        b.sync()
        _same_state(a, b)


@pytest.mark.parametrize("dtype,val,pos", [(np.float64, np.inf, (1, 2, 3)), (np.float32, np.nan, (5, 7, 9)),
                                           (np.float32, -np.inf, (19, 17, 0))])
def test_async_non_finite_batch(ob, dtype, val, pos):
    """fp64 batches take the separate non-finite scan; fp32 batches are checked
    by the tcgen05 GEMM1's conversion warps (every X element passes them)."""
    x = _data([20, 18, 40], 2, 6, 0.0).astype(dtype)
    cfg = ob.StreamConfig(rank=2, p=6, q=6, shared=2, seed=5, als=ob.AlsConfig(rank=2, max_iters=40))
    a = ob.init_stream(np.asfortranarray(x[:, :, :10]), cfg)
    b = ob.init_stream(np.asfortranarray(x[:, :, :10]), cfg)
    bad = np.array(x[:, :, 20:30], order="F")
    bad[pos] = val
    ob.ingest_batch(a, np.asfortranarray(x[:, :, 10:20]))
    with pytest.raises(ob.NumericError, match=r"^batch 2: DenseTensor: non-finite value"):
        ob.ingest_batch(a, bad)
    ob.ingest_batch(a, np.asfortranarray(x[:, :, 30:40]))
    b.ingest_async(np.asfortranarray(x[:, :, 10:20]))
    with pytest.raises(ob.NumericError, match=r"^batch 2: DenseTensor: non-finite value"):
        b.ingest_async(bad)
    b.ingest_async(np.asfortranarray(x[:, :, 30:40]))
    b.sync()
    _same_state(a, b)
