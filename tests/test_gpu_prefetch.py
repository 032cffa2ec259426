"""GPU: host-batch prefetch (octen_stream_prefetch) is an overlap mechanism
only -- a stream fed through prefetch + ingest is bit-identical to one fed by
plain ingest of the same host batches (and both to the device-batch stream's
summaries); stale prefetches are dropped; at most two may be pending."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    import paper_1807_01350_b200 as m
    return m


def _batches(seed, I=60, J=50, R=4, K0=40, t=10, nb=4):
    r = np.random.default_rng(seed)
    A, B, C = r.random((I, R)), r.random((J, R)), r.random((K0 + nb * t, R))
    x = np.einsum("ir,jr,kr->ijk", A, B, C)
    x = np.asfortranarray((x + 0.01 * r.standard_normal(x.shape)).astype(np.float32))
    first = np.asfortranarray(x[:, :, :K0])
    return first, [np.asfortranarray(x[:, :, K0 + b * t:K0 + (b + 1) * t]) for b in range(nb)]


def _cfg(ob):
    return ob.StreamConfig(rank=4, p=6, q=15, shared=3, seed=5,
                           als=ob.AlsConfig(rank=4, max_iters=40, rel_tol=1e-10, n_restarts=2))


def _state(st):
    m = st.model
    ys, hs = st.summaries()
    return [f.copy() for f in m.factors] + [m.lambda_.copy()] + ys + hs


def test_prefetch_is_bit_identical_to_plain_ingest(ob):
    first, bs = _batches(1)
    a = ob.init_stream(first, _cfg(ob))
    for b in bs:
        ob.ingest_batch(a, b)
    c = ob.init_stream(first, _cfg(ob))
    c.prefetch(bs[0])
    for i, b in enumerate(bs):
        if i + 1 < len(bs):
            c.prefetch(bs[i + 1])
        ob.ingest_batch(c, b)
    for u, v in zip(_state(a), _state(c)):
        assert np.array_equal(u, v)


def test_stale_prefetch_is_dropped_and_pending_limit(ob):
    first, bs = _batches(2)
    a = ob.init_stream(first, _cfg(ob))
    for b in bs[:2]:
        ob.ingest_batch(a, b)
    c = ob.init_stream(first, _cfg(ob))
    c.prefetch(bs[1])              # not the next batch: must not be used for bs[0]
    ob.ingest_batch(c, bs[0])      # plain path, drops the stale prefetch
    c.prefetch(bs[1])
    c.prefetch(bs[2])
    with pytest.raises(ob.ConfigError, match="already pending"):
        c.prefetch(bs[3])
    ob.ingest_batch(c, bs[1])      # consumes the first pending copy
    for u, v in zip(_state(a), _state(c)):
        assert np.array_equal(u, v)
