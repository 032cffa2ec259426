"""Streams whose temporal mode is not the last one (StreamConfig.temporal_mode,
streaming.hpp:20; the reference keeps the summaries and the model in the
tensor's own mode order, compression.cpp:117-127): the device reorders each
batch to temporal-last for its contractions and writes the summaries, the
model and the checkpoints in the stream's order.  Against the oracle."""
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


def _truth(dims, rank, seed):
    s = rng.Substream(seed)
    return O.KruskalModel([s.fill_uniform(d, rank) for d in dims], np.ones(rank))


@pytest.mark.parametrize("tm", [0, 1])
def test_temporal_mode_matches_oracle(ob, tm):
    dims = [20, 18, 16]
    dims[tm] = 24  # the temporal extent
    full = O.reconstruct_fast(_truth(dims, 3, 40 + tm))
    kw = dict(rank=3, p=6, q=8, shared=3, seed=77 + tm, temporal_mode=tm)
    st = ob.init_stream(O.slice_mode(full, tm, 0, 8), ob.StreamConfig(**kw, als=ob.AlsConfig(rank=3, max_iters=200,
                                                                                              rel_tol=1e-12)))
    ref = O.init_stream(O.slice_mode(full, tm, 0, 8), O.StreamConfig(**kw, als=O.AlsConfig(3, 200, 1e-12, 3, 0)))
    for k0 in (8, 16):
        ob.ingest_batch(st, O.slice_mode(full, tm, k0, 8))
        O.ingest_batch(ref, O.slice_mode(full, tm, k0, 8))
    ys, hs = st.summaries()
    for a, b in zip(ys, ref.summaries.y):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)  # the summaries keep the stream's mode order
    m = st.model
    assert [f.shape[0] for f in m.factors] == dims
    md = O.KruskalModel(m.factors, m.lambda_)
    assert O.fitness(full, O.reconstruct_fast(md)) >= 95.0
    assert min(O.congruence(md, ref.model)) > 1 - 1e-8
    # evaluation, checkpoint and replica models in the same order
    sl = O.slice_mode(full, tm, 16, 8)
    # |X - Xhat|^2 = |X|^2 - 2<X, Xhat> + |Xhat|^2 cancels near a perfect fit:
    # ~sqrt(eps) relative in the residual, ~1e-6 in the percentage
    assert abs(st.batch_fitness(sl, 16) - O.fitness(sl, O.slice_mode(O.reconstruct_fast(md), tm, 16, 8))) < 1e-5
    b = st.checkpoint_save()
    assert O.checkpoint_save(O.checkpoint_load(b)) == b
    back = ob.checkpoint_load(b)
    assert back.checkpoint_save() == b
    assert [f.shape[0] for f in back.model.factors] == dims
    for r, w in zip(st.replica_models(), ref.replica_models):
        assert [f.shape[0] for f in r.factors] == [8, 8, 8]
    with pytest.raises(ob.ConfigError, match="temporal mode last"):
        st.prefetch(np.asfortranarray(sl))


def test_temporal_mode_errors(ob):
    full = O.reconstruct_fast(_truth([12, 10, 9], 2, 5))
    with pytest.raises(ob.ConfigError, match="stream: temporal mode out of range"):
        ob.init_stream(full, ob.StreamConfig(rank=2, p=4, q=6, shared=2, temporal_mode=3))
    st = ob.init_stream(O.slice_mode(full, 0, 0, 6),
                        ob.StreamConfig(rank=2, p=4, q=6, shared=2, seed=3, temporal_mode=0))
    with pytest.raises(ob.ConfigError, match="ingest_batch: extent mismatch on mode 2"):
        ob.ingest_batch(st, np.zeros((3, 11, 9), order="F"))
