"""Library-owned NCCL collectives of a sharded stream (octen_stream_create_nccl,
octen_stream_ingest_sharded / _temporal) on one GPU: a world-1 communicator
runs the same phases and collectives (the all-gathers and the reduce-scatter
degenerate to copies) and must give the unsharded stream's bits.  The
multi-rank protocol is covered by the gloo tests (test_multigpu_cpu.py) and
the one-GPU emulation (test_gpu_sharded.py)."""
import numpy as np
import pytest

from oracle import octen_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    import paper_1807_01350_b200 as m
    return m


def _data():
    x, _ = O.generate_synthetic([40, 36, 50], 3, 13, 0.0, 0.0)
    x = x + 0.01 * np.sqrt(np.mean(x ** 2)) * np.random.default_rng(2).standard_normal(x.shape)
    return np.asfortranarray(x.astype(np.float32))


def _cfg(ob):
    return ob.StreamConfig(rank=3, p=8, q=10, shared=3, seed=21, als=ob.AlsConfig(rank=3, max_iters=40))


@pytest.mark.parametrize("mode", ["sharded", "temporal"])
def test_nccl_world1_equals_unsharded(ob, mode):
    x = _data()
    ref = ob.init_stream(np.asfortranarray(x[:, :, :20]), _cfg(ob))
    for k in (20, 35):
        ob.ingest_batch(ref, np.asfortranarray(x[:, :, k:k + 15]))
    st = ob.NcclStream(_cfg(ob), 0, 1, uid=ob.nccl_unique_id())
    for k0, t in ((0, 20), (20, 15), (35, 15)):
        b = np.asfortranarray(x[:, :, k0:k0 + t])
        if mode == "sharded":
            st.ingest(b)
        else:
            st.ingest_temporal(b, 0, t)
    a, b = ref.model, st.model
    same = np.array_equal if mode == "sharded" else (lambda u, v: np.allclose(u, v, rtol=1e-9, atol=1e-12))
    for f, g in zip(a.factors, b.factors):
        assert same(f, g)
    assert same(a.lambda_, b.lambda_)
    ya, _ = ref.summaries()
    yb, _ = st.summaries()
    for u, v in zip(ya, yb):
        assert np.array_equal(u, v) if mode == "sharded" else np.allclose(u, v, rtol=1e-12, atol=0)


def test_nccl_requires_communicator(ob):
    st = ob.ShardedStream(_cfg(ob), 0, 1, lambda s, r: r.copy_(s))
    with pytest.raises(ob.ConfigError, match="no NCCL communicator"):
        ob.NcclStream.ingest(st, _data()[:, :, :20])
