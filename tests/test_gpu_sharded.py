"""Replica-sharded streams (octen_stream_begin/merge/finish) on one GPU.

Two ranks of a 2-way sharded stream live in this process and exchange their
blocks through host-side concatenation between the phases (the phases run
one after the other; no kernel waits on another rank).  Every rank must end
with the same model as the unsharded stream on the same inputs -- the merge
is redundant and deterministic, and compression/CP-ALS are independent per
replica (streaming.cpp:45-69 is bit-deterministic for any worker count).
"""
import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import paper_1807_01350_b200 as m
    return m


def _cfg(ob, R, P, Q, sh, seed, **kw):
    return ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=seed, strict=kw.get("strict", False),
                           als=ob.AlsConfig(rank=R, max_iters=kw.get("iters", 30), rel_tol=kw.get("tol", 1e-8),
                                            n_restarts=kw.get("restarts", 3)))


def _drive(ranks, batch):
    import torch
    mo = [r.begin(batch).clone() for r in ranks]
    ma = torch.cat(mo)
    ro = [r.merge(ma).clone() for r in ranks]
    ra = torch.cat(ro)
    for r in ranks:
        r.finish(ra)


def _data():
    I, K0, t, R = 60, 40, 10, 3
    x, _ = O.generate_synthetic([I, I, K0 + 3 * t], R, 3, 0.0, 0.0)
    return x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape,
                                                                                                    order="F")


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_stream_matches_unsharded(ob, world):
    x = _data()
    cfg = _cfg(ob, 3, 8, 12, 3, 38)
    ref = ob.init_stream(O.slice_mode(x, 2, 0, 40), cfg)
    ranks = [ob.ShardedStream(cfg, g, world, None) for g in range(world)]
    assert [(r.p0, r.p_local) for r in ranks] == [ob.shard_range(8, world, g) for g in range(world)]
    _drive(ranks, O.slice_mode(x, 2, 0, 40))
    for b in range(3):
        batch = O.slice_mode(x, 2, 40 + 10 * b, 10)
        ob.ingest_batch(ref, batch)
        _drive(ranks, batch)
    want = ref.model
    for r in ranks:
        m = r.model
        for f, g in zip(m.factors, want.factors):
            assert np.allclose(f, g, rtol=0, atol=1e-12 * np.abs(g).max())
        assert np.allclose(m.lambda_, want.lambda_, rtol=1e-12)
        assert r.slices_seen == ref.slices_seen
        for a, b in zip(r.log, ref.log):
            assert a.batch_index == b.batch_index and a.t_new == b.t_new
            assert abs(a.temporal_residual - b.temporal_residual) <= 1e-12 * max(1.0, b.temporal_residual)
    # every rank holds the summaries of its own replicas only
    ys_ref, hs_ref = ref.summaries()
    for r in ranks:
        ys, hs = r.summaries()
        assert len(ys) == r.p_local
        for k, y in enumerate(ys):
            assert np.allclose(y, ys_ref[r.p0 + k], rtol=0, atol=1e-12 * np.abs(ys_ref[r.p0 + k]).max())
        for h, g in zip(hs, hs_ref):
            assert np.allclose(h, g, rtol=0, atol=1e-10 * max(1.0, np.abs(g).max()))


def test_sharded_errors_reach_every_rank(ob):
    # a zero first batch: CP-ALS fails on every replica; each rank must raise
    # the reference's NumericError from merge (after the exchange), not hang
    cfg = _cfg(ob, 2, 4, 6, 2, 3)
    ranks = [ob.ShardedStream(cfg, g, 2, None) for g in range(2)]
    z = np.zeros((12, 10, 4))
    import torch
    mo = [r.begin(z).clone() for r in ranks]
    ma = torch.cat(mo)
    for r in ranks:
        with pytest.raises(ob.NumericError, match="identically zero"):
            r.merge(ma)


def test_sharded_protocol_and_config_errors(ob):
    cfg = _cfg(ob, 2, 4, 6, 2, 3)
    with pytest.raises(ob.ConfigError):
        ob.ShardedStream(cfg, 0, 5, None)  # more shards than replicas
    r = ob.ShardedStream(cfg, 0, 2, None)
    import torch
    with pytest.raises(ob.ConfigError):
        r.merge(torch.zeros(2 * r.models_count, dtype=torch.float64, device="cuda"))  # merge before begin


def test_sharded_world1_ingest_path_matches_stream(ob):
    # ShardedStream.ingest (the bench.py N>1 path) with a trivial all-gather
    x = _data()
    cfg = _cfg(ob, 3, 8, 12, 3, 38)
    ref = ob.init_stream(O.slice_mode(x, 2, 0, 40), cfg)
    sh = ob.ShardedStream(cfg, 0, 1, lambda snd, rcv: rcv.copy_(snd))
    sh.ingest(O.slice_mode(x, 2, 0, 40))
    batch = O.slice_mode(x, 2, 40, 10)
    ob.ingest_batch(ref, batch)
    sh.ingest(batch)
    for f, g in zip(sh.model.factors, ref.model.factors):
        assert np.array_equal(f, g)
