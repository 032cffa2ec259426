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


def _drive_temporal(ranks, batch, world):
    """Temporal sharding: rank g compresses its contiguous slice range of the
    batch into partials of every replica; the reduce-scatter is a host-side
    sum over ranks of each owner's block."""
    import torch
    t = batch.shape[2]
    bounds = [t * g // world for g in range(world + 1)]
    parts = []
    for g, r in enumerate(ranks):
        loc = np.asfortranarray(batch[:, :, bounds[g]:bounds[g + 1]])
        parts.append(r.begin_temporal(loc, bounds[g], t).clone())
    blk = ranks[0].partial_count
    owned = [sum(p[g * blk:(g + 1) * blk] for p in parts) for g in range(world)]
    mo = [r.begin_reduced(owned[g].contiguous()).clone() for g, r in enumerate(ranks)]
    ma = torch.cat(mo)
    ro = [r.merge(ma).clone() for r in ranks]
    ra = torch.cat(ro)
    for r in ranks:
        r.finish(ra)


@pytest.mark.parametrize("world", [2, 3])
def test_temporal_sharding_matches_unsharded(ob, world):
    # compression sharded over slices + reduce-scatter of the partials: the
    # summaries equal the unsharded ones up to the summation order, the
    # models to the ALS's sensitivity to that (noisy, well-posed data)
    # noiseless low-rank data: ALS converges to the truth from either order
    # of summation (on noisy data 30 sweeps amplify 1e-16 summary differences)
    x, _ = O.generate_synthetic([60, 60, 70], 3, 3, 0.0, 0.0)
    cfg = _cfg(ob, 3, 8, 12, 3, 38, iters=100, tol=1e-12)
    ref = ob.init_stream(O.slice_mode(x, 2, 0, 40), cfg)
    ranks = [ob.ShardedStream(cfg, g, world, None) for g in range(world)]
    _drive_temporal(ranks, O.slice_mode(x, 2, 0, 40), world)
    for b in range(3):
        batch = O.slice_mode(x, 2, 40 + 10 * b, 10)
        ob.ingest_batch(ref, batch)
        _drive_temporal(ranks, batch, world)
    ys_ref, _ = ref.summaries()
    for g, r in enumerate(ranks):
        ys, _ = r.summaries()
        for i, y in enumerate(ys):
            yr = ys_ref[r.p0 + i]
            assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)
    want = ref.model
    for r in ranks:
        got = r.model
        cong = min(O.congruence(O.KruskalModel(want.factors, want.lambda_), O.KruskalModel(got.factors, got.lambda_)))
        assert cong > 1 - 1e-6
        assert r.slices_seen == ref.slices_seen


def test_temporal_sharding_nonfinite_raises_on_every_rank(ob):
    x = _data()
    cfg = _cfg(ob, 3, 8, 12, 3, 38)
    world = 2
    ranks = [ob.ShardedStream(cfg, g, world, None) for g in range(world)]
    _drive_temporal(ranks, O.slice_mode(x, 2, 0, 40), world)
    bad = np.array(O.slice_mode(x, 2, 40, 10))
    bad[3, 4, 8] = np.nan  # in rank 1's half only
    seen = [r.slices_seen for r in ranks]
    t = bad.shape[2]
    parts = [r.begin_temporal(np.asfortranarray(bad[:, :, 5 * g:5 * (g + 1)]), 5 * g, t).clone()
             for g, r in enumerate(ranks)]
    blk = ranks[0].partial_count
    owned = [sum(p[g * blk:(g + 1) * blk] for p in parts) for g in range(world)]
    for g, r in enumerate(ranks):
        with pytest.raises(ob.NumericError, match="non-finite"):
            r.begin_reduced(owned[g].contiguous())
    # the state is unchanged: the next good batch goes through on both ranks
    _drive_temporal(ranks, O.slice_mode(x, 2, 40, 10), world)
    assert [r.slices_seen for r in ranks] == [s_ + 10 for s_ in seen]
