"""Device path against the reference itself (the library compiled from
proj/src by oracle/Makefile into oracle/_ref, prebuilt in this container and
shipped with the snapshot): streams, batched CP-ALS, the generator, errors
and OCTS checkpoint interchange, on the same inputs.  The oracle-based GPU
tests stay; these close the loop to the reference without the restatement in
between.  Tolerances: summaries 1e-12 (fp64 inputs), models through
congruence (column order / sign are gauge), fits ~sqrt(eps) (the reference's
fit formula cancels near 1)."""
import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import ref_lib as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    if not R.available():
        pytest.fail("oracle/_ref/libcpstream_ref.so missing from the snapshot (make -C oracle)")
    R.lib()
    import paper_1807_01350_b200 as m
    return m


def _cfgs(ob, **kw):
    als = kw.pop("als")
    return (ob.StreamConfig(als=ob.AlsConfig(rank=kw["rank"], **als), **kw),
            O.StreamConfig(als=O.AlsConfig(rank=kw["rank"], **als), **kw))


def _ob_model(m):
    return O.KruskalModel([np.asarray(f) for f in m.factors], np.asarray(m.lambda_))


def _compare(dev, ref, tol_model=1e-8, tol_y=1e-12, tol_rec=1e-6):
    ys, _ = dev.summaries()
    yr = ref.summaries()
    for a, b in zip(ys, yr):
        assert np.abs(a - b).max() <= tol_y * max(1.0, np.abs(b).max())
    dm = _ob_model(dev.model)
    rm = ref.model()
    assert min(R.congruence(rm, dm)) > 1 - tol_model
    np.testing.assert_allclose(np.sort(dm.lambda_), np.sort(rm.lambda_), rtol=max(1e-6, 100 * tol_model))
    for a, b in zip(dev.log, ref.log()):
        assert a.batch_index == int(b["batch_index"]) and a.t_new == int(b["t_new"])
        assert abs(a.temporal_residual - b["temporal_residual"]) <= tol_rec * max(1.0, b["temporal_residual"])
        assert abs(a.min_match_similarity - b["min_match_similarity"]) <= tol_rec
        assert a.warned == bool(b["warned"])


@pytest.mark.parametrize("dims,rank,noise,p,q,sh", [([30, 25, 20], 4, 0.0, 8, 10, 3), ([30, 25, 20], 4, 0.01, 8, 10, 3),
                                                   ([40, 40, 30], 3, 0.01, 8, 12, 4)])
def test_stream_matches_reference(ob, dims, rank, noise, p, q, sh):
    """Well-posed streams.  (At 5 % noise on the first shape the alignment
    similarities fall to 0.003 - 0.04: the greedy matching decides near-ties
    and any rounding difference picks another permutation; the device's
    normal-equation merge and the reference's QR end at different, equally
    poor models there, while the oracle, with the reference's own QR, tracks
    it to 1e-11 -- tests/test_ref_pin.py.)"""
    x, _ = R.generate_synthetic(dims, rank, 41, 0.0, noise)
    dc, rc = _cfgs(ob, rank=rank, p=p, q=q, shared=sh, seed=124, als=dict(max_iters=100, rel_tol=1e-8, n_restarts=3))
    dev = ob.init_stream(x[:, :, :5], dc)
    ref = R.RefStream(x[:, :, :5], rc)
    for k in range(5, dims[2], 5):
        ob.ingest_batch(dev, x[:, :, k:k + 5])
        ref.ingest(x[:, :, k:k + 5])
    _compare(dev, ref)


def test_stream_temporal_mode_0_matches_reference(ob):
    x, _ = R.generate_synthetic([12, 18, 16], 3, 42, 0.0, 0.01)
    dc, rc = _cfgs(ob, rank=3, p=6, q=8, shared=2, seed=7, temporal_mode=0,
                   als=dict(max_iters=80, rel_tol=1e-8, n_restarts=2))
    dev = ob.init_stream(np.asfortranarray(x[:6]), dc)
    ref = R.RefStream(x[:6], rc)
    for k in (6, 9):
        ob.ingest_batch(dev, np.asfortranarray(x[k:k + 3]))
        ref.ingest(x[k:k + 3])
    _compare(dev, ref)


def test_stream_fp32_tcgen05_matches_reference(ob):
    """fp32 batches (tcgen05 split-TF32 compression): summaries within the
    fp32 input tolerance of the reference fed the same fp32 values."""
    x, _ = R.generate_synthetic([40, 36, 24], 3, 43, 0.0, 0.01)
    x32 = x.astype(np.float32)
    dc, rc = _cfgs(ob, rank=3, p=6, q=16, shared=4, seed=9, als=dict(max_iters=100, rel_tol=1e-8, n_restarts=2))
    before = ob.kernel_counts()
    dev = ob.init_stream(x32[:, :, :12], dc)
    ref = R.RefStream(x32[:, :, :12].astype(np.float64), rc)
    ob.ingest_batch(dev, x32[:, :, 12:])
    ref.ingest(x32[:, :, 12:].astype(np.float64))
    after = ob.kernel_counts()
    assert after["tcgen05"] > before["tcgen05"]
    assert after["simt_fallbacks"] == before["simt_fallbacks"]
    _compare(dev, ref, tol_model=1e-4, tol_y=2e-5, tol_rec=2e-3)


def test_cp_als_batched_matches_reference(ob):
    """The device's batched CP-ALS on several Q^3 tensors against the
    reference's cp_als with the same per-tensor seeds (well-posed data: in a
    swamp, e.g. 5 % noise here, the |dfit| < tol stop fires at a sweep that
    depends on rounding and the fits part at 1e-6)."""
    tensors, seeds = [], []
    for i, (sig, r) in enumerate([(1e-3, 4), (1e-2, 4), (0.0, 4), (3e-3, 4)]):
        t, _ = R.generate_synthetic([12, 12, 12], r, 60 + i, 0.0, sig)
        tensors.append(t)
        seeds.append(1000 + i)
    cfg = ob.AlsConfig(rank=4, max_iters=100, rel_tol=1e-8, n_restarts=3)
    models, fits, iters = ob.cp_als_batched(tensors, cfg, seeds)
    for t, s, m, f, it in zip(tensors, seeds, models, fits, iters):
        r = R.cp_als(t, 4, 100, 1e-8, 3, s)
        assert abs(f - r.fit) < 1e-7
        if r.fit < 1 - 1e-6:  # near fit 1 the stop test |dfit| < tol reads rounding noise (cp_als.cpp:340)
            assert int(it) == r.iterations
        assert min(R.congruence(r.model, _ob_model(m))) > 1 - 1e-8


def test_generator_matches_reference(ob):
    want, truth = R.generate_synthetic([33, 21, 10], 5, 77, 0.1, 0.3)
    g = ob.SynthStream((33, 21, 10), 5, 77, 0.1, 0.3)
    got = np.concatenate([g.next(t, "f64").cpu().numpy() for t in (1, 4, 5)], axis=2)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
    m = g.truth()
    for f, h in zip(m.factors, truth.factors):
        np.testing.assert_allclose(f, h, rtol=1e-14, atol=1e-15)


def test_errors_match_reference(ob):
    x, _ = R.generate_synthetic([20, 18, 12], 3, 43, 0.0, 0.0)
    for kw, exc in ((dict(p=2, enforce_bounds=True), "ConfigError"), (dict(p=2), "NumericError")):
        dc, rc = _cfgs(ob, rank=3, q=8, shared=2, seed=1, als=dict(), **kw)
        with pytest.raises(getattr(O, exc)) as a:
            R.RefStream(x[:, :, :4], rc)
        with pytest.raises(getattr(ob, exc)) as b:
            ob.init_stream(x[:, :, :4], dc)
        assert str(a.value) == str(b.value)


def test_checkpoint_interchange_with_reference(ob):
    """OCTS bytes written by the device resume in the reference and the
    reference's bytes resume on the device; both continue like the
    uninterrupted streams."""
    x, _ = R.generate_synthetic([20, 18, 16], 3, 44, 0.0, 0.01)
    dc, rc = _cfgs(ob, rank=3, p=6, q=8, shared=2, seed=9, als=dict(max_iters=60, rel_tol=1e-8, n_restarts=2))
    dev = ob.init_stream(x[:, :, :4], dc)
    ref = R.RefStream(x[:, :, :4], rc)
    ob.ingest_batch(dev, x[:, :, 4:8])
    ref.ingest(x[:, :, 4:8])
    db, rb = dev.checkpoint_save(), ref.checkpoint()
    assert len(db) == len(rb) and db[:4] == rb[:4] == b"OCTS"
    ref_from_dev = R.RefStream.load(db)
    dev_from_ref = ob.checkpoint_load(rb)
    for s in (dev, ref, ref_from_dev, dev_from_ref):
        if isinstance(s, R.RefStream):
            s.ingest(x[:, :, 8:12])
        else:
            ob.ingest_batch(s, x[:, :, 8:12])
    _compare(dev, ref_from_dev)
    _compare(dev_from_ref, ref)
