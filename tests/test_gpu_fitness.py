"""Device-side evaluation: the fitness of the stream's model
on a batch of its slices (eval.cpp:10-20), computed without materialising the
reconstruction, against numpy on the reconstructed slices."""
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


@pytest.mark.parametrize("noise,dtype", [(0.0, np.float64), (0.02, np.float64), (0.02, np.float32)])
def test_batch_fitness_matches_numpy(ob, noise, dtype):
    x, _ = O.generate_synthetic([60, 50, 70], 3, 7, 0.0, 0.0)
    if noise:
        x = x + noise * np.sqrt(np.mean(x ** 2)) * np.random.default_rng(1).standard_normal(x.shape)
    x = np.asfortranarray(x.astype(dtype))
    cfg = ob.StreamConfig(rank=3, p=8, q=12, shared=3, seed=5, als=ob.AlsConfig(rank=3, max_iters=60, rel_tol=1e-10))
    st = ob.init_stream(x[:, :, :40], cfg)
    for b in range(3):
        ob.ingest_batch(st, np.asfortranarray(x[:, :, 40 + 10 * b:50 + 10 * b]))
    m = st.model
    xh = O.reconstruct(O.KruskalModel(m.factors, m.lambda_))
    for k0, t in ((0, 40), (40, 10), (60, 10), (0, 70)):
        sl = np.asfortranarray(x[:, :, k0:k0 + t])
        want = O.fitness(sl.astype(np.float64), xh[:, :, k0:k0 + t])
        got = st.batch_fitness(sl, k0)
        # |X - Xhat|^2 = |X|^2 - 2 <X, Xhat> + |Xhat|^2 cancels when the fit is
        # near-exact: the residual norm is resolved to ~sqrt(eps) |X|, i.e.
        # the fitness to ~1e-6 percentage points
        assert abs(got - want) < 5e-6 + 1e-8 * abs(want)
    if noise == 0.0:
        assert st.batch_fitness(np.asfortranarray(x[:, :, 60:70]), 60) > 99.9
    with pytest.raises(ob.ConfigError):
        st.batch_fitness(np.asfortranarray(x[:, :, 60:70]), 65)  # past the slices seen


def test_batch_fitness_reference_errors(ob):
    # eval.cpp:13 zero-norm reference tensor; tensor.cpp DenseTensor rejects
    # non-finite values before fitness runs
    x, _ = O.generate_synthetic([30, 28, 20], 2, 9, 0.0, 0.0)
    x = np.asfortranarray(x)
    cfg = ob.StreamConfig(rank=2, p=6, q=8, shared=2, seed=3, als=ob.AlsConfig(rank=2, max_iters=50))
    st = ob.init_stream(x[:, :, :12], cfg)
    with pytest.raises(ob.NumericError, match="fitness: zero-norm reference tensor"):
        st.batch_fitness(np.zeros((30, 28, 4), order="F"), 0)
    bad = np.array(x[:, :, :4], order="F")
    bad[3, 2, 1] = np.nan
    with pytest.raises(ob.NumericError, match="DenseTensor: non-finite value"):
        st.batch_fitness(bad, 0)


def test_measured_footprint_matches_accounting(ob):
    # test_eval.cpp:104-126 on the device-resident state
    from oracle import rng
    s = rng.Substream(31)
    truth = O.KruskalModel([s.fill_uniform(d, 2) for d in (10, 9, 12)], np.ones(2))
    full = O.reconstruct_fast(truth)
    cfg = ob.StreamConfig(rank=2, p=4, q=6, shared=2, seed=7, als=ob.AlsConfig(rank=2, max_iters=120))
    st = ob.init_stream(O.slice_mode(full, 2, 0, 6), cfg)
    ob.ingest_batch(st, O.slice_mode(full, 2, 6, 6))
    fp = st.footprint()
    assert fp["summary_bytes"] == 8 * 4 * 6 * 6 * 6
    assert fp["replica_bytes"] == 8 * 4 * 6 * (10 + 9)
    assert fp["accumulator_bytes"] == 8 * 4 * 6 * 2
    assert fp["factor_bytes"] == 8 * (2 * (10 + 9 + 12) + 2)
    ref = O.init_stream(O.slice_mode(full, 2, 0, 6), O.StreamConfig(rank=2, p=4, q=6, shared=2, seed=7,
                                                                     als=O.AlsConfig(2, 120, 1e-8, 3, 0)))
    O.ingest_batch(ref, O.slice_mode(full, 2, 6, 6))
    want = O.measure_footprint(ref)
    for k in want:
        assert fp[k] == want[k]
