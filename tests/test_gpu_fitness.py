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
