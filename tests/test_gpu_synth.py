"""On-device generate_synthetic against the reference's
generator restated in the oracle (commands.cpp:110-134, rng.hpp:51-85):
factors bit-exact (host mt19937_64), the clean tensor to 1e-13 (summation
order of reconstruct), the noise in the same flat-order Box-Muller stream to a
few ulp (device log/sin/cos vs glibc), across batch boundaries with an odd
number of entries (the cached spare)."""
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


@pytest.mark.parametrize("dims,rank,sigma,batches", [((13, 7, 9), 3, 0.05, [2, 3, 4]),
                                                     ((40, 31, 12), 4, 0.0, [12]),
                                                     ((33, 21, 10), 5, 0.3, [1, 1, 5, 3])])
def test_synth_matches_reference_generator(ob, dims, rank, sigma, batches):
    want, truth = O.generate_synthetic(list(dims), rank, 77, 0.1 if sigma else 0.0, sigma)  # exact Box-Muller
    g = ob.SynthStream(dims, rank, 77, 0.1 if sigma else 0.0, sigma)
    k = 0
    for t in batches:
        got = g.next(t, "f64").cpu().numpy()
        ref = want[:, :, k:k + t]
        assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))
        k += t
    m = g.truth()  # normalize() of the bit-identical factors (norms summed in another order)
    for f, h in zip(m.factors, truth.factors):
        assert np.allclose(f, h, rtol=1e-14, atol=0)
    assert np.allclose(m.lambda_, truth.lambda_, rtol=1e-14, atol=0)
    with pytest.raises(ob.ConfigError, match="gen: slice range outside the tensor"):
        g.next(1)


def test_synth_fp32_and_errors(ob):
    want, _ = O.generate_synthetic([20, 18, 6], 2, 5, 0.0, 0.01)
    g = ob.SynthStream((20, 18, 6), 2, 5, 0.0, 0.01)
    got = g.next(6, "f32").cpu().numpy()
    assert np.array_equal(got, want.astype(np.float32))  # fp64 values within ulps round to the same fp32 (here)
    with pytest.raises(ob.ConfigError, match="gen: rank must be >= 1"):
        ob.SynthStream((5, 5, 5), 0, 1)
    with pytest.raises(ob.ConfigError, match="gen: noise sigma must be >= 0"):
        ob.SynthStream((5, 5, 5), 2, 1, 0.0, -1.0)
