"""GPU parity at the exact shapes of BASELINE.json's small configs (SURVEY
§8(d) feasibility table):

c1: dense fp64 100x100x200, R=5 U(0,1) truth + N(0, 0.01), K0=100 then 10
    batches of 10, Q=20, P=4, CP-ALS 50 iterations.
c2: dense fp32 500x500x1000, R=10, 1% noise, K0=500 then batches of 50,
    Q=50, P=8, CP-ALS 30 iterations.

At both shapes the reference's merge raises NumericError (P*Q < I, the
replica bound fails).  Parity there is the compressed summaries, the
per-replica CP-ALS models, and the same error from the stream (compared
against the oracle on the same seeded inputs).  Tolerances: fp64 summaries
1e-12 relative; fp32 summaries 1e-4 (north star); CP-ALS fit 1e-7 and
congruence 1 - 1e-6 against the oracle on identical summaries."""
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


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300))


def _cong(a, b):
    return min(O.congruence(O.KruskalModel([f.copy() for f in a.factors], np.asarray(a.lambda_).copy()),
                            O.KruskalModel([f.copy() for f in b.factors], np.asarray(b.lambda_).copy())))


def _replicas(I, J, t, Q, P, sh, seed):
    rs = O.gen_replicas([I, J], Q, P, sh, seed)
    O.extend_temporal(rs, t)
    return rs, [r.nontemporal[0] for r in rs.replicas], [r.nontemporal[1] for r in rs.replicas], \
        [r.temporal for r in rs.replicas]


def _check_config(ob, x, Q, P, sh, R, iters, seed, tol_y, n_als):
    I, J, t = x.shape
    rs, u, v, w = _replicas(I, J, t, Q, P, sh, seed)
    z = ob.compress(x, u, v, w, sh)
    ref = [O.compress(np.asarray(x, dtype=np.float64), rs, r, 0, t) for r in range(P)]
    for a, b in zip(z, ref):
        assert rel(a, b) < tol_y
    # per-replica CP-ALS on identical (oracle) summaries
    seeds = [rng.derive(seed, [8, r, 0]) for r in range(n_als)]
    cfg = ob.AlsConfig(rank=R, max_iters=iters, rel_tol=1e-8, n_restarts=3)
    models, fits, _ = ob.cp_als_batched(ref[:n_als], cfg, seeds)
    for r in range(n_als):
        o = O.cp_als(ref[r], O.AlsConfig(R, iters, 1e-8, 3, seeds[r]))
        assert abs(fits[r] - o.fit) < 1e-7
        assert _cong(models[r], o.model) > 1 - 1e-6


def test_c1_shapes_summaries_als_and_merge_error(ob):
    x, _ = O.generate_synthetic([100, 100, 200], 5, 11, 0.0, 0.01, exact_noise=False)
    first = np.asfortranarray(x[:, :, :100])
    _check_config(ob, first, 20, 4, 4, 5, 50, 21, 1e-12, 4)
    cfg = ob.StreamConfig(rank=5, p=4, q=20, shared=4, seed=21, als=ob.AlsConfig(rank=5, max_iters=50))
    with pytest.raises(ob.NumericError) as dev:
        ob.init_stream(first, cfg)
    with pytest.raises(O.NumericError) as orc:
        O.init_stream(first, O.StreamConfig(rank=5, p=4, q=20, shared=4, seed=21,
                                            als=O.AlsConfig(5, 50, 1e-8, 3, 0)))
    assert str(dev.value) == str(orc.value)


def test_c2_shapes_fp32_summaries_als_and_merge_error(ob):
    # full 500 x 500 slices; 50 slices (one c2 batch) keep the oracle fast
    x, _ = O.generate_synthetic([500, 500, 50], 10, 12, 0.0, 0.0, exact_noise=False)
    x = x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(5).normal_array(x.size, 0, 1).reshape(x.shape, order="F")
    x32 = np.asfortranarray(x.astype(np.float32))
    # tcgen05 split-TF32 with fp32 TMEM accumulation (truncating): a bias of
    # ~K/2 ulps on positive data, 2e-5 here; north-star tolerance 1e-4
    _check_config(ob, x32, 50, 8, 12, 10, 30, 22, 1e-4, 2)
    cfg = ob.StreamConfig(rank=10, p=8, q=50, shared=12, seed=22, als=ob.AlsConfig(rank=10, max_iters=30))
    with pytest.raises(ob.NumericError, match=r"recover: mode 1 projection is 400x500"):
        ob.init_stream(x32, cfg)
