"""Golden fixtures (tests/golden/*.npz, written by tests/golden/make_golden.py
from the oracle on seeded inputs).  CPU: the oracle still reproduces them
(guards the checker itself).  GPU: the device path reproduces them without
running the oracle.  Tolerances are written per comparison."""
import os
import sys

import numpy as np
import pytest

from oracle import octen_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden as G  # noqa: E402


def load(name):
    return dict(np.load(os.path.join(HERE, "golden", name + ".npz")))


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def congr(fa, la, fb, lb):
    return min(O.congruence(O.KruskalModel([f.copy() for f in fa], np.asarray(la).copy()),
                            O.KruskalModel([f.copy() for f in fb], np.asarray(lb).copy())))


@pytest.mark.parametrize("name", sorted(G.CASES))
def test_oracle_reproduces_golden(name):
    got, ref = G.CASES[name](), load(name)
    assert set(got) == set(ref)
    for k in ref:
        assert np.asarray(got[k]).shape == ref[k].shape, k
        assert rel(np.asarray(got[k], dtype=np.float64), ref[k].astype(np.float64)) < 1e-9, k


# ------------------------------------------------------------------ device

@pytest.fixture(scope="module")
def ob():
    import paper_1807_01350_b200 as m
    return m


@pytest.mark.gpu
def test_device_compress_golden(ob):
    g = load("compress")
    I, J, t, Q, P, sh, seed = (int(v) for v in g["shape"])
    rs = O.gen_replicas([I, J], Q, P, sh, seed)
    O.extend_temporal(rs, t)
    x = (G.rng.Substream(9).uniform01_array(I * J * t) * 2 - 1).reshape((I, J, t), order="F")
    z = ob.compress(x, [r.nontemporal[0] for r in rs.replicas], [r.nontemporal[1] for r in rs.replicas],
                    [r.temporal for r in rs.replicas], sh)
    for r in range(P):
        assert rel(z[r], g["z"][r]) < 1e-12  # fp64 input: accumulation order only


@pytest.mark.gpu
def test_device_als_golden(ob):
    g = load("als")
    truth = O.KruskalModel([G.rng.Substream(300 + n).fill_uniform(9, 3) for n in range(3)], np.ones(3))
    y = O.reconstruct(truth) + 1e-3 * G.rng.Substream(310).normal_array(9 ** 3, 0, 1).reshape((9, 9, 9), order="F")
    models, fits, iters = ob.cp_als_batched([y], ob.AlsConfig(rank=3, max_iters=50, rel_tol=1e-10, n_restarts=2),
                                            [1234])
    assert abs(fits[0] - g["fit"][0]) < 1e-8
    assert congr(models[0].factors, models[0].lambda_, [g["a"], g["b"], g["c"]], g["lam"]) > 1 - 1e-7
    assert np.allclose(np.sort(models[0].lambda_), np.sort(g["lam"]), rtol=1e-6)


def _device_stream(ob, x, rank, p, q, shared, seed, iters, tol, restarts, k0, t, nb):
    cfg = ob.StreamConfig(rank=rank, p=p, q=q, shared=shared, seed=seed,
                          als=ob.AlsConfig(rank=rank, max_iters=iters, rel_tol=tol, n_restarts=restarts))
    st = ob.init_stream(O.slice_mode(x, 2, 0, k0), cfg)
    for b in range(nb):
        ob.ingest_batch(st, O.slice_mode(x, 2, k0 + b * t, t))
    return st


def _check_stream(st, g, congr_tol, resid_tol):
    m = st.model
    assert congr(m.factors, m.lambda_, [g["a"], g["b"], g["c"]], g["lam"]) > 1 - congr_tol
    ys, hs = st.summaries()
    for r in range(len(ys)):
        assert rel(ys[r], g["y"][r]) < 1e-12
    assert len(st.log) == g["records"].shape[0]
    for rec, ref in zip(st.log, g["records"]):
        assert rec.batch_index == int(ref[0]) and rec.t_new == int(ref[1])
        assert abs(rec.temporal_residual - ref[2]) < resid_tol * max(1.0, ref[2])
        assert rec.warned == bool(ref[5])


@pytest.mark.gpu
def test_device_stream_noiseless_golden(ob):
    s = G.rng.Substream(91)
    truth = O.KruskalModel([s.fill_uniform(d, 4) for d in (30, 30, 20)], np.ones(4))
    st = _device_stream(ob, O.reconstruct(truth), 4, 6, 15, 3, 17, 300, 1e-12, 2, 5, 5, 3)
    _check_stream(st, load("stream_noiseless"), 1e-8, 1e-6)


@pytest.mark.gpu
def test_device_stream_noisy_golden(ob):
    st = _device_stream(ob, G.noisy_input(), 3, 8, 12, 3, 38, 30, 1e-8, 3, 40, 10, 2)
    _check_stream(st, load("stream_noisy"), 1e-6, 1e-6)
