"""Generate the golden fixtures in tests/golden/ from the CPU oracle.

    python tests/golden/make_golden.py

The fixtures are oracle outputs on small seeded inputs; the reference
compiled from its own sources (oracle/_ref) reproduces every
one of them (tests/test_ref_pin.py::test_golden_fixtures_reproduced_by_reference).
Every input is regenerated from its seed by the bit-exact host RNG
(oracle/rng.py = proj/include/cpstream/rng.hpp), so the fixtures store only
seeds, shapes and outputs.  Test infrastructure only.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import octen_oracle as O  # noqa: E402
from oracle import rng  # noqa: E402


def compress_case():
    I, J, t, Q, P, sh, seed = 40, 33, 9, 8, 4, 3, 55
    rs = O.gen_replicas([I, J], Q, P, sh, seed)
    O.extend_temporal(rs, t)
    x = (rng.Substream(9).uniform01_array(I * J * t) * 2 - 1).reshape((I, J, t), order="F")
    z = np.stack([O.compress(x, rs, r, 0, t) for r in range(P)])
    return dict(shape=np.array([I, J, t, Q, P, sh, seed]), z=z)


def als_case():
    truth = O.KruskalModel([rng.Substream(300 + n).fill_uniform(9, 3) for n in range(3)], np.ones(3))
    y = O.reconstruct(truth) + 1e-3 * rng.Substream(310).normal_array(9 ** 3, 0, 1).reshape((9, 9, 9), order="F")
    res = O.cp_als(y, O.AlsConfig(3, 50, 1e-10, 2, 1234))
    return dict(fit=np.array([res.fit]), lam=res.model.lambda_, a=res.model.factors[0], b=res.model.factors[1],
                c=res.model.factors[2], iters=np.array([res.iterations]))


def stream_noiseless_case():
    # proj/tests/test_streaming.cpp:78-96
    s = rng.Substream(91)
    truth = O.KruskalModel([s.fill_uniform(d, 4) for d in (30, 30, 20)], np.ones(4))
    full = O.reconstruct(truth)
    cfg = O.StreamConfig(rank=4, p=6, q=15, shared=3, seed=17, als=O.AlsConfig(4, 300, 1e-12, 2, 0))
    st = O.init_stream(O.slice_mode(full, 2, 0, 5), cfg)
    for b in range(1, 4):
        O.ingest_batch(st, O.slice_mode(full, 2, 5 * b, 5))
    return _stream_out(st)


def noisy_input():
    I, K0, t, R = 60, 40, 10, 3
    x, _ = O.generate_synthetic([I, I, K0 + 2 * t], R, 3, 0.0, 0.0)
    x = x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape, order="F")
    return x


def stream_noisy_case():
    x = noisy_input()
    cfg = O.StreamConfig(rank=3, p=8, q=12, shared=3, seed=38, als=O.AlsConfig(3, 30, 1e-8, 3, 0))
    st = O.init_stream(O.slice_mode(x, 2, 0, 40), cfg)
    for b in range(2):
        O.ingest_batch(st, O.slice_mode(x, 2, 40 + b * 10, 10))
    return _stream_out(st)


def _stream_out(st):
    m = st.model
    rec = np.array([[r.batch_index, r.t_new, r.temporal_residual, r.min_match_similarity,
                     r.max_offdiag_similarity, float(r.warned)] for r in st.log])
    return dict(a=m.factors[0], b=m.factors[1], c=m.factors[2], lam=m.lambda_, records=rec,
                y=np.stack(st.summaries.y), hist=np.stack(st.summaries.history))


CASES = {"compress": compress_case, "als": als_case, "stream_noiseless": stream_noiseless_case,
         "stream_noisy": stream_noisy_case}

if __name__ == "__main__":
    for name, fn in CASES.items():
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **fn())
        print("wrote", path, os.path.getsize(path))
