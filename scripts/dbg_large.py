"""Debug: multi-block paths (d > 64) of the merge against the oracle."""
import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import octen_oracle as O
from oracle import rng
import paper_1807_01350_b200 as ob


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


for (d, Q, P) in [(50, 12, 6), (100, 20, 10), (200, 30, 10), (300, 40, 10), (1000, 100, 16)]:
    rs = O.gen_replicas([d, d], Q, P, 3, 4)
    blocks = [r.nontemporal[0] for r in rs.replicas]
    proj = O.stack_projections(rs, 0)
    truth = rng.Substream(5).fill_uniform(d, 4)
    stack = proj @ truth + 1e-3 * rng.Substream(6).fill_uniform(proj.shape[0], 4)
    got = ob.recover_nontemporal(stack, blocks, 0)
    want = O.recover_nontemporal(stack, proj, 0)
    print("recover_nontemporal d=%d: rel %.3e" % (d, rel(got, want)), flush=True)

# full stream, noiseless, I=J=300
for (I, Q, P, R, sh) in [(100, 20, 8, 4, 3), (300, 40, 12, 5, 5)]:
    s = rng.Substream(91)
    truth = O.KruskalModel([s.fill_uniform(dd, R) for dd in (I, I, 60)], np.ones(R))
    full = O.reconstruct_fast(truth)
    cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=17, als=ob.AlsConfig(rank=R, max_iters=50, rel_tol=1e-10, n_restarts=2))
    st = ob.init_stream(O.slice_mode(full, 2, 0, 40), cfg)
    ob.ingest_batch(st, O.slice_mode(full, 2, 40, 20))
    m = st.model
    mk = O.KruskalModel(m.factors, m.lambda_)
    print("stream I=%d: congruence %.6f fitness %.4f" % (I, min(O.congruence(truth, mk)), O.fitness(full, O.reconstruct_fast(mk))), flush=True)
    # replica models quality
    ys, _ = st.summaries()
    reps = st.replica_models()
    fits = []
    for y, rm in zip(ys, reps):
        fits.append(O.fitness(y, O.reconstruct_fast(rm)))
    print("  replica fits min %.4f" % min(fits), flush=True)
