"""Where do the device and oracle streams part at rank 5 / 1 % noise with
fp64 inputs (identical summaries)?  Stage-by-stage after init_stream."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from threadpoolctl import threadpool_limits
from oracle import octen_oracle as O
import paper_1807_01350_b200 as ob

I, Q, P, R, SH, K0, T = int(sys.argv[1]), int(sys.argv[2]), 16, 5, 10, 200, 100
x, _ = O.generate_synthetic([I, I, K0 + T], R, 3, 0.0, 0.0)
x += 0.01 * np.sqrt(np.mean(x ** 2)) * np.random.default_rng(4).standard_normal(x.shape)
x = np.asfortranarray(x)
cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=38, als=ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3))
st = ob.init_stream(np.asfortranarray(x[:, :, :K0]), cfg)
with threadpool_limits(1):
    ref = O.init_stream(O.slice_mode(x, 2, 0, K0), O.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=38, als=O.AlsConfig(R, 30, 1e-8, 3, 0)))
ys, hs = st.summaries()
print("summaries", max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(ys, ref.summaries.y)))
rm = st.replica_models()
for p in range(P):
    c = O.congruence(O.KruskalModel(rm[p].factors, rm[p].lambda_), ref.replica_models[p])
    lam = np.max(np.abs(np.sort(rm[p].lambda_) - np.sort(ref.replica_models[p].lambda_)) / np.max(ref.replica_models[p].lambda_))
    print("replica %d FMS %.12f lam %.2e" % (p, min(c), lam))
md = O.KruskalModel(st.model.factors, st.model.lambda_)
print("model congruence", O.congruence(md, ref.model))
print("lambda dev", np.sort(md.lambda_), "ref", np.sort(ref.model.lambda_))
print("residual dev", st.log[-1].temporal_residual, "ref", ref.log[-1].temporal_residual)
print("minmatch dev", st.log[-1].min_match_similarity, "ref", ref.log[-1].min_match_similarity,
      "maxoff dev", st.log[-1].max_offdiag_similarity, "ref", ref.log[-1].max_offdiag_similarity)
for n in range(2):
    print("mode %d factor congruence" % n, [float(abs(a @ b) / np.linalg.norm(a) / np.linalg.norm(b)) for a, b in zip(md.factors[n].T, ref.model.factors[n].T)])
