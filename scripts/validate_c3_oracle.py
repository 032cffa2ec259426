"""One-off full-scale parity run (GPU box): c3 shapes with K0=200, one batch of
100, 1 % noise, exact (fp64) inputs, device stream vs the CPU oracle."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import octen_oracle as O
from oracle import rng
import paper_1807_01350_b200 as ob

I, Q, P, R, sh, K0, t = 1000, 100, 16, 20, 10, 200, 100
x, truth = O.generate_synthetic([I, I, K0 + t], R, 3, 0.0, 0.0)
x = x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape, order="F")
cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=38, als=ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3))
t0 = time.time()
st = ob.init_stream(O.slice_mode(x, 2, 0, K0), cfg)
ob.ingest_batch(st, O.slice_mode(x, 2, K0, t))
td = time.time() - t0
md = O.KruskalModel(st.model.factors, st.model.lambda_)
ys, _ = st.summaries()
t0 = time.time()
ocfg = O.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=38, als=O.AlsConfig(R, 30, 1e-8, 3, 0))
ref = O.init_stream(O.slice_mode(x, 2, 0, K0), ocfg)
O.ingest_batch(ref, O.slice_mode(x, 2, K0, t))
to = time.time() - t0
yerr = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(ys, ref.summaries.y))
fd = O.fitness(x, O.reconstruct_fast(md))
fo = O.fitness(x, O.reconstruct_fast(ref.model))
print("summaries max rel err %.3e" % yerr)
print("fitness device %.6f oracle %.6f" % (fd, fo))
print("congruence device vs oracle %.6f" % min(O.congruence(md, ref.model)))
print("temporal residuals device", [r.temporal_residual for r in st.log], "oracle", [r.temporal_residual for r in ref.log])
print("time device %.1fs oracle %.1fs" % (td, to))
