"""ALS on c3-shape noisy summaries: device cp_als_batched vs the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from oracle import octen_oracle as O
from oracle import rng
import paper_1807_01350_b200 as ob

I, Q, P, R, sh, K0 = 1000, 100, 16, 20, 10, 200
x, truth = O.generate_synthetic([I, I, K0], R, 3, 0.0, 0.0)
x = x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape, order="F")
rs = O.gen_replicas([I, I], Q, P, sh, 38)
O.extend_temporal(rs, K0)
u = [r.nontemporal[0] for r in rs.replicas][:4]
v = [r.nontemporal[1] for r in rs.replicas][:4]
w = [r.temporal for r in rs.replicas][:4]
ys = ob.compress(x, u, v, w, sh)
seeds = [rng.derive(38, [rng.K_STREAM_ALS, r, 0]) for r in range(4)]
for iters, tol in [(30, 1e-8), (300, 1e-10)]:
    models, fits, its = ob.cp_als_batched(ys, ob.AlsConfig(rank=R, max_iters=iters, rel_tol=tol, n_restarts=3), seeds)
    for r in range(4):
        t0 = time.time()
        ref = O.cp_als(ys[r], O.AlsConfig(R, iters, tol, 3, seeds[r]))
        c = min(O.congruence(O.KruskalModel(models[r].factors, models[r].lambda_), ref.model))
        print("iters %d replica %d: fit dev %.8f ora %.8f  its %d/%d  congruence %.4f (%.0fs)" %
              (iters, r, fits[r], ref.fit, its[r], ref.iterations, c, time.time() - t0), flush=True)
