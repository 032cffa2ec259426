"""Phase timing of als_update (block 0, last launch) and batched CP-ALS wall
time on c3-shape summaries (P=16, Q=100, R=20, 3 restarts, 30 sweeps).
Run with OCTEN_DEBUG_ALS_TSC=1 for the phase cycles."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1807_01350_b200 as ob

P, Q, R = 16, 100, 20
g = np.random.default_rng(0)
ys = []
for p in range(P):
    a, b, c = (g.random((Q, R)) for _ in range(3))
    y = np.einsum('ir,jr,kr->ijk', a, b, c) + 0.01 * g.standard_normal((Q, Q, Q))
    ys.append(np.asfortranarray(y))
seeds = list(range(P))
cfg = ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-30, n_restarts=3)
for rep in range(4):
    t0 = time.time()
    models, fits, its = ob.cp_als_batched(ys, cfg, seeds)
    print("wall %.2f ms  its %s" % ((time.time() - t0) * 1e3, its[:4]), flush=True)
