"""CP-ALS at c5 replica shapes (Q=128, R=32, 3 restarts) on noisy low-rank
summaries: the int8 digit-split and the DMMA T-GEMM engines side by side."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_01350_b200 as ob

P, Q, R = int(os.environ.get("P", "8")), 128, 32
g = np.random.default_rng(1)
ys = []
for p in range(P):
    a, b, c = (g.random((Q, R)) for _ in range(3))
    y = np.einsum('ir,jr,kr->ijk', a, b, c)
    y += 0.001 * np.sqrt(np.mean(y * y)) * g.standard_normal(y.shape)
    ys.append(np.asfortranarray(y))
cfg = ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3)
res = {}
for eng in ("i8", "dmma"):
    os.environ["OCTEN_ALS_TGEMM"] = eng
    models, fits, its = ob.cp_als_batched(ys, cfg, list(range(100, 100 + P)))
    res[eng] = (models, fits, its)
    print(eng, "fits", np.round(fits, 10), "its", its, flush=True)
from oracle import octen_oracle as O
for p in range(P):
    mi, md = res["i8"][0][p], res["dmma"][0][p]
    cg = min(O.congruence(O.KruskalModel(mi.factors, mi.lambda_), O.KruskalModel(md.factors, md.lambda_)))
    print("replica %d: fit diff %.3e congruence %.12f" % (p, res["i8"][1][p] - res["dmma"][1][p], cg))
