"""T-GEMM micro run at the c3 lane shape (4 replicas, Q=100, S=3, R=20):
both engines, every mode (for ncu launch timing)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_01350_b200 as ob

rng = np.random.default_rng(0)
p, q, s, r = 4, 100, 3, 20
y = np.abs(rng.standard_normal((p, q, q, q))) + 1.0
f = rng.standard_normal((p, s, 3, q, r))
f /= np.linalg.norm(f, axis=3, keepdims=True)
for rep in range(2):
    for mode in range(3):
        for eng in (1, 0):
            ob.als_tgemm(y, f, mode, engine=eng)
print("ok")
