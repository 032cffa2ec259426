import sys, os
import numpy as np
sys.path.insert(0, '.')
from oracle import octen_oracle as O
from oracle import rng
import paper_1807_01350_b200 as ob
I = J = int(os.environ.get("DBG_I", "1000")); Q = 100; P = 16; sh = 10
for t in [int(a) for a in os.environ.get("DBG_T", "10 100 167 168 200 400").split()]:
    rs = O.gen_replicas([I, J], Q, P, sh, 55)
    O.extend_temporal(rs, t)
    u = [r.nontemporal[0] for r in rs.replicas]; v = [r.nontemporal[1] for r in rs.replicas]; w = [r.temporal for r in rs.replicas]
    x = (rng.Substream(9).uniform01_array(I * J * t)).reshape((I, J, t), order="F")
    z64 = ob.compress(x, u, v, w, sh)
    z32 = ob.compress(x.astype(np.float32), u, v, w, sh)
    errs = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(z32, z64)]
    print("t=%d rel err fp32-tc vs fp64: max %.3e min %.3e" % (t, max(errs), min(errs)), flush=True)
