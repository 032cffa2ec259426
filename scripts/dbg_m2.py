import sys, numpy as np
sys.path.insert(0, '.')
from oracle import octen_oracle as O
from oracle import rng
import paper_1807_01350_b200 as ob
def run(I, J, t, Q, P, sh):
    rs = O.gen_replicas([I, J], Q, P, sh, 55); O.extend_temporal(rs, t)
    u = [r.nontemporal[0] for r in rs.replicas]; v = [r.nontemporal[1] for r in rs.replicas]; w = [r.temporal for r in rs.replicas]
    x = rng.Substream(10).uniform01_array(I*J*t).reshape((I, J, t), order='F').astype(np.float32)
    got = ob.compress(x, u, v, w, sh)
    want = O.compress(x.astype(np.float64), rs, 0, 0, t)
    print((I,J,t,Q,P,sh), np.linalg.norm(got[0]-want)/np.linalg.norm(want), flush=True)
shape = tuple(int(a) for a in sys.argv[1:])
run(*shape)
