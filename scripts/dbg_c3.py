"""Debug: c3-scale noiseless stream, fp64/fp32, replica fits."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle import octen_oracle as O
import paper_1807_01350_b200 as ob

I = int(os.environ.get("DBG_I", "1000")); Q = int(os.environ.get("DBG_Q", "100")); P = int(os.environ.get("DBG_P", "16"))
R = int(os.environ.get("DBG_R", "20")); sh = int(os.environ.get("DBG_SH", "10")); K0 = int(os.environ.get("DBG_K0", "1000"))
t = 100
g = torch.Generator(device="cuda"); g.manual_seed(3)
A = torch.rand((I, R), generator=g, device="cuda", dtype=torch.float64)
B = torch.rand((I, R), generator=g, device="cuda", dtype=torch.float64)
C = torch.rand((K0 + t, R), generator=g, device="cuda", dtype=torch.float64)
x = torch.einsum("kr,jr,ir->kji", C, B, A)
for dt in (torch.float64, torch.float32):
    xx = x.to(dt).permute(2, 1, 0)
    cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=3, als=ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3))
    st = ob.init_stream(xx[:, :, :K0], cfg)
    truth = O.KruskalModel([A.cpu().numpy(), B.cpu().numpy(), C[:K0].cpu().numpy()], np.ones(R))
    m = st.model
    print(dt, "init congruence", min(O.congruence(truth, O.KruskalModel(m.factors, m.lambda_))), flush=True)
    ys, _ = st.summaries()
    reps = st.replica_models()
    fits = [O.fitness(y, O.reconstruct_fast(rm)) for y, rm in zip(ys, reps)]
    print("  replica fits", np.round(fits, 3).tolist(), flush=True)
    print("  log", [(r.temporal_residual, r.min_match_similarity) for r in st.log], flush=True)
