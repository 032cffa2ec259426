"""Fitness (eval.cpp:10-20) of the streamed model on its last batches, c3 bench data (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1807_01350_b200 as ob
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
noise = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
I, J, K0, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
dev = torch.device("cuda", 0)
syn = bench.Synth(torch, dev, I, J, K0 + 6 * t, R, seed=1234, noise=noise)
st = ob.init_stream(syn.batch(0, K0), ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * 1234 + 3,
                    als=ob.AlsConfig(max_iters=cfg["iters"], rel_tol=1e-8, n_restarts=3)))
for b in range(5):
    x = syn.batch(K0 + b * t, t)
    ob.ingest_batch(st, x)
    m = st.model
    f = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in m.factors]
    lam = torch.from_numpy(np.asarray(m.lambda_)).to(dev)
    k0 = K0 + b * t
    xh = torch.einsum("kr,jr,ir->kji", f[2][k0:k0 + t] * lam[None, :], f[1], f[0])
    xd = x.permute(2, 1, 0).to(torch.float64)
    fit = 100.0 * (1.0 - float((xd - xh).norm() / xd.norm()))
    # the truth's own fitness (noise floor)
    xt = torch.einsum("kr,jr,ir->kji", syn.C[k0:k0 + t], syn.B, syn.A)
    fit_t = 100.0 * (1.0 - float((xd - xt).norm() / xd.norm()))
    rec = st.log[-1]
    print("batch %d: model fitness %.4f%%  (ground truth %.4f%%)  temporal residual %.3g" % (b + 1, fit, fit_t, rec.temporal_residual), flush=True)
