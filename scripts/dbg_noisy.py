"""Noisy stream: device vs oracle at reduced scale, and device fitness at c3."""
import sys, os, time
import numpy as np
sys.path.insert(0, '.')
from oracle import octen_oracle as O
from oracle import rng
import paper_1807_01350_b200 as ob

def run(I, Q, P, R, sh, K0, t, nb, noise, oracle=True):
    x, truth = O.generate_synthetic([I, I, K0 + nb * t], R, 3, 0.0, 0.0)
    x = x + noise * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape, order="F")
    cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=38, als=ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3))
    st = ob.init_stream(O.slice_mode(x, 2, 0, K0), cfg)
    fits = [O.fitness(O.slice_mode(x, 2, 0, K0), O.reconstruct_fast(O.KruskalModel(st.model.factors, st.model.lambda_)))]
    for b in range(nb):
        ob.ingest_batch(st, O.slice_mode(x, 2, K0 + b * t, t))
        xs = O.slice_mode(x, 2, 0, K0 + (b + 1) * t)
        fits.append(O.fitness(xs, O.reconstruct_fast(O.KruskalModel(st.model.factors, st.model.lambda_))))
    print("device", (I, Q, P, R, sh), "fits", np.round(fits, 3).tolist(), "resid", [round(r.temporal_residual, 6) for r in st.log], flush=True)
    if oracle:
        t0 = time.time()
        ocfg = O.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=38, als=O.AlsConfig(R, 30, 1e-8, 3, 0))
        ref = O.init_stream(O.slice_mode(x, 2, 0, K0), ocfg)
        ofits = [O.fitness(O.slice_mode(x, 2, 0, K0), O.reconstruct_fast(ref.model))]
        for b in range(nb):
            O.ingest_batch(ref, O.slice_mode(x, 2, K0 + b * t, t))
            xs = O.slice_mode(x, 2, 0, K0 + (b + 1) * t)
            ofits.append(O.fitness(xs, O.reconstruct_fast(ref.model)))
        print("oracle", "fits", np.round(ofits, 3).tolist(), "resid", [round(r.temporal_residual, 6) for r in ref.log], "%.0fs" % (time.time() - t0), flush=True)

for spec in os.environ.get("DBG_SPECS", "120,20,10,10,4,60,20,2").split(";"):
    I, Q, P, R, sh, K0, t, nb = [int(v) for v in spec.split(",")]
    run(I, Q, P, R, sh, K0, t, nb, 0.01, oracle=I <= 300)
