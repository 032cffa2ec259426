"""Device stream vs the CPU oracle at the c3 shapes (I = J = 1000, Q = 100,
P = 16, shared = 10, CP-ALS 30 x 3; K0 = 200 + one batch of 100 slices),
fp32 inputs: rank 20 (BASELINE c3) at 1 % and 0.1 % noise, and rank 5 at
1 % noise (a well-posed stream at the same shapes).  Writes the
comparison (summary error, per-replica fits, final fitness, congruence,
temporal residuals) to profiles/r2_c3_parity.json.  GPU box; test-only use
of the oracle."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from threadpoolctl import threadpool_limits
from oracle import octen_oracle as O
import paper_1807_01350_b200 as ob

I, Q, P, SH, K0, T = 1000, 100, 16, 10, 200, 100
out = {"config": {"I": I, "J": I, "K0": K0, "t": T, "Q": Q, "P": P, "shared": SH, "iters": 30,
                  "restarts": 3, "inputs": "fp32 (oracle: the same values in fp64)"}, "runs": []}
for noise, R in ((0.01, 20), (0.001, 20), (0.01, 5)):
    x, _ = O.generate_synthetic([I, I, K0 + T], R, 3, 0.0, 0.0)
    x += noise * np.sqrt(np.mean(x ** 2)) * np.random.default_rng(4).standard_normal(x.shape)
    x32 = np.asfortranarray(x.astype(np.float32))
    x64 = x32.astype(np.float64)
    cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=38,
                          als=ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3))
    t0 = time.time()
    st = ob.init_stream(np.asfortranarray(x32[:, :, :K0]), cfg)
    ob.ingest_batch(st, np.asfortranarray(x32[:, :, K0:]))
    td = time.time() - t0
    with threadpool_limits(limits=1):
        t0 = time.time()
        ocfg = O.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=38, als=O.AlsConfig(R, 30, 1e-8, 3, 0))
        ref = O.init_stream(O.slice_mode(x64, 2, 0, K0), ocfg)
        O.ingest_batch(ref, O.slice_mode(x64, 2, K0, T))
        to = time.time() - t0
    ys, _ = st.summaries()
    yerr = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(ys, ref.summaries.y))
    md = O.KruskalModel(st.model.factors, st.model.lambda_)
    fd = O.fitness(x64, O.reconstruct_fast(md))
    fo = O.fitness(x64, O.reconstruct_fast(ref.model))
    cong = O.congruence(md, ref.model)
    # per-replica CP-ALS of the last batch on the oracle's summaries (identical inputs)
    seeds = [O.rng.derive(38, [O.rng.K_STREAM_ALS, r, 1]) for r in range(P)]
    dm, dfits, _ = ob.cp_als_batched(ref.summaries.y, ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8,
                                                                      n_restarts=3), seeds)
    reps = []
    with threadpool_limits(limits=1):
        for r in range(P):
            w = O.cp_als(ref.summaries.y[r], O.AlsConfig(R, 30, 1e-8, 3, seeds[r]))
            reps.append({"replica": r, "fit_device": float(dfits[r]), "fit_oracle": float(w.fit),
                         "fms": float(min(O.congruence(O.KruskalModel(dm[r].factors, dm[r].lambda_), w.model)))})
    run = {"noise": noise, "rank": R, "summary_max_rel_err": yerr, "fitness_device_pct": fd, "fitness_oracle_pct": fo,
           "congruence_min": float(min(cong)), "congruence_mean": float(np.mean(cong)),
           "temporal_residual_device": [r.temporal_residual for r in st.log],
           "temporal_residual_oracle": [r.temporal_residual for r in ref.log],
           "replica_als": reps, "seconds_device": td, "seconds_oracle": to}
    out["runs"].append(run)
    print(json.dumps({k: v for k, v in run.items() if k != "replica_als"}), flush=True)
    print("replica fit |diff| max %.3e, FMS min %.6f" % (max(abs(a["fit_device"] - a["fit_oracle"]) for a in reps),
                                                        min(a["fms"] for a in reps)), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "r2_c3_parity.json"), "w") as f:
    json.dump(out, f, indent=1)
