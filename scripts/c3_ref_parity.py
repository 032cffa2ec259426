"""Device stream vs the reference compiled from its own sources (oracle/_ref)
and vs the oracle restatement, at the c3 shapes (I = J = 1000, Q = 100,
P = 16, shared = 10, CP-ALS 30 x 3; K0 = 200 + one batch of 100 slices), fp32
device inputs (the reference and the oracle get the same values in fp64):
rank 20 (BASELINE c3) at 1 % and 0.1 % noise, rank 5 at 1 % noise.  Also the
per-replica CP-ALS of the last batch on the reference's own summaries
(identical inputs): device cp_als_batched vs the reference's cp_als.
Writes gpurun_out/r2_c3_ref_parity.json.  GPU box; test-only use of
oracle/."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle import octen_oracle as O  # noqa: E402
from oracle import ref_lib as RL  # noqa: E402
import paper_1807_01350_b200 as ob  # noqa: E402

I, Q, P, SH, K0, T = 1000, 100, 16, 10, 200, 100
out = {"config": {"I": I, "J": I, "K0": K0, "t": T, "Q": Q, "P": P, "shared": SH, "iters": 30, "restarts": 3,
                  "inputs": "fp32 on the device; the same values in fp64 for the reference and the oracle"},
       "runs": []}
threadpool_limits(limits=1)
RL.lib()
for noise, R in ((0.01, 20), (0.001, 20), (0.01, 5)):
    x, _ = O.generate_synthetic([I, I, K0 + T], R, 3, 0.0, 0.0)
    x += noise * np.sqrt(np.mean(x ** 2)) * np.random.default_rng(4).standard_normal(x.shape)
    x32 = np.asfortranarray(x.astype(np.float32))
    x64 = x32.astype(np.float64)
    del x
    cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=38,
                          als=ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3))
    ocfg = O.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=38, als=O.AlsConfig(R, 30, 1e-8, 3, 0))
    t0 = time.time()
    st = ob.init_stream(np.asfortranarray(x32[:, :, :K0]), cfg)
    ob.ingest_batch(st, np.asfortranarray(x32[:, :, K0:]))
    td = time.time() - t0
    t0 = time.time()
    ref = RL.RefStream(np.asfortranarray(x64[:, :, :K0]), ocfg)
    ref.ingest(np.asfortranarray(x64[:, :, K0:]))
    tr = time.time() - t0
    O.MERGE_PROCESSES = True
    t0 = time.time()
    orc = O.init_stream(O.slice_mode(x64, 2, 0, K0), ocfg)
    O.ingest_batch(orc, O.slice_mode(x64, 2, K0, T))
    to = time.time() - t0
    ys, _ = st.summaries()
    yr = ref.summaries()
    y_dev = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(ys, yr))
    y_orc = max(float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(orc.summaries.y, yr))
    md = O.KruskalModel(st.model.factors, st.model.lambda_)
    mr = ref.model()
    fd = O.fitness(x64, O.reconstruct_fast(md))
    fr = O.fitness(x64, O.reconstruct_fast(mr))
    fo = O.fitness(x64, O.reconstruct_fast(orc.model))
    c_dev = RL.congruence(mr, md)
    c_orc = RL.congruence(mr, orc.model)
    # per-replica CP-ALS of the last batch on the reference's summaries
    seeds = [O.rng.derive(38, [O.rng.K_STREAM_ALS, r, 1]) for r in range(P)]
    dm, dfits, dits = ob.cp_als_batched(list(yr), ob.AlsConfig(rank=R, max_iters=30, rel_tol=1e-8, n_restarts=3),
                                        seeds)
    reps = []
    for r in range(P):
        w = RL.cp_als(yr[r], R, 30, 1e-8, 3, seeds[r])
        reps.append({"replica": r, "fit_device": float(dfits[r]), "fit_reference": float(w.fit),
                     "iters_device": int(dits[r]), "iters_reference": int(w.iterations),
                     "fms": float(min(RL.congruence(w.model, O.KruskalModel(dm[r].factors, dm[r].lambda_))))})
    rl = ref.log()
    run = {"noise": noise, "rank": R,
           "summary_max_rel_err_device_vs_reference": y_dev, "summary_max_rel_err_oracle_vs_reference": y_orc,
           "fitness_pct": {"device": fd, "reference": fr, "oracle": fo},
           "congruence_vs_reference": {"device_min": float(min(c_dev)), "device_mean": float(np.mean(c_dev)),
                                       "oracle_min": float(min(c_orc)), "oracle_mean": float(np.mean(c_orc))},
           "temporal_residual": {"device": [r.temporal_residual for r in st.log],
                                 "reference": [float(r["temporal_residual"]) for r in rl],
                                 "oracle": [r.temporal_residual for r in orc.log]},
           "min_match_similarity": {"device": [r.min_match_similarity for r in st.log],
                                    "reference": [float(r["min_match_similarity"]) for r in rl],
                                    "oracle": [r.min_match_similarity for r in orc.log]},
           "replica_als_on_reference_summaries": reps,
           "replica_fit_absdiff_max": max(abs(a["fit_device"] - a["fit_reference"]) for a in reps),
           "replica_fms_min": min(a["fms"] for a in reps),
           "seconds": {"device": td, "reference": tr, "oracle": to}}
    out["runs"].append(run)
    print(json.dumps({k: v for k, v in run.items() if k != "replica_als_on_reference_summaries"}), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "r2_c3_ref_parity.json"), "w") as f:
    json.dump(out, f, indent=1)
