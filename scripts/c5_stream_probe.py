"""c5 stream (bench's synthetic data, 0.1 % noise) batch by batch with both
CP-ALS T-GEMM engines: where do the replica models part ways?"""
import importlib.util
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)
import paper_1807_01350_b200 as ob
from oracle import octen_oracle as O

cfg = bench.CONFIGS["c5"]
I, J, K0, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
dev = torch.device("cuda", 0)
nb = int(os.environ.get("NB", "3"))
syn = bench.Synth(torch, dev, I, J, K0 + nb * t, R, seed=1234, noise=float(os.environ.get("NOISE", "0.001")))
batches = [syn.batch(0, K0)] + [syn.batch(K0 + i * t, t) for i in range(nb)]
scfg = lambda: ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * 1234 + 3,
                               als=ob.AlsConfig(max_iters=cfg["iters"], rel_tol=1e-8, n_restarts=cfg["restarts"]))
out = {}
for eng in os.environ.get("ENGINES", "dmma,i8").split(","):
    os.environ["OCTEN_ALS_TGEMM"] = eng
    st = ob.init_stream(batches[0], scfg())
    hist = [st.replica_models()]
    for b in range(nb):
        try:
            ob.ingest_batch(st, batches[1 + b])
        except Exception as e:
            print(eng, "batch", b + 1, "raised:", e, flush=True)
            break
        hist.append(st.replica_models())
    out[eng] = hist
for b in (range(min(len(out["dmma"]), len(out["i8"]))) if len(out) == 2 else []):
    md, mi = out["dmma"][b], out["i8"][b]
    worst = []
    for p in range(P):
        cg = min(O.congruence(O.KruskalModel(md[p].factors, md[p].lambda_), O.KruskalModel(mi[p].factors, mi[p].lambda_)))
        worst.append(cg)
    print("after batch %d: replica congruence dmma vs i8: min %.6f, replicas < 0.999: %s" % (
        b, min(worst), [p for p, c in enumerate(worst) if c < 0.999]), flush=True)
