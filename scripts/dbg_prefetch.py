"""Time host-batch ingest with and without prefetch on c3 shapes (diagnostic)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1807_01350_b200 as ob
cfg = bench.CONFIGS["c3"]
I, J, K0, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
dev = torch.device("cuda", 0)
syn = bench.Synth(torch, dev, I, J, K0 + 12 * t, R, seed=1234)
st = ob.init_stream(syn.batch(0, K0), ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7,
                    als=ob.AlsConfig(max_iters=30, rel_tol=1e-8, n_restarts=3)))
hb = []
for i in range(10):
    d = syn.batch(K0 + i * t, t)
    h = torch.empty((t, J, I), dtype=torch.float32, pin_memory=True)
    h.copy_(d.permute(2, 1, 0))
    hb.append(h.permute(2, 1, 0))
torch.cuda.synchronize()
ob.ingest_batch(st, hb[0])
for mode in ("plain", "prefetch", "plain"):
    ts = []
    idx = list(range(1, 5)) if mode == "plain" else list(range(5, 10))
    if mode == "prefetch":
        st.prefetch(hb[idx[0]])
    for n, i in enumerate(idx):
        a = time.perf_counter()
        if mode == "prefetch" and n + 1 < len(idx):
            st.prefetch(hb[idx[n + 1]])
        b = time.perf_counter()
        ob.ingest_batch(st, hb[i])
        c = time.perf_counter()
        _ = st.model
        e = time.perf_counter()
        rec = st.log[-1]
        ts.append((b - a, c - b, e - c, rec.compress_seconds, rec.als_seconds, rec.recover_seconds))
    print(mode, ["%.1f/%.1f/%.1f c%.1f a%.1f r%.1f" % tuple(x * 1e3 for x in r) for r in ts], flush=True)
    idx = None
