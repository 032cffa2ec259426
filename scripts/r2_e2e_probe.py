"""Where does the e2e step lose time against the device-resident step?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1807_01350_b200 as ob
import atexit

dev = torch.device("cuda", 0)
c = bench.CONFIGS["c3"]
I, J, K0, t, Q, P, R, sh = (c[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
syn = bench.Synth(torch, dev, I, J, K0 + 40 * t, R, seed=1234)
cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * 1234 + 3,
                      als=ob.AlsConfig(max_iters=30, rel_tol=1e-8, n_restarts=3))
st = ob.init_stream(syn.batch(0, K0), cfg)
dbat = [syn.batch(K0 + i * t, t) for i in range(8)]
hb = []
for i in range(8):
    h = torch.empty((t, J, I), dtype=torch.float32, pin_memory=True)
    h.copy_(dbat[i].permute(2, 1, 0))
    hb.append(h.permute(2, 1, 0))
torch.cuda.synchronize()

def stimes():
    return bench.ctypes_stage_times(ob, st)


def run(name, fn, n=6):
    st.sync(); torch.cuda.synchronize()
    s0 = stimes()
    a = time.perf_counter()
    marks = []
    for i in range(n):
        fn(i)
        marks.append(time.perf_counter())
    st.sync(); torch.cuda.synchronize()
    e = time.perf_counter()
    s1 = stimes()
    d = [(y - x) / n for x, y in zip(s0, s1)]
    recs = st.log[-n:]
    print("%-40s %.2f ms/step  marks %s  dev compress/als/merge %.2f/%.2f/%.2f  host c/a/r %s" % (
        name, (e - a) * 1e3 / n, [round((b - x) * 1e3, 1) for x, b in zip([a] + marks[:-1], marks)],
        d[0], d[1], d[2], [(round(r.compress_seconds * 1e3, 1), round(r.als_seconds * 1e3, 1),
                              round(r.recover_seconds * 1e3, 1)) for r in recs[:3]]), flush=True)

run("device async", lambda i: st.ingest_async(dbat[i]))
run("device sync", lambda i: ob.ingest_batch(st, dbat[i]))
run("host async no prefetch", lambda i: st.ingest_async(hb[i]))
def pf(i):
    if i == 0:
        st.prefetch(hb[0])
    if i + 1 < 6:
        st.prefetch(hb[i + 1])
    st.ingest_async(hb[i])
run("host async + prefetch", pf)
st.set_publish(True)
def pf2(i):
    pf(i)
    st.last_model()
run("host async + prefetch + last_model", pf2)
if os.environ.get("PROBE_NOPULL"):
    pass
