"""CUPTI kernel timeline (torch.profiler, process-wide) of a few pipelined c3
ingest steps: per-stream kernel lists + gaps, for finding host-sync bubbles.
Writes gpurun_out/r2_trace.json (compact: name, stream, start, dur)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_1807_01350_b200 as ob

cfg = bench.CONFIGS["c3"]
I, J, K0, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
dev = torch.device("cuda:0")
nb = 6
syn = bench.Synth(torch, dev, I, J, K0 + nb * t, R, seed=1234, noise=0.01)
scfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * 1234 + 3,
                       als=ob.AlsConfig(rank=R, max_iters=cfg["iters"], rel_tol=1e-8, n_restarts=cfg["restarts"]))
st = ob.init_stream(syn.batch(0, K0), scfg)
bs = [syn.batch(K0 + i * t, t) for i in range(nb)]
torch.cuda.synchronize()
for i in range(3):
    st.ingest_async(bs[i])
st.sync()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(3, nb):
        st.ingest_async(bs[i])
    st.sync()
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace.json")
d = json.load(open("/tmp/trace.json"))
ev = [e for e in d["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset",
                                                                             "cuda_runtime", "cuda_driver")]
out = [{"n": e["name"][:60], "c": e["cat"], "s": e.get("args", {}).get("stream", e.get("tid")), "t": e["ts"],
        "d": e.get("dur", 0)} for e in ev]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "r2_trace.json"), "w"))
print("events", len(out))
