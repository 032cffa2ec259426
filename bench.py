#!/usr/bin/env python
"""bench.py -- OCTen per-batch update throughput on B200.

One step = one ingest_batch (compress -> per-replica CP-ALS -> align/merge)
of a temporal batch on the BASELINE c3 workload: dense fp32 1000x1000 slices,
batches of 100 slices after an initial block of K0=1000, Q=100, P=16
replicas, rank R=20, shared=10, CP-ALS 30 sweeps x 3 restarts, rel_tol 1e-8
(SURVEY.md §8(d)).  Metric: tensor entries streamed per second per batch
update (I*J*t / step time).  Inputs are synthetic (rank-20 U(0,1) factors +
1% Gaussian noise, generated on the device) and each 400 MB batch exceeds the
126 MB L2, so no flush is needed.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 (torchrun): by default ONE stream sharded by replica over the ranks
(rank g compresses into and decomposes replicas [p0, p0+p_local), the merge
runs redundantly after NCCL all-gathers of the replica models and temporal
rows; strong scaling, value = batch entries / max-over-ranks step time).
--multi replicas runs N independent streams instead (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: I, J, K0, t, Q, P, R, shared, als_iters
    "c3": dict(I=1000, J=1000, K0=1000, t=100, Q=100, P=16, R=20, shared=10, iters=30, restarts=3),
    "c5": dict(I=2000, J=2000, K0=200, t=200, Q=128, P=32, R=32, shared=32, iters=30, restarts=3),
    "c2": dict(I=500, J=500, K0=500, t=50, Q=50, P=8, R=10, shared=12, iters=30, restarts=3),
    "small": dict(I=200, J=200, K0=100, t=20, Q=20, P=16, R=5, shared=5, iters=30, restarts=3),
}
# c4: sparse COO 1e5 x 1e5 x 2e4 (~1e8 nnz), batches of 1000 slices (~5e6 nnz),
# Zipf(1.2) rows/columns, uniform slices, U(0,1) values; compression + CP-ALS
# (the reference's merge throws NumericError at this shape)
C4 = dict(I=100000, J=100000, t=1000, Q=64, P=16, R=16, nnz=5_000_000, zipf=1.2, iters=30, restarts=3)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def pipe_peaks():
    """Measured arithmetic peaks of the pipes the path uses
    (scripts/micro/peaks.cu on this pool's B200, profiles/peaks_b200.json):
    tcgen05 kind::tf32 and kind::i8 (scripts/micro/i8_rate.cu), DMMA fp64,
    FFMA fp32."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_b200.json")) as f:
            d = json.load(f)
        return {"tf32": float(d["tcgen05_tf32_tflops"]), "dmma": float(d["dmma_f64_tflops"]),
                "ffma": float(d["ffma_f32_tflops"]), "i8": float(d.get("tcgen05_i8_tops", 4500.0)),
                "source": "measured (profiles/peaks_b200.json)"}
    except Exception:
        return {"tf32": 1100.0, "dmma": 37.0, "ffma": 72.0, "i8": 4500.0, "source": "nominal (peaks file missing)"}


def isolated_launch_ms():
    """Mean per-launch duration (ms) of the CP-ALS kernels in the committed
    ncu launch list of the c3 bench (profiles/r2s4_launches_c3.csv)."""
    out = {}
    try:
        import csv
        with open(os.path.join(ROOT, "profiles", "r2s4_launches_c3.csv")) as f:
            rows = [r for r in csv.reader(f)]
        h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[h]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        acc = {}
        for r in rows[h + 1:]:
            if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                continue
            for kname in ("oz_tgemm_kernel", "als_mttkrp_T_kernel"):
                if kname in r[ki]:
                    t, n = acc.get(kname, (0.0, 0))
                    acc[kname] = (t + float(r[vi].replace(",", "")) * 1e-6, n + 1)  # ns -> ms
        out = {k: t / n for k, (t, n) in acc.items() if n}
    except Exception:
        out = {}
    return out


def ref_backend():
    """The CPU implementation the reference arm and cpu_baseline time: the
    reference library compiled from its own sources (oracle/_ref, built by
    oracle/Makefile against the Eigen stand-in; kind "reference") when the
    snapshot carries it, else the oracle port (kind "port")."""
    try:
        from oracle import ref_lib
        if ref_lib.available():
            ref_lib.lib()
            return "reference"
    except Exception:  # pragma: no cover
        pass
    return "port"


def ref_workers(cfg):
    """min(cores, P) like the reference's resolve_workers (streaming.cpp:
    36-43), capped so the per-worker copies of the batch the reference's
    compress makes (compression.cpp:116, plus its matricize / product
    temporaries, ~3 batch sizes) fit the host's free memory."""
    I, J, t, P = (cfg[k] for k in ("I", "J", "t", "P"))
    w = min(os.cpu_count() or 1, P)
    try:
        import psutil
        avail = psutil.virtual_memory().available
        w = max(1, min(w, int(0.8 * avail // (3 * 8 * I * J * t))))
    except Exception:  # pragma: no cover
        pass
    return w


def cpu_baseline_step(cfg, noise):
    """cpu_baseline of the own arm: the reference (oracle/_ref, else the
    oracle port) timed on ONE full ingest_batch of a workload batch
    (compression of t slices into P replicas, CP-ALS on every replica, the
    whole merge) after an untimed init_stream on t slices (the per-batch work
    does not depend on K0 beyond the temporal factor's row count)."""
    from threadpoolctl import threadpool_limits
    from oracle import octen_oracle as O
    I, J, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "t", "Q", "P", "R", "shared"))
    kind = ref_backend()
    workers = ref_workers(cfg) if kind == "reference" else 0
    scfg = O.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * 1234 + 3,
                          als=O.AlsConfig(R, cfg["iters"], 1e-8, cfg["restarts"], 0), workers=workers)
    syn = HostSynth(I, J, 2 * t, R, 1234, noise)
    with threadpool_limits(limits=1):
        if kind == "reference":
            from oracle import ref_lib
            st = ref_lib.RefStream(syn.batch(0, t), scfg)
            b = syn.batch(t, t)
            a = time.perf_counter()
            st.ingest(b)
            sec = time.perf_counter() - a
            tm = st.timers()[-1]
            stages = {"compress_s": float(tm[0]), "als_s": float(tm[1]), "recover_s": float(tm[2]), "total_s": sec}
            what = ("the reference library compiled from its own sources (oracle/_ref: proj/src/*.cpp + the "
                    "Eigen stand-in on single-threaded OpenBLAS), %d replica workers" % workers)
        else:
            O.MERGE_PROCESSES = True
            st = O.init_stream(syn.batch(0, t), scfg)
            b = syn.batch(t, t)
            a = time.perf_counter()
            O.ingest_batch(st, b)
            sec = time.perf_counter() - a
            rec = st.log[-1]
            stages = {"compress_s": rec.compress_seconds, "als_s": rec.als_seconds,
                      "recover_s": rec.recover_seconds, "total_s": sec}
            workers = O.resolve_workers(scfg)
            what = ("the oracle port (compress + CP-ALS over %d replica threads, merge column solves over %d "
                    "processes, single-threaded BLAS)" % (workers, os.cpu_count()))
    return {"value": I * J * t / sec, "unit": "entries/s", "cores": workers, "kind": kind,
            "sample": "one full ingest_batch of a %dx%dx%d batch through %s, after an untimed init_stream on %d "
                      "slices" % (I, J, t, what, t),
            "stages_s": stages}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.n0 = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Start of the timed region: only samples from here on count (the
        sampler is started earlier, so nvidia-smi's own start-up -- process
        spawn, NVML init -- stays out of the timed region)."""
        self.n0 = len(self.lines)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[self.n0:]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# synthetic data (device)
# ---------------------------------------------------------------------------

class Synth:
    """Rank-R U(0,1) factors + N(0, sigma) noise with sigma = 1% of the clean
    RMS (BASELINE.json c3), generated on the device in fp64 and rounded to
    fp32; batches are Fortran-ordered (I, J, t) views of (t, J, I) storage."""

    def __init__(self, torch, dev, I, J, K, R, seed, noise=0.01):
        self.torch = torch
        self.dev = dev
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.g = g
        self.A = torch.rand((I, R), generator=g, device=dev, dtype=torch.float64)
        self.B = torch.rand((J, R), generator=g, device=dev, dtype=torch.float64)
        self.C = torch.rand((K, R), generator=g, device=dev, dtype=torch.float64)
        clean = torch.einsum("kr,jr,ir->kji", self.C[:10], self.B, self.A)
        self.sigma = noise * float(clean.pow(2).mean().sqrt())
        del clean

    def batch(self, k0, t, out=None):
        torch = self.torch
        if out is None:
            out = torch.empty((t, self.B.shape[0], self.A.shape[0]), device=self.dev, dtype=torch.float32)
        step = 50
        for s in range(0, t, step):
            e = min(t, s + step)
            x = torch.einsum("kr,jr,ir->kji", self.C[k0 + s:k0 + e], self.B, self.A)
            x += self.sigma * torch.randn(x.shape, generator=self.g, device=self.dev, dtype=torch.float64)
            out[s:e].copy_(x)
            del x
        return out.permute(2, 1, 0)


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on the host cores, staged sample
# ---------------------------------------------------------------------------

def cpu_sample(cfg, seed=7, slices=5, replicas=1, cols=2):
    """Time the oracle (numpy/LAPACK restatement of the reference) on a bounded
    sample of one c3 batch update and scale to the full batch:
      compress: `slices` of the t slices for `replicas` of the P replicas;
      CP-ALS:   `replicas` of the P replicas (full sweeps/restarts);
      merge:    align + the unweighted solve + `cols` of the R weighted
                column solves per non-temporal mode + the temporal append.
    Returns (seconds_per_batch_estimate, detail)."""
    from oracle import octen_oracle as O
    from oracle import rng as R_
    I, J, t, Q, P, R, sh = cfg["I"], cfg["J"], cfg["t"], cfg["Q"], cfg["P"], cfg["R"], cfg["shared"]
    g = np.random.default_rng(seed)
    rs = O.gen_replicas([I, J], Q, P, sh, seed)
    O.extend_temporal(rs, t)
    x = g.random((I, J, slices)).astype(np.float32).astype(np.float64)
    x = np.asfortranarray(x)
    # compression
    t0 = time.perf_counter()
    zs = [O.compress(x, rs, r, 0, slices) for r in range(replicas)]
    tc = (time.perf_counter() - t0) * (t / slices) * (P / replicas)
    # CP-ALS on a realistic summary (rank-R signal)
    del zs
    fa = [g.random((d, R)) for d in (I, J, t)]
    y = None
    for r in range(replicas):
        ct = [rs.replicas[r].nontemporal[0].T @ fa[0], rs.replicas[r].nontemporal[1].T @ fa[1],
              rs.replicas[r].temporal.T @ fa[2]]
        y = O.reconstruct_fast(O.KruskalModel(ct, np.ones(R)))
        y = y + 0.01 * np.sqrt(np.mean(y ** 2)) * g.standard_normal(y.shape)
    t0 = time.perf_counter()
    models = []
    for r in range(replicas):
        models.append(O.cp_als(y, O.AlsConfig(R, cfg["iters"], 1e-8, cfg["restarts"],
                                              R_.derive(seed, [8, r, 1]))).model)
    ta = (time.perf_counter() - t0) * (P / replicas)
    # merge
    proj = O.stack_projections(rs, 0)
    stack = proj @ fa[0] + 1e-3 * g.standard_normal((P * Q, R))
    t0 = time.perf_counter()
    O.recover_nontemporal(stack, proj, 0)
    t_solve1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    w = np.ones((P, R))
    w[0, :cols] = 0.7
    O.recover_nontemporal_weighted(stack[:, :cols], proj, 0, Q, w[:, :cols])
    t_wcol = (time.perf_counter() - t0) / cols
    summ = O.init_summaries(rs)
    t0 = time.perf_counter()
    O.recover_temporal_append(g.random((P * Q, R)), rs, summ, np.zeros((0, R)), t)
    t_app = time.perf_counter() - t0
    tm = 2 * (t_solve1 + 2 * R * t_wcol) + t_app
    total = tc + ta + tm
    detail = ("oracle port, 1 batch of %dx%dx%d estimated from: compress %d/%d slices x %d/%d replicas, "
              "CP-ALS %d/%d replicas, merge 1+%d/%d column solves per mode + temporal append"
              % (I, J, t, slices, t, replicas, P, replicas, P, cols, 2 * R))
    return total, {"compress_s": tc, "als_s": ta, "merge_s": tm}, detail


class HostSynth:
    """The c3/c5 workload on the host for the reference arm: the same recipe as
    Synth (rank-R U(0,1) factors, lambda = 1, N(0, sigma) noise with sigma =
    `noise` x the clean RMS of the first slices), generated with numpy, fp32
    rounded like the device arm's input and handed to the port as fp64."""

    def __init__(self, I, J, K, R, seed, noise):
        self.g = np.random.default_rng(seed)
        self.A = self.g.random((I, R))
        self.B = self.g.random((J, R))
        self.C = self.g.random((K, R))
        self.sigma = noise * float(np.sqrt(np.mean(self._clean(0, min(10, K)) ** 2)))

    def _clean(self, k0, t):
        # X_(0) = A KR(C, B)^T (tensor.cpp unfolding identity), then fold
        kr = (self.C[k0:k0 + t, None, :] * self.B[None, :, :]).reshape(t * self.B.shape[0], -1)
        x = self.A @ kr.T  # I x (J t), column j + J k
        return x.reshape((self.A.shape[0], self.B.shape[0], t), order="F")

    def batch(self, k0, t):
        x = self._clean(k0, t)
        x += self.sigma * self.g.standard_normal(x.shape)
        return np.asfortranarray(x.astype(np.float32).astype(np.float64))


def run_reference(args, cfg, rank, world):
    """The reference arm: the reference library compiled from its own sources
    (oracle/_ref: proj/src/*.cpp unmodified, Eigen replaced by the stand-in in
    oracle/ref_shim on single-threaded OpenBLAS; tests/test_ref_pin.py runs the
    reference's own unit tests on it) through its public API, full
    ingest_batch steps (streaming.cpp:262-348) on the same workload, its own
    std::thread fan-out over min(cores, P) replica workers
    (parallel_replicas, streaming.cpp:45-69).  Falls back to the oracle port
    (oracle/octen_oracle.py) when the snapshot has no oracle/_ref.  The
    untimed init_stream runs on t slices (the reference copies the batch per
    worker, compression.cpp:116; K0 = 1000 slices would need ~8 GB per
    worker); the timed per-batch work does not depend on K0 beyond the
    temporal factor's row count.  Rank 0 only; the step time is the mean of
    the timed ingest_batch calls, the reference's BatchRecord stage timers
    beside it."""
    if rank != 0:
        return
    from oracle import octen_oracle as O
    from threadpoolctl import threadpool_limits
    threadpool_limits(limits=1)
    kind = ref_backend()
    cores = os.cpu_count()
    I, J, K0, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
    nb = args.warmup + args.steps
    dseed = 1234
    workers = ref_workers(cfg) if kind == "reference" else 0
    scfg = O.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * dseed + 3,
                          als=O.AlsConfig(R, cfg["iters"], 1e-8, cfg["restarts"], 0), workers=workers)
    k_init = t if kind == "reference" else K0
    syn = HostSynth(I, J, k_init + nb * t, R, dseed, args.noise)
    times, stage_rows = [], []
    t0 = time.perf_counter()
    if kind == "reference":
        from oracle import ref_lib
        st = ref_lib.RefStream(syn.batch(0, k_init), scfg)
        t_init = time.perf_counter() - t0
        for i in range(nb):
            b = syn.batch(k_init + i * t, t)
            a = time.perf_counter()
            st.ingest(b)
            e = time.perf_counter() - a
            if i >= args.warmup:
                times.append(e)
                stage_rows.append(st.timers()[-1][:3])
        impl = ("the reference library compiled from its own sources (oracle/_ref: proj/src/*.cpp with the Eigen "
                "stand-in on single-threaded OpenBLAS)")
        # the reference model's fitness (eval.cpp:10-20) on its last batch,
        # beside the device arm's model_quality
        try:
            m = st.model()
            k_last = k_init + (nb - 1) * t
            A, B, Cm = m.factors
            xh = np.einsum("ir,jr,kr->ijk", A * m.lambda_, B, Cm[k_last:k_last + t], optimize=True)
            nx = float(np.linalg.norm(b))
            quality = {"batch_fitness_pct": 100.0 * (1.0 - float(np.linalg.norm(b - xh)) / nx),
                       "slices": [k_last, k_last + t],
                       "note": "fitness (eval.cpp:10-20) of the reference's model after its last batch on that batch"}
        except Exception as exc:  # pragma: no cover
            quality = {"error": repr(exc)}
    else:
        O.MERGE_PROCESSES = True
        st = O.init_stream(syn.batch(0, k_init), scfg)
        t_init = time.perf_counter() - t0
        for i in range(nb):
            b = syn.batch(k_init + i * t, t)
            a = time.perf_counter()
            O.ingest_batch(st, b)
            e = time.perf_counter() - a
            if i >= args.warmup:
                times.append(e)
                r = st.log[-1]
                stage_rows.append([r.compress_seconds, r.als_seconds, r.recover_seconds])
        workers = O.resolve_workers(scfg)
        impl = "the oracle port (numpy/LAPACK restatement of the reference; oracle/_ref was not built)"
        quality = None
    sec = float(np.mean(times))
    v = I * J * t / sec
    sr = np.asarray(stage_rows, dtype=float)
    stages = {"compress_s": float(sr[:, 0].mean()), "als_s": float(sr[:, 1].mean()),
              "recover_s": float(sr[:, 2].mean()), "init_s": t_init}
    sample = ("full ingest_batch steps of %s on the %s workload: %d timed + %d warm-up batches of %dx%dx%d after "
              "an untimed init_stream on %d slices; %d replica workers" %
              (impl, args.config, args.steps, args.warmup, I, J, t, k_init, workers))
    line = {"metric": "tensor entries streamed/sec per batch update", "value": v, "unit": "entries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(args, cfg, int(os.environ.get("WORLD_SIZE", "1"))),
            "stages_s": stages, "step_s": [round(x, 3) for x in times], "model_quality": quality,
            "cpu_baseline": {"value": v, "unit": "entries/s", "cores": workers, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_config(args, cfg, world):
    """The `config` of a bench line (both arms print the same one)."""
    I, J, t = cfg["I"], cfg["J"], cfg["t"]
    sharded = world > 1 and args.multi in ("sharded", "temporal")
    temporal = world > 1 and args.multi == "temporal"
    par = (("temporal-sharded compression x%d (NCCL reduce-scatter of partial summaries) + replica-sharded "
            "CP-ALS (NCCL all-gather)" % world) if temporal else
           ("replica-sharded x%d (NCCL all-gather of replica models)" % world if sharded else
            ("independent streams x%d" % world if world > 1 else "single")))
    return {"workload": args.config, **cfg, "noise": args.noise,
            "l2": "inputs larger than L2 (%d MB fp32 batch)" % (I * J * t * 4 // 10**6), "parallelism": par}


# ---------------------------------------------------------------------------
# c4: sparse COO batches
# ---------------------------------------------------------------------------

class CooSynth:
    """c4 batches generated on the device: i, j ~ truncated Zipf(1.2) on the
    extents (inverse CDF), k uniform in the batch, values U(0,1); duplicate
    (i, j, k) are dropped (the reference rejects them, tensor.cpp:99-100) and
    the survivors shuffled into arbitrary input order."""

    def __init__(self, torch, dev, c, seed):
        self.torch, self.dev, self.c = torch, dev, c
        self.g = torch.Generator(device=dev)
        self.g.manual_seed(seed)
        w = torch.arange(1, c["I"] + 1, device=dev, dtype=torch.float64).pow(-c["zipf"])
        self.cdf = torch.cumsum(w, 0) / w.sum()

    def batch(self):
        torch, c, g = self.torch, self.c, self.g
        n = int(c["nnz"] * 1.7)  # Zipf(1.2) pairs collide: ~1/3 of the draws are duplicates
        I, J, t = c["I"], c["J"], c["t"]
        i = torch.searchsorted(self.cdf, torch.rand(n, generator=g, device=self.dev, dtype=torch.float64))
        j = torch.searchsorted(self.cdf, torch.rand(n, generator=g, device=self.dev, dtype=torch.float64))
        i.clamp_(max=I - 1)
        j.clamp_(max=J - 1)
        k = torch.randint(0, t, (n,), generator=g, device=self.dev)
        key = torch.unique((k * I + i) * J + j)
        key = key[torch.randperm(key.numel(), generator=g, device=self.dev)][: c["nnz"]]
        jj = (key % J).to(torch.int32)
        ii = ((key // J) % I).to(torch.int32)
        kk = (key // (I * J)).to(torch.int32)
        v = torch.rand(key.numel(), generator=g, device=self.dev, dtype=torch.float32)
        return ii.contiguous(), jj.contiguous(), kk.contiguous(), v


def run_sparse(args, torch, dev, ob, steps, warmup, with_cpu):
    """c4 step = compress one ~5e6-nnz COO batch into the P=16 summaries +
    CP-ALS on every replica.  Each call of the C-ABI is synchronous (the
    batch is validated before the summaries change), so a step is timed by
    the host clock between device synchronizations; the L2 is flushed
    between steps outside the timed region."""
    c = C4
    I, J, t, Q, P, R = (c[k] for k in ("I", "J", "t", "Q", "P", "R"))
    r = np.random.default_rng(11)
    u = [r.random((I, Q)) for _ in range(P)]
    v = [r.random((J, Q)) for _ in range(P)]
    t0 = time.perf_counter()
    hs = ob.CooSummaries(u, v, device=dev.index or 0)
    t_setup = time.perf_counter() - t0
    syn = CooSynth(torch, dev, c, 99)
    nb = warmup + steps
    batches = [syn.batch() for _ in range(nb)]
    ws = [torch.rand((P, Q, t), generator=syn.g, device=dev, dtype=torch.float64) for _ in range(nb)]
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    cfg = ob.AlsConfig(max_iters=c["iters"], rel_tol=1e-8, n_restarts=c["restarts"])
    cfg.rank = R
    seeds = list(range(100, 100 + P))
    torch.cuda.synchronize()
    tot = tc = 0.0
    nnz_timed = 0
    launches = 0
    st0 = None
    for s in range(nb):
        ii, jj, kk, vv = batches[s]
        flush.fill_(float(s))
        torch.cuda.synchronize()
        if s == warmup:
            st0 = hs.stage_times()
            l0 = ob._capi.LIB.octen_launch_count()
        a = time.perf_counter()
        hs.compress_device(t, ws[s], ii, jj, kk, vv)
        b = time.perf_counter()
        hs.cp_als(cfg, seeds, fetch=False)
        e = time.perf_counter()
        if s >= warmup:
            tot += e - a
            tc += b - a
            nnz_timed += vv.numel()
    launches = ob._capi.LIB.octen_launch_count() - l0
    st1 = hs.stage_times()
    d = {k: st1[k] - st0[k] for k in st1}
    nb_t = max(d["batches"], 1)
    nnz_step = nnz_timed / steps
    groups = d["groups"] / nb_t
    slice_ms = d["slice_ms"] / nb_t
    flops = 2.0 * P * (nnz_step * Q + groups * Q * Q)  # useful flops of the slice kernel per launch
    pk = pipe_peaks()
    fp32_peak = pk["ffma"]
    out = {"metric": "nnz streamed/sec per batch update", "value": nnz_timed / tot, "unit": "nnz/s",
           "ms_per_step": tot * 1e3 / steps, "steps": steps, "warmup": warmup,
           "compress_nnz_per_s": nnz_timed / tc,
           "config": {"workload": "c4", **c, "nnz_per_batch": nnz_step, "groups_per_batch": groups,
                      "l2": "flushed between steps (256 MB write)", "projections": "U(0,1) fp64, fp32 on device"},
           "stages_ms": {"validate_sort": d["prep_ms"] / nb_t, "slice_kernel": slice_ms,
                         "mode3_accumulate": d["accum_ms"] / nb_t, "cp_als": d["als_ms"] / max(d["als_runs"], 1),
                         "compress_host_clock": tc * 1e3 / steps},
           "roofline": {"kernel": "coo_slice_kernel (gather-accumulate + per-(k,i) rank-1 updates)",
                        "bound": "fp32 FFMA", "achieved": flops / (slice_ms * 1e-3) / 1e12 if slice_ms else 0.0,
                        "peak": fp32_peak, "unit": "TFLOP/s",
                        "frac": flops / (slice_ms * 1e-3) / 1e12 / fp32_peak if slice_ms else 0.0,
                        "peak_source": "FP32 FFMA, %s" % pk["source"],
                        "flops_per_launch": flops, "traffic": c4_traffic(),
                        "traffic_unit": "bytes/launch (ncu dram__bytes_read+write, profiles/r1_c4_roofline.json)"},
           "gpu_launches": int(launches), "setup_s": t_setup}
    # e2e: host COO arrays + host temporal rows through the public API, model read back
    if args.e2e_steps > 0:
        hb = []
        for s in range(args.e2e_steps + 1):
            ii, jj, kk, vv = syn.batch()
            # pinned host arrays (the COO entries as a loader would hand them over)
            pin = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True).copy_(x) for x in (ii, jj, kk, vv)]
            sp = ob.SparseTensor.from_arrays((I, J, t), *[x.numpy() for x in pin])
            sp._keep = pin
            hb.append((sp, [r.random((t, Q)) for _ in range(P)]))
        hs.compress(*hb[0])
        hs.cp_als(cfg, seeds)
        torch.cuda.synchronize()
        a = time.perf_counter()
        nn = 0
        for sp, w in hb[1:]:
            hs.compress(sp, w)
            hs.cp_als(cfg, seeds)
            nn += sp.nnz
        e2e_s = time.perf_counter() - a
        out["e2e"] = {"value": nn / e2e_s, "unit": "nnz/s",
                      "h2d_bytes_per_step": int(nn / args.e2e_steps * 16 + P * t * Q * 8),
                      "d2h_bytes_per_step": P * (3 * Q * R + R) * 8}
    if with_cpu:
        out["cpu_baseline"] = cpu_sample_sparse(batches[0], ws[0], u, v, P, R, c)
    return out


def c4_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "r1_c4_roofline.json")) as f:
            return json.load(f)["traffic_bytes_per_launch"]
    except Exception:
        return None


def cpu_sample_sparse(batch, w, u, v, P, R, c, sample=50_000):
    """Oracle port on the host: the entry-wise compress (compress_coo_direct,
    = compress(to_dense(batch))) of `sample` entries for one replica, scaled
    to the batch's nnz and P replicas, + CP-ALS (cp_als.cpp) on one Q^3
    replica summary scaled by P."""
    from oracle import octen_oracle as O
    ii, jj, kk, vv = (x.cpu().numpy() for x in batch)
    wh = w[0].cpu().numpy().T  # t x Q
    n = min(sample, ii.size)
    a = time.perf_counter()
    z = O.compress_coo_direct(ii[:n], jj[:n], kk[:n], vv[:n].astype(np.float64), u[0], v[0], wh)
    tcomp = (time.perf_counter() - a) * (ii.size / n) * P
    a = time.perf_counter()
    O.cp_als(z, O.AlsConfig(R, c["iters"], 1e-8, c["restarts"], 5))
    tals = (time.perf_counter() - a) * P
    sec = tcomp + tals
    return {"value": ii.size / sec, "unit": "nnz/s", "cores": os.cpu_count(), "kind": "port",
            "sample": "oracle port: entry-wise compress of %d of %d nnz for 1 of %d replicas + CP-ALS on 1 replica, "
                      "scaled" % (n, ii.size, P),
            "stages_s": {"compress_s": tcomp, "als_s": tals}}


# ---------------------------------------------------------------------------
# own arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="octen", choices=["octen", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS) + ["c4"])
    ap.add_argument("--noise", type=float, default=0.01, help="Gaussian noise sigma relative to the clean RMS")
    ap.add_argument("--als-iters", type=int, default=0, help="override the config's CP-ALS max_iters")
    ap.add_argument("--no-sparse", action="store_true", help="skip the c4 sparse leg of the default line")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--collectives", default="library", choices=["library", "torch"],
                    help="N>1 sharded modes: the library's own NCCL communicator (default) or the caller's "
                         "torch.distributed collectives between the library's phases")
    ap.add_argument("--multi", default="sharded", choices=["sharded", "temporal", "replicas"],
                    help="N>1: one replica-sharded stream over all ranks (NCCL all-gathers, strong scaling); "
                         "'temporal': the same with the compression sharded over the batch's slices "
                         "(NCCL reduce-scatter of the partial summaries); or N independent streams (weak scaling)")
    args = ap.parse_args()
    cfg = dict(CONFIGS.get(args.config, C4))
    if args.als_iters > 0:
        cfg["iters"] = args.als_iters
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    import paper_1807_01350_b200 as ob
    if args.config == "c4":
        sp = run_sparse(args, torch, dev, ob, args.steps, args.warmup,
                        rank == 0 and world == 1 and not args.no_cpu_baseline)
        if rank == 0:
            sp.update({"n_gpus": world, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                       "dtype": "f32 slice products + f64 mode-3 accumulate / CP-ALS", "data": "synthetic"})
            print(json.dumps(sp), flush=True)
        return
    I, J, K0, t, Q, P, R, sh = (cfg[k] for k in ("I", "J", "K0", "t", "Q", "P", "R", "shared"))
    nb = args.warmup + args.steps + args.e2e_steps + 2
    sharded = world > 1 and args.multi in ("sharded", "temporal")
    temporal = world > 1 and args.multi == "temporal"
    # sharded: every rank sees the same batches and seeds (one stream);
    # replicas: independent streams with per-rank data
    dseed = 1234 if sharded else 1234 + rank
    syn = Synth(torch, dev, I, J, K0 + nb * t, R, seed=dseed, noise=args.noise)
    first = syn.batch(0, K0)
    scfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=7 * dseed + 3,
                           als=ob.AlsConfig(max_iters=cfg["iters"], rel_tol=1e-8, n_restarts=cfg["restarts"]),
                           device=local)
    torch.cuda.synchronize()
    t_init = time.perf_counter()
    if sharded and args.collectives == "library":
        # the library's own NCCL communicator (octen_stream_create_nccl): rank
        # 0's unique id travels over the torch process group once
        uid = torch.tensor(list(ob.nccl_unique_id() if rank == 0 else bytes(128)), dtype=torch.uint8, device=dev)
        dist.broadcast(uid, 0)
        st = ob.NcclStream(scfg, rank, world, uid=bytes(uid.cpu().tolist()))
        if temporal:
            def ingest(b):
                tb = b.shape[2]
                lo, hi = tb * rank // world, tb * (rank + 1) // world
                st.ingest_temporal(b[:, :, lo:hi], lo, tb)
        else:
            ingest = st.ingest
        ingest(first)
    elif sharded:
        st = ob.ShardedStream(scfg, rank, world, lambda snd, rcv: dist.all_gather_into_tensor(rcv, snd))
        if temporal:
            def ingest(b):
                tb = b.shape[2]
                lo, hi = tb * rank // world, tb * (rank + 1) // world
                st.ingest_temporal(b[:, :, lo:hi], lo, tb,
                                   lambda snd, rcv: dist.reduce_scatter_tensor(rcv, snd, op=dist.ReduceOp.SUM))
            ingest(first)
        else:
            st.ingest(first)
            ingest = st.ingest
    else:
        st = ob.init_stream(first, scfg)
        # pipelined ingest: batch b's merge overlaps batch b+1's compression
        # and CP-ALS (same bits as ingest_batch; st.sync() drains it)
        ingest = st.ingest_async
        if os.environ.get("OCTEN_BENCH_SYNC"):  # diagnostics: the stages one after another
            ingest = lambda b: ob.ingest_batch(st, b)
    pipelined = not sharded and not os.environ.get("OCTEN_BENCH_SYNC")
    t_init = time.perf_counter() - t_init
    del first
    batches = [syn.batch(K0 + i * t, t) for i in range(args.warmup + args.steps)]
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    for i in range(args.warmup):
        ingest(batches[i])
    if pipelined:
        st.sync()
    times0 = (ctypes_stage_times(ob, st))
    ks0 = st.kernel_stats() if hasattr(st, "kernel_stats") else None
    l0 = ob._capi.LIB.octen_launch_count()
    clk.mark()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        ingest(batches[args.warmup + i])
    if pipelined:
        st.sync()  # the last batch's merge is inside the timed region
    e1.record()
    barrier()
    clocks = clk.stop()
    # model quality (outside the timed region): eval.cpp fitness of the
    # streamed model on the last timed batch, computed on the device
    quality = None
    try:
        kl = K0 + (args.warmup + args.steps - 1) * t
        quality = {"batch_fitness_pct": st.batch_fitness(batches[args.warmup + args.steps - 1], kl),
                   "slices": [kl, kl + t],
                   "note": "fitness (eval.cpp:10-20) of the model after the last timed batch on that batch; "
                           "rank-%d U(0,1) truth + %.2g%% noise" % (R, 100 * args.noise)}
    except Exception as exc:  # pragma: no cover
        quality = {"error": repr(exc)}
    if os.environ.get("OCTEN_BENCH_STEPLOG") and not sharded:
        for rec in st.log[-args.steps:]:
            print("step %d: compress %.2f als %.2f recover %.2f total %.2f ms" % (
                rec.batch_index, rec.compress_seconds * 1e3, rec.als_seconds * 1e3, rec.recover_seconds * 1e3,
                rec.total_seconds * 1e3), file=sys.stderr)
    ms = e0.elapsed_time(e1) / args.steps
    launches = ob._capi.LIB.octen_launch_count() - l0
    times1 = ctypes_stage_times(ob, st)
    ks1 = st.kernel_stats() if hasattr(st, "kernel_stats") else None  # the timed steps only
    dt = [b - a for a, b in zip(times0, times1)]
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    entries = I * J * t
    jobs = 1 if sharded else world  # batches the whole job processes per step
    value = jobs * entries / (ms * 1e-3)

    # e2e through the C-ABI with pinned host buffers (H2D inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        hb = []
        # pinned host batches: at most ~8 GB of them
        e2e_steps = max(2, min(args.e2e_steps, int(8e9 // (entries * 4)) - 2))
        for i in range(e2e_steps + 2):  # +2: untimed warm-up of the host-input path
            d = syn.batch(K0 + (args.warmup + args.steps + i) * t, t)
            h = torch.empty((t, J, I), dtype=torch.float32, pin_memory=True)
            h.copy_(d.permute(2, 1, 0))
            hb.append(h.permute(2, 1, 0))
        torch.cuda.synchronize()
        use_pf = not temporal  # a temporal shard reads only its slices: no whole-batch prefetch
        if use_pf:
            st.prefetch(hb[0])  # warm-up: copy streams, both prefetch slots, staging buffers
            st.prefetch(hb[1])
        if pipelined:
            st.set_publish(True)
        ingest(hb[0])
        ingest(hb[1])
        if pipelined:
            st.sync()
        _ = st.model
        if pipelined:
            _ = st.last_model()
        hb = hb[2:]
        barrier()
        tw = time.perf_counter()
        d2h = 0
        # the next batch's H2D copy is started (prefetch) before the current
        # batch is ingested, so it overlaps this batch's device work; every
        # step's copy is inside the timed region
        if use_pf:
            st.prefetch(hb[0])
        e2e_marks = []
        for i, h in enumerate(hb):
            if use_pf and i + 1 < len(hb):
                st.prefetch(hb[i + 1])
            ingest(h)
            if pipelined:
                # the step's result: the model of the batch whose merge just
                # completed (D2H by the library when that merge finished)
                m, _ = st.last_model()
            else:
                m = st.model  # D2H of the updated model (factors + lambda)
            d2h = sum(f.nbytes for f in m.factors) + m.lambda_.nbytes
            e2e_marks.append(time.perf_counter())
        if pipelined:
            st.sync()
            m = st.model  # the last batch's model
        barrier()
        e2e_s = (time.perf_counter() - tw) / e2e_steps
        if world > 1:
            tt = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e = {"value": jobs * entries / e2e_s, "unit": "entries/s", "h2d_bytes_per_step": entries * 4,
               "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "overlap": ("batch i+1 H2D (pinned, StreamState.prefetch) overlaps batch i's device work" +
                           ("; batch i's merge overlaps batch i+1's compression + CP-ALS (ingest_async), the "
                            "model of batch i is read back at step i+1 and the last one after the loop"
                            if pipelined else "")),
               "step_ms": [round((b - a) * 1e3, 2) for a, b in zip([tw] + e2e_marks[:-1], e2e_marks)]}

    hbm, bf16, peak_kind = peaks()
    pk = pipe_peaks()
    tf32_peak = pk["tf32"]
    g1_ms = dt[3] / max(dt[5], 1)  # per launch
    g1_flops = dt[4] / max(dt[5], 1)
    achieved = g1_flops / (g1_ms * 1e-3) / 1e12 if g1_ms > 0 else 0.0
    traffic = None
    pipe_pct = None
    try:  # dram read+write bytes per GEMM1 launch from the committed ncu --set full capture (c3)
        with open(os.path.join(ROOT, "profiles", "r1_roofline.json")) as f:
            rj = json.load(f)
        if args.config == "c3":
            traffic = rj["traffic_bytes_per_launch"]
            pipe_pct = rj.get("tensor_pipe_active_pct")
    except Exception:
        traffic = None
    n_mma = 3.0 if os.environ.get("OCTEN_G1_3MMA") else 2.0  # the library's GEMM1 split (tc_gemm.cu)
    kd = {k: ks1[k] - ks0[k] for k in ks1} if (ks1 and ks0) else None
    rooflines = {
        "gemm1": {"kernel": "tc_gemm_tf32x3_persistent_kernel (compression mode-1 contraction, GEMM1)",
                  "bound": "tensor (tcgen05 kind::tf32)", "achieved": achieved, "peak": tf32_peak,
                  "unit": "TFLOP/s", "frac": achieved / tf32_peak, "traffic": traffic,
                  "traffic_unit": "bytes/launch (ncu dram__bytes_read+write, profiles/r1_roofline.json)",
                  "peak_source": pk["source"], "flops_per_launch": g1_flops, "ms_per_launch": g1_ms,
                  "issued_tflops": n_mma * achieved, "issued_frac": n_mma * achieved / tf32_peak,
                  "issued_note": ("split-TF32: 2 tcgen05 MMAs per useful product (A_hi X_rn + A_lo X_rn, X rounded "
                                  "to the nearest TF32)" if n_mma == 2 else
                                  "split-TF32: 3 tcgen05 MMAs (hi*hi, hi*lo, lo*hi) per useful product"),
                  "tensor_pipe_active_pct_ncu": pipe_pct}}
    if pipelined:  # GEMM1 runs on half the SMs beside the previous batch's sweeps
        nsm = torch.cuda.get_device_properties(local).multi_processor_count
        g1_env = os.environ.get("OCTEN_G1_SMS")
        g1_ctas = int(g1_env) if g1_env is not None else nsm // 2
        if 0 < g1_ctas < nsm:
            rooflines["gemm1"].update({
                "ctas": g1_ctas, "sms": nsm,
                "frac_of_grid_sms": achieved / (tf32_peak * g1_ctas / nsm),
                "grid_note": "the pipelined ingest caps GEMM1's persistent grid at %d of %d SMs so the previous "
                             "batch's CP-ALS sweeps keep the rest (11.43 -> 11.17 ms per step); frac_of_grid_sms "
                             "is the fraction of the peak those SMs give" % (g1_ctas, nsm)})
    if kd and kd["gemm_launches"] > 0:
        gms = kd["gemm_ms"] / kd["gemm_launches"]
        gfl = kd["gemm_flops"] / kd["gemm_launches"]
        live_note = ("duration from CUDA events on the launching lane stream (sampled: lane 0, every fifth sweep) "
                     "while the other lanes, the next batch's compression and the pipelined merge share the GPU")
        if os.environ.get("OCTEN_ALS_TGEMM") == "dmma" or Q > 128:
            rooflines["als_tgemm"] = {
                "kernel": "gemm_dmma_pipe_kernel (CP-ALS partial contractions T = Y x_n F, all restarts of a lane's "
                          "replicas)", "bound": "FP64 tensor (DMMA)", "achieved": gfl / (gms * 1e-3) / 1e12,
                "peak": pk["dmma"], "unit": "TFLOP/s", "frac": gfl / (gms * 1e-3) / 1e12 / pk["dmma"],
                "flops_per_launch": gfl, "ms_per_launch": gms, "sampled_launches": kd["gemm_launches"],
                "peak_source": pk["source"], "note": live_note}
        else:
            # issued int8 tensor work of one lane launch (csrc/ozaki.cu): per
            # 128-row tile and 64-column group, 34 slice pairs (i + j <= 9, i, j
            # <= 7) x 64 columns x 128 rows x 32 ceil(Q / 32) K bytes
            lane_p = P / 4.0
            tiles = lane_p * -(-Q * Q // 128) * -(-(cfg["restarts"] * R) // 64)
            iops = 2.0 * 34 * 64 * 128 * 32 * -(-Q // 32) * tiles
            rooflines["als_tgemm"] = {
                "kernel": "oz_tgemm_kernel (CP-ALS partial contractions T = Y x_n F in fp64 on the int8 tensor cores "
                          "by exact digit splitting, all restarts of a lane's replicas; csrc/ozaki.cu)",
                "bound": "tensor (tcgen05 kind::i8)", "achieved": iops / (gms * 1e-3) / 1e12, "peak": pk["i8"],
                "unit": "TOP/s", "frac": iops / (gms * 1e-3) / 1e12 / pk["i8"], "issued_ops_per_launch": iops,
                "fp64_flops_per_launch": gfl, "fp64_equiv_tflops": gfl / (gms * 1e-3) / 1e12,
                "fp64_equiv_frac_of_dmma_peak": gfl / (gms * 1e-3) / 1e12 / pk["dmma"],
                "ms_per_launch": gms, "sampled_launches": kd["gemm_launches"], "peak_source": pk["source"],
                "note": live_note}
    if kd and kd["mttkrp_launches"] > 0:
        mms = kd["mttkrp_ms"] / kd["mttkrp_launches"]
        mby = kd["mttkrp_bytes"] / kd["mttkrp_launches"]
        rooflines["als_mttkrp"] = {
            "kernel": "als_mttkrp_T_kernel (contraction of T with a factor + the fused mode update)",
            "bound": "hbm", "achieved": mby / (mms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": mby / (mms * 1e-3) / 1e9 / hbm, "bytes_per_launch": mby, "ms_per_launch": mms,
            "sampled_launches": kd["mttkrp_launches"], "peak_source": "%s HBM copy" % peak_kind,
            "note": "the launch includes the serial R x R update of the last column block per problem"}
    if kd and kd["sweeps"] > 0:
        # every sweep: 1.5 T-GEMMs of 2 Q^3 S R flops per replica
        als_flops = kd["sweeps"] / args.steps * 1.5 * 2.0 * Q ** 3 * cfg["restarts"] * R * P
        rooflines["als_stage"] = {"bound": "FP64 (fp64 T-GEMM flops vs the DMMA peak)",
                                  "achieved": als_flops / (dt[1] / args.steps * 1e-3) / 1e12,
                                  "peak": pk["dmma"], "unit": "TFLOP/s",
                                  "frac": als_flops / (dt[1] / args.steps * 1e-3) / 1e12 / pk["dmma"],
                                  "flops_per_step": als_flops, "sweeps_per_step": kd["sweeps"] / args.steps,
                                  "note": "T-GEMM flops (1.5 per sweep, 2 Q^3 S R each, per replica) over the "
                                          "device-timed CP-ALS stage"}
    # merge: Gram-formulation flops of one batch (2 passes x 2 modes x R
    # bordered Cholesky factorizations of order d+1 + the weighted Grams)
    d = I
    merge_flops = 2 * 2 * (R * (d + 1) ** 3 / 3.0 + 2.0 * R * P * d * d)
    mms_step = dt[2] / args.steps
    rooflines["merge_stage"] = {"bound": "FP64 tensor (DMMA)", "achieved": merge_flops / (mms_step * 1e-3) / 1e12,
                                "peak": pk["dmma"], "unit": "TFLOP/s",
                                "frac": merge_flops / (mms_step * 1e-3) / 1e12 / pk["dmma"],
                                "flops_per_step": merge_flops,
                                "note": "runs on the merge stream concurrently with the next batch's compression "
                                        "and CP-ALS (pipelined ingest); its time includes that sharing"}
    # the headline roofline: the kernel with the largest device-time share
    shares = {"gemm1": dt[3]}
    if kd:
        shares["als_tgemm"] = kd["gemm_ms"]
        shares["als_mttkrp"] = kd["mttkrp_ms"]
    if kd:  # sampled kernel timing -> per-step totals
        nl = float(kd["sweeps"]) / args.steps  # sweeps per step (all lanes run them)
        shares["als_tgemm"] = rooflines.get("als_tgemm", {}).get("ms_per_launch", 0.0) * 1.5 * nl * 4 * args.steps
        shares["als_mttkrp"] = rooflines.get("als_mttkrp", {}).get("ms_per_launch", 0.0) * 3 * nl * 4 * args.steps
    top = max(shares, key=shares.get)
    # the same kernels alone: per-launch durations of the committed ncu
    # launch list (cold caches, serialised launches; profiles/), for reading
    # the live figures, which include the sharing of the GPU
    iso = isolated_launch_ms() if args.config == "c3" else {}
    for k, kname in (("als_tgemm", "oz_tgemm_kernel"), ("als_mttkrp", "als_mttkrp_T_kernel")):
        if k in rooflines and kname in iso and iso[kname] > 0:
            r = rooflines[k]
            live = r["ms_per_launch"]
            r["isolated"] = {"ms_per_launch": iso[kname], "achieved": r["achieved"] * live / iso[kname],
                             "frac": r["frac"] * live / iso[kname],
                             "source": "ncu launch list profiles/r2s4_launches_c3.csv (gpu__time_duration, "
                                       "serialised, cold caches)"}
            if "fp64_equiv_tflops" in r:
                r["isolated"]["fp64_equiv_frac_of_dmma_peak"] = r["fp64_equiv_frac_of_dmma_peak"] * live / iso[kname]
    roofline = dict(rooflines[top])
    roofline["why"] = "largest summed device time of the step's kernels (%s)" % ", ".join(
        "%s %.2f ms" % (k, v / args.steps) for k, v in shares.items())
    stage = {"compress_ms": dt[0] / args.steps, "als_ms": dt[1] / args.steps, "merge_ms": dt[2] / args.steps,
             "gemm1_ms": dt[3] / args.steps, "init_s": t_init}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_step(cfg, args.noise)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "entries/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": "failed: %r" % (exc,)}

    sparse = None
    if rank == 0 and world == 1 and not args.no_sparse and args.config == "c3":
        del batches
        try:
            sparse = run_sparse(args, torch, dev, ob, 3, 3, not args.no_cpu_baseline)
        except Exception as exc:  # pragma: no cover
            sparse = {"error": repr(exc)}

    if rank == 0:
        line = {"metric": "tensor entries streamed/sec per batch update", "value": value, "unit": "entries/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
                "dtype": "f32 compress (split-TF32/FP32) + f64 CP-ALS/merge", "data": "synthetic",
                "config": bench_config(args, cfg, world),
                "stages": stage, "roofline": roofline, "rooflines": rooflines, "cpu_baseline": cpu, "e2e": e2e,
                "model_quality": quality,
                "gpu_launches": int(launches), "clocks": clocks}
        if sparse is not None:
            line["sparse_c4"] = sparse
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def ctypes_stage_times(ob, st):
    import ctypes
    out = (ctypes.c_double * 6)()
    ob._check(ob._capi.LIB.octen_stream_get_stage_times(st._h, out))
    return list(out)


if __name__ == "__main__":
    main()
