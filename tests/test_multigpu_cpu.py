"""Host logic of the replica-sharded multi-GPU path on CPU: two gloo ranks
(world_size 2, 127.0.0.1) run the sharded protocol of include/octen_b200.h
(begin -> all-gather models -> merge -> all-gather rows -> finish) with the
oracle standing in for the device stages, packing the exchanged blocks with
paper_1807_01350_b200.sharding (the device layout).  Both ranks must end
bit-identical to each other and equal to the unsharded oracle stream."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import octen_oracle as O
from oracle import rng
from paper_1807_01350_b200 import sharding as S

P, Q, R, SH, SEED = 6, 12, 3, 3, 38
ITERS, TOL, RESTARTS = 20, 1e-8, 2
K0, T, NB = 30, 8, 2


def _data():
    x, _ = O.generate_synthetic([40, 36, K0 + NB * T], R, 3, 0.0, 0.0)
    return x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape,
                                                                                                    order="F")


def _cfg():
    return O.StreamConfig(rank=R, p=P, q=Q, shared=SH, seed=SEED, als=O.AlsConfig(R, ITERS, TOL, RESTARTS, 0))


def _allgather(vec, world):
    t = torch.from_numpy(vec)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return torch.cat(out).numpy()


def _sharded_rank(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _data()
        cfg = _cfg()
        p0, pl = S.shard_range(P, world, rank)
        rs = O.gen_replicas([x.shape[0], x.shape[1]], Q, P, SH, SEED)  # all replicas (host RNG)
        summ = O.init_summaries(rs)  # only owned y are ever filled; history kept for all
        model, k = None, 0
        for b in range(NB + 1):
            t0, t = (0, K0) if b == 0 else (K0 + (b - 1) * T, T)
            batch = O.slice_mode(x, 2, t0, t)
            # begin: compress + CP-ALS of the owned replicas
            O.extend_temporal(rs, t)
            for r in range(p0, p0 + pl):
                summ.y[r] = summ.y[r] + O.compress(batch, rs, r, k, k + t)
            fac, lam = [], []
            for r in range(p0, p0 + pl):
                res = O.cp_als(summ.y[r], O.AlsConfig(R, ITERS, TOL, RESTARTS,
                                                      rng.derive(SEED, [rng.K_STREAM_ALS, r, b])))
                fac.append(res.model.factors)
                lam.append(res.model.lambda_)
            status, facs, lams = S.unpack_models(_allgather(S.pack_models(fac, lam, P, Q, R, world), world),
                                                 P, Q, R, world)
            assert all(s == (0, 0, 0) for s in status)
            models = [O.KruskalModel([f.copy() for f in fs], l) for fs, l in zip(facs, lams)]
            # merge: redundant alignment + A/B recovery, rows of the owned replicas
            aligned = O.align_replicas(models, rs)
            stored = [] if model is None else [model.factors[0], model.factors[1]]
            final, _ = O._recover_nontemporal_final(aligned, rs, stored)
            own = O.temporal_stack_from_summaries(rs, summ, final)[p0 * Q:(p0 + pl) * Q]
            rows_local = [own[i * Q:(i + 1) * Q] for i in range(pl)]
            tstack = S.unpack_rows(_allgather(S.pack_rows(rows_local, P, Q, R, world), world), P, Q, R, world)
            # finish: temporal append + model assembly
            c_old = np.zeros((0, R)) if model is None else model.factors[2] * model.lambda_[None, :]
            temporal = O.recover_temporal_append(tstack, rs, summ, c_old, t)
            model = O._assemble_model(final, np.vstack([c_old, temporal.new_rows]), 2)
            O.drop_temporal_history(rs)
            k += t
        np.savez(os.path.join(out_dir, "rank%d.npz" % rank), a=model.factors[0], b=model.factors[1],
                 c=model.factors[2], lam=model.lambda_)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_cover_every_replica_once():
    for p in range(1, 20):
        for world in range(1, p + 1):
            seen = []
            for g in range(world):
                p0, pl = S.shard_range(p, world, g)
                seen += list(range(p0, p0 + pl))
            assert seen == list(range(p))
    with pytest.raises(ValueError):
        S.shard_range(3, 4, 0)


def test_exchange_layout_round_trip():
    s = rng.Substream(5)
    world = 3
    blocks = []
    facs_all, lams_all, rows_all = [], [], []
    for g in range(world):
        p0, pl = S.shard_range(7, world, g)
        f = [[s.fill_uniform(4, 2) for _ in range(3)] for _ in range(pl)]
        lm = [s.uniform01_array(2) for _ in range(pl)]
        facs_all += f
        lams_all += lm
        blocks.append(S.pack_models(f, lm, 7, 4, 2, world))
        rows_all.append([s.fill_uniform(4, 2) for _ in range(pl)])
    status, facs, lams = S.unpack_models(np.concatenate(blocks), 7, 4, 2, world)
    assert status == [(0, 0, 0)] * world
    for a, b in zip(facs, facs_all):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert all(np.array_equal(a, b) for a, b in zip(lams, lams_all))
    stack = S.unpack_rows(np.concatenate([S.pack_rows(r, 7, 4, 2, world) for r in rows_all]), 7, 4, 2, world)
    assert np.array_equal(stack, np.vstack([m for r in rows_all for m in r]))


def test_gloo_two_rank_sharded_stream_matches_unsharded(tmp_path):
    port = _free_port()
    mp.start_processes(_sharded_rank, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    r0, r1 = (np.load(tmp_path / ("rank%d.npz" % g)) for g in range(2))
    for k in ("a", "b", "c", "lam"):
        assert np.array_equal(r0[k], r1[k])  # redundant merge: bit-identical ranks
    x = _data()
    ref = O.init_stream(O.slice_mode(x, 2, 0, K0), _cfg())
    for b in range(NB):
        O.ingest_batch(ref, O.slice_mode(x, 2, K0 + b * T, T))
    for k, f in zip("abc", ref.model.factors):
        assert np.allclose(r0[k], f, rtol=0, atol=1e-12 * np.abs(f).max())
    assert np.allclose(r0["lam"], ref.model.lambda_, rtol=1e-12)


def _temporal_rank(rank, world, port, out_dir):
    """Temporal sharding on CPU: each rank compresses its slice range into
    partials of EVERY replica (oracle compress with the batch's temporal rows
    at its offset), the partials are reduce-scattered by owner over gloo, and
    the owners' summaries must equal the unsharded oracle's."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _data()
        p0, pl = S.shard_range(P, world, rank)
        chunk = -(-P // world)
        rs = O.gen_replicas([x.shape[0], x.shape[1]], Q, P, SH, SEED)
        y = [np.zeros((Q, Q, Q)) for _ in range(P)]
        k = 0
        for b in range(NB + 1):
            t0, t = (0, K0) if b == 0 else (K0 + (b - 1) * T, T)
            O.extend_temporal(rs, t)  # every rank draws the whole batch's rows
            lo, hi = t * rank // world, t * (rank + 1) // world
            part = np.zeros(world * (chunk * Q ** 3 + 1))
            if hi > lo:
                loc = O.slice_mode(x, 2, t0 + lo, hi - lo)
                for r in range(P):
                    z = O.compress(loc, rs, r, k + lo, k + hi)
                    g, i = r // chunk, r % chunk
                    off = g * (chunk * Q ** 3 + 1) + i * Q ** 3
                    part[off:off + Q ** 3] = z.ravel(order="F")
            send = torch.from_numpy(part)
            recv = torch.zeros(chunk * Q ** 3 + 1, dtype=torch.float64)
            dist.reduce_scatter(recv, list(send.chunk(world)))
            got = recv.numpy()
            for i in range(pl):
                y[p0 + i] = y[p0 + i] + got[i * Q ** 3:(i + 1) * Q ** 3].reshape((Q, Q, Q), order="F")
            k += t
        np.save(os.path.join(out_dir, "y%d.npy" % rank), np.stack([y[p0 + i] for i in range(pl)]))
    finally:
        dist.destroy_process_group()


def test_temporal_sharding_reduce_scatter_two_ranks(tmp_path):
    world = 2
    port = _free_port()
    mp.spawn(_temporal_rank, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    x = _data()
    rs = O.gen_replicas([x.shape[0], x.shape[1]], Q, P, SH, SEED)
    summ = O.init_summaries(rs)
    k = 0
    for b in range(NB + 1):
        t0, t = (0, K0) if b == 0 else (K0 + (b - 1) * T, T)
        O.extend_temporal(rs, t)
        O.update_summaries(summ, [O.compress(O.slice_mode(x, 2, t0, t), rs, r, k, k + t) for r in range(P)])
        k += t
    for g in range(world):
        p0, pl = S.shard_range(P, world, g)
        ys = np.load(os.path.join(str(tmp_path), "y%d.npy" % g))
        for i in range(pl):
            ref = summ.y[p0 + i]
            assert np.linalg.norm(ys[i] - ref) <= 1e-12 * np.linalg.norm(ref)
