"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on
the same seeded inputs, stage by stage and end to end.

Tolerances (written per test): fp64 stages match to 1e-9..1e-12 relative;
the fp32-input compression to 1e-5 relative Frobenius (BASELINE north star:
<= 1e-4); whole-pipeline factors are compared after permutation/sign matching
(congruence, eval.cpp:22-46) because eigen-solver column order is not part of
the reference contract (SURVEY.md §7 hard part 4).
"""
import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ob():
    import torch
    assert torch.cuda.is_available()
    import paper_1807_01350_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def random_truth(dims, rank, seed):
    s = rng.Substream(seed)
    return O.KruskalModel([s.fill_uniform(d, rank) for d in dims], np.ones(rank))


def model_congruence(a, b):
    """min over components of the FMS-style product of |cos| after matching."""
    return min(O.congruence(O.KruskalModel([f.copy() for f in a.factors], np.asarray(a.lambda_).copy()),
                            O.KruskalModel([f.copy() for f in b.factors], np.asarray(b.lambda_).copy())))


def _small_replicas(I=12, J=10, t=7, Q=5, P=3, sh=2, seed=55):
    rs = O.gen_replicas([I, J], Q, P, sh, seed)
    O.extend_temporal(rs, t)
    u = [r.nontemporal[0] for r in rs.replicas]
    v = [r.nontemporal[1] for r in rs.replicas]
    w = [r.temporal for r in rs.replicas]
    return rs, u, v, w


# ---------------------------------------------------------------- compression

@pytest.mark.parametrize("shape", [(12, 10, 7, 5, 3, 2), (40, 33, 9, 8, 4, 3), (64, 48, 20, 16, 5, 4)])
def test_compress_f64_matches_oracle(ob, shape):
    I, J, t, Q, P, sh = shape
    rs, u, v, w = _small_replicas(I, J, t, Q, P, sh)
    x = (rng.Substream(9).uniform01_array(I * J * t) * 2 - 1).reshape((I, J, t), order="F")
    c0 = ob.kernel_counts()
    got = ob.compress(x, u, v, w, sh)
    c1 = ob.kernel_counts()
    assert c1["dmma_compress"] - c0["dmma_compress"] == 2  # GEMM1 and mode-2 on the FP64 tensor cores
    for r in range(P):
        want = O.compress(x, rs, r, 0, t)
        assert rel(got[r], want) < 1e-12  # fp64 path


def test_compress_f32_within_tolerance(ob):
    I, J, t, Q, P, sh = 100, 90, 12, 20, 6, 5
    rs, u, v, w = _small_replicas(I, J, t, Q, P, sh)
    x = rng.Substream(10).uniform01_array(I * J * t).reshape((I, J, t), order="F").astype(np.float32)
    got = ob.compress(x, u, v, w, sh)
    for r in range(P):
        want = O.compress(x.astype(np.float64), rs, r, 0, t)
        assert rel(got[r], want) < 1e-5  # fp32 inputs: BASELINE tolerance is 1e-4


@pytest.mark.parametrize("shape", [(200, 300, 12, 40, 5, 4), (1000, 64, 9, 100, 4, 10), (96, 50, 7, 30, 9, 6),
                                   (300, 200, 6, 128, 3, 32), (160, 128, 5, 120, 2, 8)])
def test_compress_f32_tcgen05_vs_simt_and_oracle(ob, shape, monkeypatch):
    # the tcgen05 split-TF32 mode-1 kernel (M/N/K tails: several tiles, K not a
    # multiple of 32) against the fp64 oracle and the SIMT fp32 path
    I, J, t, Q, P, sh = shape
    rs, u, v, w = _small_replicas(I, J, t, Q, P, sh, seed=I + J)
    x = rng.Substream(I * J).uniform01_array(I * J * t).reshape((I, J, t), order="F").astype(np.float32)
    c0 = ob.kernel_counts()
    got_tc = ob.compress(x, u, v, w, sh)
    c1 = ob.kernel_counts()
    # the tensor-core path ran: GEMM1 on tcgen05, and mode-2 too unless J is
    # not a multiple of 4 (a TMA box alignment limit: that chunk's mode-2 is
    # the counted SIMT fallback)
    mode2_tc = J % 4 == 0
    assert c1["tcgen05"] - c0["tcgen05"] == (2 if mode2_tc else 1)
    assert c1["simt_fallbacks"] - c0["simt_fallbacks"] == (0 if mode2_tc else 1)
    monkeypatch.setenv("OCTEN_DISABLE_TCGEN05", "1")
    got_simt = ob.compress(x, u, v, w, sh)
    monkeypatch.delenv("OCTEN_DISABLE_TCGEN05")
    for r in range(P):
        want = O.compress(x.astype(np.float64), rs, r, 0, t)
        # split-TF32 with the tensor core's fp32 accumulation: the accumulator
        # rounds toward zero, a bias of ~K/2 ulps on positive data (2e-5 at
        # K=1000); BASELINE tolerance is 1e-4 relative Frobenius.
        assert rel(got_tc[r], want) < 1e-4 * max(1.0, I / 1000.0)
        assert rel(got_simt[r], want) < 5e-6


def test_compress_zero_and_rank1(ob):
    # test_compression.cpp:108-144
    rs, u, v, w = _small_replicas(6, 5, 4, 3, 2, 1, seed=77)
    s = rng.Substream(31)
    a, b, c = s.uniform01_array(6), s.uniform01_array(5), s.uniform01_array(4)
    t = O.rank1_outer([a, b, c])
    z = ob.compress(t, u, v, w, 1)
    expect = O.rank1_outer([u[1].T @ a, v[1].T @ b, w[1].T @ c])
    assert rel(z[1], expect) < 1e-10
    z0 = ob.compress(np.zeros((6, 5, 4)), u, v, w, 1)
    assert all(np.all(zz == 0.0) for zz in z0)


# ---------------------------------------------------------------- CP-ALS

def _summaries(I, J, K, R, Q, P, sh, seed, noise=0.0):
    truth = random_truth([I, J, K], R, seed)
    x = O.reconstruct(truth)
    if noise:
        x = x + noise * (rng.Substream(seed + 1).uniform01_array(x.size) - 0.5).reshape(x.shape, order="F")
    rs = O.gen_replicas([I, J], Q, P, sh, seed + 2)
    O.extend_temporal(rs, K)
    return [O.compress(x, rs, r, 0, K) for r in range(P)]


@pytest.mark.parametrize("noise", [0.0, 0.01])
def test_cp_als_matches_oracle(ob, noise):
    ys = _summaries(30, 28, 25, 4, 12, 4, 3, seed=5, noise=noise)
    cfg = ob.AlsConfig(rank=4, max_iters=60, rel_tol=1e-10, n_restarts=3)
    seeds = [rng.derive(100, [r]) for r in range(len(ys))]
    models, fits, iters = ob.cp_als_batched(ys, cfg, seeds)
    for r, y in enumerate(ys):
        ref = O.cp_als(y, O.AlsConfig(4, 60, 1e-10, 3, seeds[r]))
        assert abs(fits[r] - ref.fit) < 1e-7
        assert model_congruence(models[r], ref.model) > 1 - 1e-6
        assert np.allclose(np.sort(models[r].lambda_), np.sort(ref.model.lambda_), rtol=1e-5)
        for f in models[r].factors:
            assert np.allclose(np.linalg.norm(f, axis=0), 1.0, atol=1e-12)


def test_cp_als_known_answers(ob):
    # test_cp_als.cpp:65-93: rank-1 noiseless and the indicator tensor (Q=4/3 cubes)
    s = rng.Substream(17)
    vecs = [0.1 + 0.9 * s.uniform01_array(4) for _ in range(3)]
    m, fit, _ = ob.cp_als_batched([O.rank1_outer(vecs)], ob.AlsConfig(rank=1, seed=0), [99])
    assert fit[0] >= 0.999999
    e1 = np.zeros(3)
    e1[0] = 1.0
    m, fit, _ = ob.cp_als_batched([O.rank1_outer([e1, e1, e1])], ob.AlsConfig(rank=1), [3])
    assert abs(m[0].lambda_[0] - 1.0) < 1e-9
    for f in m[0].factors:
        assert abs(abs(f[0, 0]) - 1.0) < 1e-8 and abs(f[1, 0]) < 1e-7


def test_cp_als_zero_tensor_raises(ob):
    with pytest.raises(ob.NumericError, match="identically zero"):
        ob.cp_als_batched([np.zeros((3, 3, 3))], ob.AlsConfig(rank=1), [1])


# ---------------------------------------------------------------- alignment / recovery

def _oracle_models(I, J, K, R, Q, P, sh, seed, noise=0.0):
    truth = random_truth([I, J, K], R, seed)
    x = O.reconstruct(truth)
    if noise:
        x = x + noise * (rng.Substream(seed + 1).uniform01_array(x.size) - 0.5).reshape(x.shape, order="F")
    rs = O.gen_replicas([I, J], Q, P, sh, seed + 2)
    O.extend_temporal(rs, K)
    models = [O.cp_als(O.compress(x, rs, r, 0, K), O.AlsConfig(R, 200, 1e-12, 2, rng.derive(seed, [r]))).model
              for r in range(P)]
    return rs, models, x, truth


@pytest.mark.parametrize("dims", [(40, 35, 10, 3, 8, 6, 3), (12, 10, 6, 3, 8, 3, 2)])
def test_align_matches_oracle(ob, dims):
    I, J, K, R, Q, P, sh = dims  # second case exercises the pair-solve branch (2Q >= I+1)
    rs, models, _, _ = _oracle_models(I, J, K, R, Q, P, sh, seed=11)
    ref = O.align_replicas(models, rs)
    u = [r.nontemporal[0] for r in rs.replicas]
    v = [r.nontemporal[1] for r in rs.replicas]
    stacks, perms, scales, mn, mx = ob.align_replicas(models, u, v, rs.temporal_shared_gram, sh)
    for rep in range(P):
        assert perms[rep].tolist() == ref.perms[rep]
    for n in range(3):
        assert rel(stacks[n], ref.stacks[n]) < 1e-9
    assert abs(mn - ref.min_match_similarity) < 1e-6
    assert abs(mx - ref.max_offdiag_similarity) < 1e-6


def test_recover_nontemporal_matches_oracle(ob):
    rs = O.gen_replicas([50, 40], 12, 6, 3, 4)
    blocks = [r.nontemporal[0] for r in rs.replicas]
    proj = O.stack_projections(rs, 0)
    truth = rng.Substream(5).fill_uniform(50, 4)
    stack = proj @ truth + 1e-3 * rng.Substream(6).fill_uniform(proj.shape[0], 4)
    got = ob.recover_nontemporal(stack, blocks, 0)
    want = O.recover_nontemporal(stack, proj, 0)
    assert rel(got, want) < 1e-9


def _near_dependent_blocks(eps, d=40, q=15, p=4, seed=41):
    """Projection blocks whose stacked projection has one column within
    `eps` (relative) of the span of two others: |r_nn| / |r_00| ~ eps."""
    rs = O.gen_replicas([d, 10], q, p, 3, seed)
    blocks = [r.nontemporal[0].copy() for r in rs.replicas]
    noise = rng.Substream(seed + 1)
    for b in blocks:
        b[d - 1, :] = 0.5 * (b[0, :] + b[1, :]) + eps * (noise.fill_uniform(1, q)[0] - 0.5)
    proj = np.vstack([b.T for b in blocks])
    return blocks, proj


@pytest.mark.parametrize("eps", [1e-7, 1e-8])
def test_recover_nontemporal_qr_band(ob, eps):
    # |r_nn| / |r_00| between the reference's QR threshold (1e-10,
    # recovery.cpp:26-38) and what a Gram pivot can resolve (~3e-6): the
    # reference solves, so must the device (column-pivoted QR fallback)
    blocks, proj = _near_dependent_blocks(eps)
    assert O.colpiv_qr_rank(proj, O.K_RANK_TOL) == proj.shape[1]
    truth = rng.Substream(7).fill_uniform(proj.shape[1], 3)
    stack = proj @ truth + 1e-9 * rng.Substream(8).fill_uniform(proj.shape[0], 3)
    got = ob.recover_nontemporal(stack, blocks, 0)
    want = O.recover_nontemporal(stack, proj, 0)
    # conditioning ~1/eps: the two least-squares solutions agree to ~eps^-1 ulp
    assert rel(got, want) < 1e-16 / eps * 1e3


def test_recover_nontemporal_qr_band_rank_deficient(ob):
    # below the reference's threshold both raise the same rank message
    blocks, proj = _near_dependent_blocks(1e-13)
    rk = O.colpiv_qr_rank(proj, O.K_RANK_TOL)
    assert rk == proj.shape[1] - 1
    stack = np.ones((proj.shape[0], 2))
    with pytest.raises(O.NumericError):
        O.recover_nontemporal(stack, proj, 0)
    with pytest.raises(ob.NumericError, match=r"recover: rank-deficient projection on mode 1 \(rank %d of %d\)"
                       % (rk, proj.shape[1])):
        ob.recover_nontemporal(stack, blocks, 0)


def test_recover_nontemporal_error_messages(ob):
    # test_recovery.cpp:224-236
    rs = O.gen_replicas([4, 4], 2, 3, 2, 8)
    with pytest.raises(ob.NumericError, match=r"recover: rank-deficient projection on mode 1 \(rank 2 of 4\)"):
        ob.recover_nontemporal(np.ones((6, 2)), [r.nontemporal[0] for r in rs.replicas], 0)
    thin = O.gen_replicas([10, 10], 2, 2, 1, 8)
    with pytest.raises(ob.NumericError, match=r"recover: mode 1 projection is 4x10; p\*Q must reach"):
        ob.recover_nontemporal(np.ones((4, 2)), [r.nontemporal[0] for r in thin.replicas], 0)


def test_temporal_stack_and_append_match_oracle(ob):
    I, J, K, R, Q, P, sh = 40, 35, 10, 3, 8, 9, 3  # rank of the stacked U: 3 + 9*5 = 48 >= 40
    rs, models, x, truth = _oracle_models(I, J, K, R, Q, P, sh, seed=21)
    summ = O.init_summaries(rs)
    O.update_summaries(summ, [O.compress(x, rs, r, 0, K) for r in range(P)])
    al = O.align_replicas(models, rs)
    projs = [O.stack_projections(rs, n) for n in range(2)]
    a = O.column_normalized(O.recover_nontemporal(al.stacks[0], projs[0], 0))
    b = O.column_normalized(O.recover_nontemporal(al.stacks[1], projs[1], 1))
    want = O.temporal_stack_from_summaries(rs, summ, [a, b])
    got = ob.temporal_stack_from_summaries(summ.y, [r.nontemporal[0] for r in rs.replicas],
                                           [r.nontemporal[1] for r in rs.replicas], a, b)
    assert rel(got, want) < 1e-9
    # first batch append == plain solve (test_recovery.cpp:282-302)
    hist = [np.zeros((Q, 0)) for _ in range(P)]
    rows, res = ob.recover_temporal_append(want, [r.temporal for r in rs.replicas], hist)
    ref = O.recover_temporal_append(want, rs, summ, np.zeros((0, R)), K)
    assert rel(rows, ref.new_rows) < 1e-9
    assert abs(res - ref.solve_residual) < 1e-9
    for r in range(P):
        assert rel(hist[r], summ.history[r]) < 1e-9
    # a second batch with history: the gauge path
    O.extend_temporal(rs, 4)
    w2 = [r.temporal_rows(K, K + 4) for r in rs.replicas]
    stack2 = want + 0.01 * rng.Substream(3).fill_uniform(P * Q, R)
    rows2, res2 = ob.recover_temporal_append(stack2, w2, hist)
    ref2 = O.recover_temporal_append(stack2, rs, summ, np.zeros((K, R)), 4)
    assert rel(rows2, ref2.new_rows) < 1e-8
    assert abs(res2 - ref2.solve_residual) < 1e-8


# ---------------------------------------------------------------- end to end

def _desk(ob, rank, p, q, shared, seed, **kw):
    return ob.StreamConfig(rank=rank, p=p, q=q, shared=shared, seed=seed,
                           als=ob.AlsConfig(max_iters=kw.get("iters", 300), rel_tol=kw.get("tol", 1e-12),
                                            n_restarts=kw.get("restarts", 2)))


def _ocfg(c):
    return O.StreamConfig(rank=c.rank, p=c.p, q=c.q, shared=c.shared, seed=c.seed,
                          als=O.AlsConfig(c.als.rank, c.als.max_iters, c.als.rel_tol, c.als.n_restarts, 0))


def test_noiseless_stream_tracks_and_matches_oracle(ob):
    # test_streaming.cpp:78-96 on the device, and against the oracle run
    truth = random_truth([30, 30, 20], 4, 91)
    full = O.reconstruct(truth)
    cfg = _desk(ob, 4, 6, 15, 3, 17)
    st = ob.init_stream(O.slice_mode(full, 2, 0, 5), cfg)
    ref = O.init_stream(O.slice_mode(full, 2, 0, 5), _ocfg(cfg))
    for b in range(1, 4):
        ob.ingest_batch(st, O.slice_mode(full, 2, 5 * b, 5))
        O.ingest_batch(ref, O.slice_mode(full, 2, 5 * b, 5))
    assert st.slices_seen == 20
    m = st.model
    mk = O.KruskalModel(m.factors, m.lambda_)
    assert O.fitness(full, O.reconstruct(mk)) >= 95.0
    assert min(O.congruence(truth, mk)) >= 0.99
    assert model_congruence(mk, ref.model) > 1 - 1e-8
    ys, hs = st.summaries()
    for r in range(cfg.p):
        assert rel(ys[r], ref.summaries.y[r]) < 1e-12


def test_noisy_stream_matches_oracle(ob):
    I, K0, t, Q, P, R, sh = 60, 40, 10, 12, 8, 3, 3
    x, truth = O.generate_synthetic([I, I, K0 + 2 * t], R, 3, 0.0, 0.0)
    x = x + 0.01 * np.sqrt(np.mean(x ** 2)) * rng.Substream(4).normal_array(x.size, 0, 1).reshape(x.shape, order="F")
    cfg = _desk(ob, R, P, Q, sh, 38, iters=30, tol=1e-8, restarts=3)
    st = ob.init_stream(O.slice_mode(x, 2, 0, K0), cfg)
    ref = O.init_stream(O.slice_mode(x, 2, 0, K0), _ocfg(cfg))
    for b in range(2):
        ob.ingest_batch(st, O.slice_mode(x, 2, K0 + b * t, t))
        O.ingest_batch(ref, O.slice_mode(x, 2, K0 + b * t, t))
    m = st.model
    mk = O.KruskalModel(m.factors, m.lambda_)
    f_dev = O.fitness(x, O.reconstruct(mk))
    f_ref = O.fitness(x, O.reconstruct(ref.model))
    assert abs(f_dev - f_ref) < 1e-3
    assert model_congruence(mk, ref.model) > 1 - 1e-6
    for a, b in zip(st.log, ref.log):
        assert abs(a.temporal_residual - b.temporal_residual) < 1e-6 * max(1.0, b.temporal_residual)


def test_stream_fp32_input(ob):
    import torch
    truth = random_truth([30, 30, 20], 4, 91)
    full = O.reconstruct(truth).astype(np.float32)
    cfg = _desk(ob, 4, 6, 15, 3, 17)
    dev = torch.from_numpy(np.ascontiguousarray(full.transpose(2, 1, 0))).cuda().permute(2, 1, 0)
    st = ob.init_stream(dev[:, :, :5], cfg)
    for b in range(1, 4):
        ob.ingest_batch(st, dev[:, :, 5 * b:5 * b + 5])
    m = st.model
    mk = O.KruskalModel(m.factors, m.lambda_)
    assert O.fitness(full.astype(np.float64), O.reconstruct(mk)) >= 95.0
    assert min(O.congruence(truth, mk)) >= 0.99


def test_reference_error_paths(ob):
    # c1 shape: P*Q = 80 < I = 100 -> NumericError from recover
    x = (rng.Substream(1).uniform01_array(100 * 100 * 10)).reshape((100, 100, 10), order="F")
    cfg = ob.StreamConfig(rank=5, p=4, q=20, shared=4, seed=3, als=ob.AlsConfig(max_iters=5))
    with pytest.raises(ob.NumericError, match=r"recover: mode 1 projection is 80x100"):
        ob.init_stream(x, cfg)
    with pytest.raises(ob.ConfigError, match="tensor order must be >= 3"):
        ob.init_stream(np.ones((4, 4)), _desk(ob, 2, 2, 3, 1, 5))
    c = _desk(ob, 5, 1, 30, 5, 11)
    c.enforce_bounds = True
    with pytest.raises(ob.ConfigError, match="need p >= 2"):
        ob.init_stream(O.reconstruct(random_truth([50, 50, 5], 5, 1)), c)
    full = O.reconstruct(random_truth([10, 9, 8], 2, 5))
    st = ob.init_stream(O.slice_mode(full, 2, 0, 4), _desk(ob, 2, 4, 6, 2, 3))
    with pytest.raises(ob.ConfigError, match="extent mismatch on mode 2 at batch 1"):
        ob.ingest_batch(st, np.zeros((10, 7, 2)))
    bad = np.zeros((10, 9, 2))
    bad[0, 0, 0] = np.nan
    with pytest.raises(ob.NumericError, match="non-finite"):
        ob.ingest_batch(st, bad)


def test_strict_mode_rolls_back(ob):
    # test_streaming.cpp:175-186
    full = O.reconstruct(random_truth([10, 9, 8], 2, 59))
    cfg = _desk(ob, 2, 4, 6, 2, 3)
    cfg.strict = True
    cfg.residual_warning = 0.0
    with pytest.raises(ob.NumericError, match="exceeds strict threshold"):
        ob.init_stream(O.slice_mode(full, 2, 0, 4), cfg)


def test_history_telescopes(ob):
    # test_recovery.cpp:270-280 on the device
    truth = random_truth([10, 9, 12], 2, 5)
    truth.normalize()
    full = O.reconstruct(truth)
    cfg = ob.StreamConfig(rank=2, p=4, q=6, shared=2, seed=1001, als=ob.AlsConfig(max_iters=400, rel_tol=1e-13))
    st = ob.init_stream(O.slice_mode(full, 2, 0, 4), cfg)
    ob.ingest_batch(st, O.slice_mode(full, 2, 4, 4))
    ob.ingest_batch(st, O.slice_mode(full, 2, 8, 4))
    shadow = O.gen_replicas([10, 9], 6, 4, 2, 1001, 2)
    for _ in range(3):
        O.extend_temporal(shadow, 4)
    m = st.model
    c_raw = m.factors[2] * m.lambda_[None, :]
    _, hs = st.summaries()
    for r in range(4):
        assert np.max(np.abs(shadow.replicas[r].temporal.T @ c_raw - hs[r])) < 1e-8


# ------------------------------------------------- full-size property checks

def _truth_stream(ob, dims, R, K0, t, nb, Q, P, sh, seed, iters=30, noise=0.0, dtype="f32"):
    """Rank-R U(0,1) truth (+ noise) streamed as device batches (fp32: the
    BASELINE fp32 configs; fp64: exact inputs)."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    I, J = dims
    K = K0 + nb * t
    A = torch.rand((I, R), generator=g, device="cuda", dtype=torch.float64)
    B = torch.rand((J, R), generator=g, device="cuda", dtype=torch.float64)
    C = torch.rand((K, R), generator=g, device="cuda", dtype=torch.float64)
    x = torch.einsum("kr,jr,ir->kji", C, B, A)
    if noise:
        x += noise * x.pow(2).mean().sqrt() * torch.randn(x.shape, generator=g, device="cuda", dtype=torch.float64)
    xd = (x.to(torch.float32) if dtype == "f32" else x).permute(2, 1, 0)  # (I, J, K) first-index-fastest view
    cfg = ob.StreamConfig(rank=R, p=P, q=Q, shared=sh, seed=seed,
                          als=ob.AlsConfig(rank=R, max_iters=iters, rel_tol=1e-8, n_restarts=3))
    st = ob.init_stream(xd[:, :, :K0], cfg)
    for b in range(nb):
        ob.ingest_batch(st, xd[:, :, K0 + b * t:K0 + (b + 1) * t])
    return st, (A.cpu().numpy(), B.cpu().numpy(), C.cpu().numpy()), x


def _fit_gpu(x, m):
    """fitness (eval.cpp:10-20) of a model against the device tensor (K, J, I)."""
    import torch
    f = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in m.factors]
    lam = torch.from_numpy(np.asarray(m.lambda_)).cuda()
    xh = torch.einsum("kr,jr,ir->kji", f[2] * lam[None, :], f[1], f[0])
    return 100.0 * (1.0 - float((x - xh).norm() / x.norm()))


def test_c3_scale_noiseless_stream_recovers_truth(ob):
    # BASELINE c3 shapes (I=J=1000, Q=100, P=16, R=20, batches of 100 after
    # K0=1000; shared=10), exact (fp64) inputs, two batches: the
    # model recovers the ground truth (size-independent property)
    st, (A, B, C), x = _truth_stream(ob, (1000, 1000), 20, 1000, 100, 2, 100, 16, 10, 3, dtype="f64")
    m = st.model
    assert st.slices_seen == 1200
    truth = O.KruskalModel([A, B, C], np.ones(20))
    assert min(O.congruence(truth, O.KruskalModel(m.factors, m.lambda_))) > 0.999
    for rec in st.log:
        assert rec.temporal_residual < 1e-6


def test_c3_scale_fp32_compression_within_tolerance(ob):
    # the north-star tolerance at the full c3 batch shape: the fp32 batch
    # through the split-TF32 tcgen05 path stays within 1e-4 relative Frobenius
    # error of the exact (fp64) compression of the same values, every replica
    I = J = 1000
    t, Q, P, sh = 100, 100, 16, 10
    rs = O.gen_replicas([I, J], Q, P, sh, 55)
    O.extend_temporal(rs, t)
    u = [r.nontemporal[0] for r in rs.replicas]
    v = [r.nontemporal[1] for r in rs.replicas]
    w = [r.temporal for r in rs.replicas]
    x = rng.Substream(9).uniform01_array(I * J * t).reshape((I, J, t), order="F").astype(np.float32)
    z32 = ob.compress(x, u, v, w, sh)
    z64 = ob.compress(x.astype(np.float64), u, v, w, sh)
    for a, b in zip(z32, z64):
        assert rel(a, b) < 1e-4


def test_c5_shapes_noiseless_stream_recovers_truth(ob):
    # BASELINE c5 per-GPU shapes (I=J=2000, Q=128, P=32, R=32; shared=32 <= 67
    # per the replica bound), exact inputs, a short stream
    st, (A, B, C), x = _truth_stream(ob, (2000, 2000), 32, 200, 200, 1, 128, 32, 32, 5, iters=30, dtype="f64")
    m = st.model
    assert all(np.isfinite(f).all() for f in m.factors) and np.isfinite(m.lambda_).all()
    truth = O.KruskalModel([A, B, C], np.ones(32))
    assert min(O.congruence(truth, O.KruskalModel(m.factors, m.lambda_))) > 0.999
