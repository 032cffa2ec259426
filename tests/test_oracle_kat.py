"""Pin the CPU oracle against the reference's own known-answer and property
tests.  Each test names the reference test it restates.
CPU only."""
import math

import numpy as np
import pytest

from oracle import octen_oracle as O
from oracle import rng


def random_tensor(shape, seed):
    """tests/test_tensor.cpp:71-76 random_tensor: uniform(-1,1), flat order."""
    s = rng.Substream(seed)
    n = int(np.prod(shape))
    return (s.uniform01_array(n) * 2.0 - 1.0).reshape(shape, order="F")


def random_truth(dims, rank, seed):
    """tests/test_streaming.cpp:15-25."""
    s = rng.Substream(seed)
    return O.KruskalModel([s.fill_uniform(d, rank) for d in dims], np.ones(rank))


# --- rng.hpp ---------------------------------------------------------------

def test_mt19937_64_standard_known_answer():
    # C++ [rand.predef]: 10000th output of default-seeded mt19937_64.
    e = rng.MT19937_64(5489)
    assert int(e.next_u64_array(10000)[-1]) == 9981545732273789042


def test_mt19937_64_chunked_draws_match_single_draws():
    a = rng.MT19937_64(123)
    b = rng.MT19937_64(123)
    big = a.next_u64_array(1000)
    small = np.array([b.next_u64() for _ in range(1000)], dtype=np.uint64)
    assert np.array_equal(big, small)


def test_derive_is_splitmix_chain():
    # rng.hpp:23-29 restated by hand for one path.
    z = rng.mix(42)
    for k in (1, 2, 3):
        z = rng.mix(z ^ rng.mix(k))
    assert rng.derive(42, [1, 2, 3]) == z
    assert rng.derive(42, [1, 2, 3]) != rng.derive(42, [1, 3, 2])


def test_uniform01_is_53_bit():
    s = rng.Substream(7)
    u = s.uniform01_array(10000)
    assert u.min() >= 0.0 and u.max() < 1.0
    assert np.all(u * 2.0 ** 53 == np.floor(u * 2.0 ** 53))


# --- tensor.cpp (tests/test_tensor.cpp) -------------------------------------

def test_matricize_2mode_identity():  # test_tensor.cpp:78-89
    t = np.array([1.0, 2, 3, 4]).reshape((2, 2), order="F")
    m = O.matricize(t, 0)
    assert m.tolist() == [[1, 3], [2, 4]]


def test_matricize_frozen_2x2x2():  # test_tensor.cpp:91-102
    t = np.arange(1.0, 9.0).reshape((2, 2, 2), order="F")
    assert O.matricize(t, 0).tolist() == [[1, 3, 5, 7], [2, 4, 6, 8]]


def test_matricize_round_trip_bit_exact():  # test_tensor.cpp:110-118
    t = random_tensor((4, 5, 6, 3), 42)
    for mode in range(4):
        m = O.matricize(t, mode)
        assert np.array_equal(O.dematricize(m, t.shape, mode), t)


def test_mode_product_identity_and_oracle():  # test_tensor.cpp:120-151
    t = random_tensor((3, 4, 2), 7)
    for mode in range(3):
        assert np.array_equal(O.mode_n_product(t, np.eye(t.shape[mode]), mode), t)
    ones = np.ones((2, 2, 2))
    out = O.mode_n_product(ones, np.array([[1.0, 1.0]]), 0)
    assert out.shape == (1, 2, 2) and np.allclose(out, 2.0)
    t = random_tensor((3, 4, 2), 11)
    m = rng.Substream(12).fill_uniform(5, 4)
    got = O.mode_n_product(t, m, 1)
    want = np.einsum("qj,ijk->iqk", m, t)
    assert np.allclose(got, want, rtol=1e-12, atol=0)
    with pytest.raises(O.ConfigError):
        O.mode_n_product(np.zeros((3, 4, 2)), np.zeros((2, 3)), 1)


def test_khatri_rao_frozen():  # test_tensor.cpp:198-218
    eye = np.eye(2)
    expect = np.zeros((4, 2))
    expect[0, 0] = 1
    expect[3, 1] = 1
    assert np.array_equal(O.khatri_rao(eye, eye), expect)
    x = np.array([[1.0, 2], [3, 4]])
    y = np.array([[0.0, 1], [1, 0]])
    assert O.khatri_rao(x, y).tolist() == [[0, 2], [1, 0], [0, 4], [3, 0]]
    with pytest.raises(O.ConfigError):
        O.khatri_rao(x, np.zeros((2, 3)))


def test_rank1_unfolding_identity():  # test_tensor.cpp:239-258
    s = rng.Substream(3)
    vecs = [s.uniform01_array(d) * 2 - 1 for d in (3, 4, 2)]
    t = O.rank1_outer(vecs)
    cols = [v[:, None] for v in vecs]
    for mode in range(3):
        chain = O.khatri_rao_chain(cols, mode)
        assert np.max(np.abs(O.matricize(t, mode) - cols[mode] @ chain.T)) < 1e-12


# --- compression.cpp (tests/test_compression.cpp) ---------------------------

def test_gen_replicas_validation():  # test_compression.cpp:24-28
    with pytest.raises(O.ConfigError):
        O.gen_replicas([4, 4], 3, 2, 4, 1)
    with pytest.raises(O.ConfigError):
        O.gen_replicas([4, 4], 0, 2, 0, 1)
    with pytest.raises(O.ConfigError):
        O.gen_replicas([4, 4], 3, 0, 1, 1)


def test_gen_replicas_sharing():  # test_compression.cpp:30-55
    rs = O.gen_replicas([5, 6], 4, 2, 4, 11)
    for m in range(2):
        assert np.array_equal(rs.replicas[0].nontemporal[m], rs.replicas[1].nontemporal[m])
    rs = O.gen_replicas([5, 6], 4, 2, 0, 11)
    for m in range(2):
        assert not np.array_equal(rs.replicas[0].nontemporal[m], rs.replicas[1].nontemporal[m])
    rs = O.gen_replicas([50, 50], 30, 20, 5, 42)
    for rep in rs.replicas:
        assert rep.nontemporal[0].shape == (50, 30)
        for m in range(2):
            assert np.array_equal(rep.nontemporal[m][:, :5], rs.replicas[0].nontemporal[m][:, :5])


def test_extend_temporal():  # test_compression.cpp:66-106
    rs = O.gen_replicas([4, 4], 3, 2, 1, 5)
    O.extend_temporal(rs, 5)
    first = rs.replicas[0].temporal.copy()
    O.extend_temporal(rs, 5)
    assert rs.replicas[0].temporal.shape[0] == 10
    assert np.array_equal(rs.replicas[0].temporal[:5], first)
    with pytest.raises(O.ConfigError):
        O.extend_temporal(rs, 0)
    rs = O.gen_replicas([4, 4], 4, 3, 2, 6)
    O.extend_temporal(rs, 3)
    O.extend_temporal(rs, 2)
    for r in (1, 2):
        assert np.array_equal(rs.replicas[r].temporal[:, :2], rs.replicas[0].temporal[:, :2])
    assert not np.array_equal(rs.replicas[1].temporal[:, 2:], rs.replicas[0].temporal[:, 2:])


def test_compress_rank1_stays_rank1():  # test_compression.cpp:108-144
    s = rng.Substream(31)
    a, b, c = s.uniform01_array(6), s.uniform01_array(5), s.uniform01_array(4)
    t = O.rank1_outer([a, b, c])
    rs = O.gen_replicas([6, 5], 3, 2, 1, 77)
    O.extend_temporal(rs, 4)
    z = O.compress(t, rs, 1, 0, 4)
    rep = rs.replicas[1]
    expect = O.rank1_outer([rep.nontemporal[0].T @ a, rep.nontemporal[1].T @ b, rep.temporal.T @ c])
    assert np.allclose(z, expect, rtol=1e-10, atol=0)


def test_summary_additivity():  # test_compression.cpp:182-226
    x_old = random_tensor((6, 6, 4), 101)
    x_new = random_tensor((6, 6, 3), 102)
    full = np.concatenate([x_old, x_new], axis=2)
    rs = O.gen_replicas([6, 6], 4, 3, 1, 55)
    O.extend_temporal(rs, 4)
    O.extend_temporal(rs, 3)
    for r in range(3):
        y = O.compress(x_old, rs, r, 0, 4)
        z = O.compress(x_new, rs, r, 4, 7)
        assert np.allclose(y + z, O.compress(full, rs, r, 0, 7), rtol=1e-10, atol=1e-12)


# --- cp_als.cpp (tests/test_cp_als.cpp) -------------------------------------

def test_cp_als_rank1_noiseless():  # test_cp_als.cpp:65-77
    s = rng.Substream(17)
    vecs = [0.1 + 0.9 * s.uniform01_array(4) for _ in range(3)]
    res = O.cp_als(O.rank1_outer(vecs), O.AlsConfig(rank=1, seed=99))
    assert res.fit >= 0.999999


def test_cp_als_indicator():  # test_cp_als.cpp:79-93
    e1 = np.zeros(3)
    e1[0] = 1.0
    res = O.cp_als(O.rank1_outer([e1, e1, e1]), O.AlsConfig(rank=1, seed=3))
    assert abs(res.model.lambda_[0] - 1.0) < 1e-9
    for f in res.model.factors:
        assert abs(abs(f[0, 0]) - 1.0) < 1e-8 and abs(f[1, 0]) < 1e-7 and abs(f[2, 0]) < 1e-7


def test_cp_als_rank3_congruence():  # test_cp_als.cpp:95-116
    s = rng.Substream(5)
    truth = O.KruskalModel([(s.uniform01_array(30) * 2 - 1).reshape((10, 3), order="F")
                            for _ in range(3)], np.ones(3))
    res = O.cp_als(O.reconstruct(truth), O.AlsConfig(rank=3, seed=1234, max_iters=300))
    assert min(O.congruence(truth, res.model)) >= 0.99


def test_cp_als_error_paths():  # test_cp_als.cpp:118-125
    with pytest.raises(O.NumericError):
        O.cp_als(np.zeros((3, 3, 3)), O.AlsConfig())
    with pytest.raises(O.ConfigError):
        O.cp_als(np.ones((2, 2, 2)), O.AlsConfig(rank=5))


def test_als_residual_monotone():  # test_cp_als.cpp:141-162
    for seed in (1, 2, 3, 4):
        s = rng.Substream(seed)
        truth = O.KruskalModel([s.fill_uniform(5, 3) for _ in range(3)], np.ones(3))
        t = O.reconstruct(truth)
        noise = rng.Substream(seed + 100)
        t = t + 0.01 * (noise.uniform01_array(t.size) - 0.5).reshape(t.shape, order="F")
        res = O.cp_als(t, O.AlsConfig(rank=2, seed=seed, n_restarts=1, max_iters=60))
        slack = 1e-9 * O.frobenius_norm(t)
        h = res.residual_history
        assert len(h) >= 2
        assert all(h[i] <= h[i - 1] + slack for i in range(1, len(h)))


def _oracle_mode_update(t, factors, mode):
    """test_cp_als.cpp:38-61 normal-equations oracle."""
    chain = O.khatri_rao_chain(factors, mode)
    return np.linalg.lstsq(chain, O.matricize(t, mode).T, rcond=None)[0].T


def test_mode_update_equals_normal_equations():  # test_cp_als.cpp:189-205
    s = rng.Substream(33)
    for _ in range(10):
        t = (s.uniform01_array(27) * 2 - 1).reshape((3, 3, 3), order="F")
        factors = [s.fill_uniform(3, 2) for _ in range(3)]
        for mode in range(3):
            got = O.als_solve_mode(O.matricize(t, mode), factors, mode)
            want = _oracle_mode_update(t, factors, mode)
            assert np.max(np.abs(got - want)) < 1e-8


def test_model_fit_known_answer():  # test_cp_als.cpp:229-252
    e1 = np.zeros(2)
    e1[0] = 1.0
    point = O.KruskalModel([e1[:, None].copy() for _ in range(3)], np.array([9.0]))
    target = np.zeros((2, 2, 2))
    target[0, 0, 0] = 10.0
    assert abs(O.model_fit(target, point) - 0.9) < 1e-12


# --- recovery.cpp (tests/test_recovery.cpp) ---------------------------------

def test_greedy_vs_exhaustive():  # test_recovery.cpp:49-70
    s = rng.Substream(1)
    for _ in range(50):
        r = 2 + int(s.uniform01() * 4.99)
        truth = list(range(r))
        for i in range(r - 1, 0, -1):
            j = int(s.uniform01() * (i + 1))
            truth[i], truth[j] = truth[j], truth[i]
        sim = np.zeros((r, r))
        for i in range(r):
            for j in range(r):
                sim[i, j] = 0.8 + 0.2 * s.uniform01() if truth[i] == j else 0.6 * s.uniform01()
        g = O.greedy_match(sim)
        assert g == O.exhaustive_match(sim) == truth


def test_greedy_ties_lowest_index():  # test_recovery.cpp:72-79
    log = []
    assert O.greedy_match(np.full((2, 2), 0.5), 1e-9, log) == [0, 1]
    assert log


def _random_normal_model(dims, rank, seed):
    m = random_truth(dims, rank, seed)
    m.normalize()
    return m


def test_align_identical_and_permutation():  # test_recovery.cpp:81-122
    rs = O.gen_replicas([6, 5], 4, 3, 2, 7)
    O.extend_temporal(rs, 4)
    m = _random_normal_model([4, 4, 4], 3, 9)
    st = O.align_replicas([m, m, m], rs)
    for rep in range(3):
        assert st.perms[rep] == [0, 1, 2]
        for sc in st.scales[rep]:
            assert np.allclose(sc, 1.0, rtol=1e-12)
    rs = O.gen_replicas([6, 5], 4, 2, 2, 7)
    O.extend_temporal(rs, 4)
    ref = _random_normal_model([4, 4, 4], 3, 9)
    perm = [2, 0, 1]
    sh = O.KruskalModel([f.copy() for f in ref.factors], ref.lambda_.copy())
    for n in range(3):
        for c in range(3):
            sh.factors[n][:, perm[c]] = ref.factors[n][:, c]
    for c in range(3):
        sh.lambda_[perm[c]] = ref.lambda_[c]
    st = O.align_replicas([ref, sh], rs)
    assert st.perms[1] == perm
    for n in range(3):
        assert np.max(np.abs(st.stacks[n][:4] - st.stacks[n][4:])) < 1e-9


def test_align_rejects_missing_shared():  # test_recovery.cpp:161-166
    rs = O.gen_replicas([6, 5], 4, 2, 0, 7)
    O.extend_temporal(rs, 4)
    m = _random_normal_model([4, 4, 4], 2, 9)
    with pytest.raises(O.ConfigError):
        O.align_replicas([m, m], rs)


def test_stacked_projection_full_rank():  # test_recovery.cpp:185-192
    rs = O.gen_replicas([50, 50], 30, 20, 5, 4)
    proj = O.stack_projections(rs, 0)
    assert proj.shape == (600, 50)
    assert O.colpiv_qr_rank(proj, 1e-10) == 50


def test_recover_nontemporal_known_answers():  # test_recovery.cpp:194-222
    s = rng.Substream(3)
    stack = s.fill_uniform(4, 2)
    a = O.recover_nontemporal(stack, np.eye(4), 0)
    assert np.max(np.abs(a - stack)) < 1e-12
    proj = s.fill_uniform(12, 5)
    truth = s.fill_uniform(5, 3)
    solved = O.recover_nontemporal(proj @ truth, proj, 0)
    for c in range(3):
        assert np.linalg.norm(solved[:, c] - truth[:, c]) <= 1e-8 * np.linalg.norm(truth[:, c])


def test_recover_nontemporal_rejects_deficient():  # test_recovery.cpp:224-236
    rs = O.gen_replicas([4, 4], 2, 3, 2, 8)
    with pytest.raises(O.NumericError, match=r"rank-deficient projection on mode 1 \(rank 2 of 4\)"):
        O.recover_nontemporal(np.ones((6, 2)), O.stack_projections(rs, 0), 0)
    thin = O.gen_replicas([10, 10], 2, 2, 1, 8)
    with pytest.raises(O.NumericError, match=r"projection is 4x10"):
        O.recover_nontemporal(np.ones((4, 2)), O.stack_projections(thin, 0), 0)


def test_kruskal_check_and_replica_bound():  # test_recovery.cpp:255-268; acceptance.cpp criterion 4
    assert O.kruskal_check(30, [5, 5, 5], 5)
    assert not O.kruskal_check(1, [1, 1, 1], 1)
    assert O.kruskal_check(4, [4, 4, 4], 5)
    assert not O.kruskal_check(4, [4, 4, 3], 5)
    assert O.replica_bound(1000, 1000, 100, 50, 10) == 25
    assert O.replica_bound(30, 30, 30, 30, 0) == 1
    with pytest.raises(O.ConfigError):
        O.replica_bound(10, 10, 10, 5, 5)


def test_memory_account_known_answer():  # test_eval.cpp:88-102
    cfg = O.StreamConfig(rank=5, p=20, q=30)
    # T = 100 split over two non-temporal modes, t_old = t_new = 5:
    # 600*(2000 + 5 + 5) + 105*5 + 27000 = 1,233,525
    sm = O.memory_account(cfg, [50, 50], 5, 5)
    assert sm["formula_elements"] == 1233525
    assert sm["predicted_summary_elements"] == 20 * 27000
    assert sm["predicted_elements"] == (sm["predicted_replica_elements"] + sm["predicted_summary_elements"] +
                                        sm["predicted_factor_elements"] + sm["predicted_accumulator_elements"])
    assert sm["ratio"] == pytest.approx(sm["predicted_elements"] / 1233525.0)
    with pytest.raises(O.ConfigError):
        O.memory_account(O.StreamConfig(rank=0, p=20, q=30), [50, 50], 5, 5)


def test_measured_footprint_matches_accounting():  # test_eval.cpp:104-126
    truth = random_truth([10, 9, 12], 2, 31)
    full = O.reconstruct_fast(truth)
    cfg = O.StreamConfig(rank=2, p=4, q=6, shared=2, seed=7, als=O.AlsConfig(2, 120, 1e-8, 3, 0))
    st = O.init_stream(O.slice_mode(full, 2, 0, 6), cfg)
    O.ingest_batch(st, O.slice_mode(full, 2, 6, 6))
    fp = O.measure_footprint(st)
    assert fp["summary_bytes"] == 8 * 4 * 6 * 6 * 6
    assert fp["replica_bytes"] == 8 * 4 * 6 * (10 + 9)
    assert fp["accumulator_bytes"] == 8 * 4 * 6 * 2
    assert fp["factor_bytes"] == 8 * (2 * (10 + 9 + 12) + 2)


def test_match_columns_known_gauge():  # test_recovery.cpp:304-337
    s = rng.Substream(66)
    stored = []
    for d in (6, 5):
        f = s.fill_uniform(d, 3)
        stored.append(f / np.linalg.norm(f, axis=0))
    perm = [2, 0, 1]
    flips = [[-1, 1, -1], [1, -1, 1]]
    stretch = [[2.0, 0.5, 3.0], [1.5, 1.0, 0.25]]
    current = []
    for n in range(2):
        f = np.zeros_like(stored[n])
        for c in range(3):
            f[:, perm[c]] = stored[n][:, c] * flips[n][c] * stretch[n][c]
        current.append(f)
    gm = O.match_columns(current, stored)
    assert gm.perm == perm
    for n in range(2):
        assert gm.signs[n].tolist() == flips[n]
        assert np.allclose(gm.norms[n], stretch[n])


def test_temporal_append_first_batch_plain_solve():  # test_recovery.cpp:282-302
    truth = _random_normal_model([8, 7, 5], 2, 3)
    t = O.reconstruct(truth)
    rs = O.gen_replicas([8, 7], 5, 3, 2, 41)
    O.extend_temporal(rs, 5)
    models = []
    for r in range(3):
        cfg = O.AlsConfig(rank=2, seed=rng.derive(8, [r]), max_iters=400, rel_tol=1e-12)
        models.append(O.cp_als(O.compress(t, rs, r, 0, 5), cfg).model)
    st = O.align_replicas(models, rs)
    summ = O.init_summaries(rs)
    res = O.recover_temporal_append(st.stacks[2], rs, summ, np.zeros((0, 2)), 5)
    direct = O.recover_nontemporal(st.stacks[2], O.stack_projections(rs, 2, 0, 5), 2)
    assert np.max(np.abs(res.new_rows - direct)) < 1e-12
    assert res.solve_residual < 1e-6


# --- streaming.cpp (tests/test_streaming.cpp, acceptance.cpp) ----------------

def _desk(rank, p, q, shared, seed):
    return O.StreamConfig(rank=rank, p=p, q=q, shared=shared, seed=seed,
                          als=O.AlsConfig(max_iters=300, rel_tol=1e-12, n_restarts=2), workers=1)


def test_noiseless_stream_tracks():  # test_streaming.cpp:78-96
    truth = random_truth([30, 30, 20], 4, 91)
    full = O.reconstruct(truth)
    st = O.init_stream(O.slice_mode(full, 2, 0, 5), _desk(4, 6, 15, 3, 17))
    for b in range(1, 4):
        O.ingest_batch(st, O.slice_mode(full, 2, 5 * b, 5))
    assert st.slices_seen == 20
    assert O.fitness(full, O.reconstruct(st.model)) >= 95.0
    assert min(O.congruence(truth, st.model)) >= 0.99


def test_history_telescopes():  # test_recovery.cpp:270-280 (history accumulators)
    truth = _random_normal_model([10, 9, 12], 2, 5)
    full = O.reconstruct(truth)
    cfg = O.StreamConfig(rank=2, p=4, q=6, shared=2, seed=1001,
                         als=O.AlsConfig(max_iters=400, rel_tol=1e-13), workers=1)
    st = O.init_stream(O.slice_mode(full, 2, 0, 4), cfg)
    O.ingest_batch(st, O.slice_mode(full, 2, 4, 4))
    O.ingest_batch(st, O.slice_mode(full, 2, 8, 4))
    shadow = O.gen_replicas([10, 9], 6, 4, 2, 1001, 2)
    for _ in range(3):
        O.extend_temporal(shadow, 4)
    c_raw = st.model.factors[2] * st.model.lambda_[None, :]
    for r in range(4):
        expected = shadow.replicas[r].temporal.T @ c_raw
        assert np.max(np.abs(expected - st.summaries.history[r])) < 1e-8


def test_config_failures_reproduce_reference_errors():
    # c1 shape: P*Q = 80 < I = 100 -> recover: NumericError
    x = random_tensor((100, 100, 10), 1)
    cfg = O.StreamConfig(rank=5, p=4, q=20, shared=4, seed=3, als=O.AlsConfig(max_iters=5))
    with pytest.raises(O.NumericError, match=r"recover: mode 1 projection is 80x100"):
        O.init_stream(x, cfg)
    with pytest.raises(O.ConfigError, match="tensor order must be >= 3"):
        O.init_stream(np.ones((4, 4)), _desk(2, 2, 3, 1, 5))
    with pytest.raises(O.ConfigError, match="need p >= 2"):
        c = _desk(5, 1, 30, 5, 11)
        c.enforce_bounds = True
        O.init_stream(O.reconstruct(random_truth([50, 50, 5], 5, 1)), c)


def test_ingest_wraps_batch_context():  # streaming.cpp:336-345
    truth = random_truth([10, 9, 8], 2, 5)
    full = O.reconstruct(truth)
    st = O.init_stream(O.slice_mode(full, 2, 0, 4), _desk(2, 4, 6, 2, 3))
    with pytest.raises(O.ConfigError, match="extent mismatch on mode 2 at batch 1"):
        O.ingest_batch(st, np.zeros((10, 7, 2)))
