// The reference's streaming tests (proj/tests/test_streaming.cpp) restated
// against the C++ host mirror include/cpstream_b200.hpp, i.e. through the
// C-ABI and the B200 kernels.  Test infrastructure: built by
// tests/test_cpp_shim.py (compile + link on CPU, run with -m gpu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "cpstream_b200.hpp"
#include "rng_host.hpp"

using namespace cpstream_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_fail;                                                                 \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                             \
    } while (0)

template <class E>
static bool throws_as(const std::function<void()>& f, const char* contains = nullptr) {
    try {
        f();
    } catch (const E& e) {
        return contains == nullptr || std::string(e.what()).find(contains) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

namespace {

// test_streaming.cpp:14-24 (rng::Substream fill_uniform, lambda = 1)
KruskalModel random_truth(const std::vector<std::int64_t>& dims, int rank, std::uint64_t seed) {
    octen::rng::Substream s(seed);
    KruskalModel m;
    for (std::int64_t d : dims) {
        Matrix f(d, rank);
        s.fill_uniform(f.data(), d, rank, d);
        m.factors.push_back(f);
    }
    m.lambda.assign((size_t)rank, 1.0);
    return m;
}

// cp_als.cpp:361-367 (3-mode)
DenseTensor reconstruct(const KruskalModel& m) {
    const std::int64_t I = m.factors[0].rows(), J = m.factors[1].rows(), K = m.factors[2].rows();
    DenseTensor t = DenseTensor::zeros({I, J, K});
    for (int r = 0; r < m.rank(); ++r)
        for (std::int64_t k = 0; k < K; ++k)
            for (std::int64_t j = 0; j < J; ++j) {
                const double s = m.lambda[(size_t)r] * m.factors[2](k, r) * m.factors[1](j, r);
                for (std::int64_t i = 0; i < I; ++i) t.data[(size_t)(i + I * (j + J * k))] += s * m.factors[0](i, r);
            }
    return t;
}

// tensor.cpp:275-293 on the last mode
DenseTensor slice_last(const DenseTensor& t, std::int64_t start, std::int64_t count) {
    const std::int64_t plane = t.dims[0] * t.dims[1];
    std::vector<double> d(t.data.begin() + plane * start, t.data.begin() + plane * (start + count));
    return DenseTensor({t.dims[0], t.dims[1], count}, d);
}

// eval.cpp:10-20
double fitness(const DenseTensor& x, const DenseTensor& xh) {
    double nx = 0, nd = 0;
    for (size_t e = 0; e < x.data.size(); ++e) {
        nx += x.data[e] * x.data[e];
        nd += (x.data[e] - xh.data[e]) * (x.data[e] - xh.data[e]);
    }
    return 100.0 * (1.0 - std::sqrt(nd) / std::sqrt(nx));
}

// eval.cpp:22-46 (greedy matching of the per-component product of |cos|)
std::vector<double> congruence(const KruskalModel& g, const KruskalModel& e) {
    const int R = g.rank();
    std::vector<double> sim((size_t)R * R, 1.0);
    for (size_t m = 0; m < g.factors.size(); ++m)
        for (int a = 0; a < R; ++a)
            for (int b = 0; b < R; ++b) {
                double ab = 0, aa = 0, bb = 0;
                for (std::int64_t i = 0; i < g.factors[m].rows(); ++i) {
                    ab += g.factors[m](i, a) * e.factors[m](i, b);
                    aa += g.factors[m](i, a) * g.factors[m](i, a);
                    bb += e.factors[m](i, b) * e.factors[m](i, b);
                }
                sim[(size_t)(a + R * b)] *= std::fabs(ab) / std::sqrt(aa * bb);
            }
    std::vector<double> out((size_t)R, 0.0);
    std::vector<char> ua((size_t)R, 0), ub((size_t)R, 0);
    for (int step = 0; step < R; ++step) {
        int ba = -1, bb = -1;
        double best = -1;
        for (int a = 0; a < R; ++a)
            for (int b = 0; b < R; ++b)
                if (!ua[(size_t)a] && !ub[(size_t)b] && sim[(size_t)(a + R * b)] > best) {
                    best = sim[(size_t)(a + R * b)];
                    ba = a;
                    bb = b;
                }
        ua[(size_t)ba] = ub[(size_t)bb] = 1;
        out[(size_t)ba] = best;
    }
    return out;
}

// test_streaming.cpp:26-38
StreamConfig desk_config(int rank, int p, int q, int shared, std::uint64_t seed) {
    StreamConfig cfg;
    cfg.rank = rank;
    cfg.p = p;
    cfg.q = q;
    cfg.shared = shared;
    cfg.seed = seed;
    cfg.als.max_iters = 300;
    cfg.als.rel_tol = 1e-12;
    cfg.als.n_restarts = 2;
    cfg.workers = 1;
    return cfg;
}

}  // namespace

int main() {
    // TEST_CASE("init_stream on the reference configuration")
    {
        const KruskalModel truth = random_truth({50, 50, 5}, 5, 2024);
        const DenseTensor first = reconstruct(truth);
        const StreamState st = init_stream(first, desk_config(5, 20, 30, 5, 11));
        CHECK(st.slices_seen == 5);
        CHECK(fitness(first, reconstruct(st.model)) >= 90.0);
        CHECK(st.log.size() == 1);
    }
    {
        const DenseTensor first = reconstruct(random_truth({50, 50, 5}, 5, 1));
        StreamConfig cfg = desk_config(5, 1, 30, 5, 11);
        cfg.enforce_bounds = true;
        CHECK(throws_as<ConfigError>([&] { init_stream(first, cfg); }, "need p >= 2"));
    }
    {
        const DenseTensor first = reconstruct(random_truth({6, 6, 4}, 4, 1));
        StreamConfig cfg = desk_config(4, 5, 2, 1, 11);  // sum min(Q, krank) = 6 < 10
        cfg.enforce_bounds = true;
        CHECK(throws_as<ConfigError>([&] { init_stream(first, cfg); }));
    }
    {
        const DenseTensor first = reconstruct(random_truth({8, 8, 1}, 2, 3));
        const StreamState st = init_stream(first, desk_config(2, 4, 5, 2, 7));
        CHECK(st.slices_seen == 1);
        CHECK(st.model.factors[2].rows() == 1);
    }
    {
        DenseTensor flat({4, 4}, std::vector<double>(16, 1.0));
        CHECK(throws_as<ConfigError>([&] { init_stream(flat, desk_config(2, 2, 3, 1, 5)); }));
    }
    // TEST_CASE("noiseless stream tracks the batch decomposition")
    {
        const KruskalModel truth = random_truth({30, 30, 20}, 4, 91);
        const DenseTensor full = reconstruct(truth);
        StreamState st = init_stream(slice_last(full, 0, 5), desk_config(4, 6, 15, 3, 17));
        for (int b = 1; b < 4; ++b) ingest_batch(st, slice_last(full, 5 * b, 5));
        CHECK(st.slices_seen == 20);
        CHECK(st.model.factors[2].rows() == 20);
        CHECK(fitness(full, reconstruct(st.model)) >= 95.0);
        for (double sc : congruence(truth, st.model)) CHECK(sc >= 0.99);
        CHECK(st.log.size() == 4);
        CHECK(st.log.back().batch_index == 3);
    }
    // TEST_CASE("zero batch leaves the factors essentially unchanged")
    {
        const KruskalModel truth = random_truth({12, 10, 8}, 2, 5);
        const DenseTensor full = reconstruct(truth);
        StreamState st = init_stream(slice_last(full, 0, 8), desk_config(2, 4, 6, 2, 3));
        const KruskalModel before = st.model;
        ingest_batch(st, DenseTensor::zeros({12, 10, 2}));
        KruskalModel bnt, ant;
        bnt.factors = {before.factors[0], before.factors[1]};
        bnt.lambda = {1.0, 1.0};
        ant.factors = {st.model.factors[0], st.model.factors[1]};
        ant.lambda = {1.0, 1.0};
        for (double sc : congruence(bnt, ant)) CHECK(sc >= 0.999);
        double mx = 0.0;
        const Matrix& c = st.model.factors[2];
        for (std::int64_t k = c.rows() - 2; k < c.rows(); ++k)
            for (int r = 0; r < 2; ++r) mx = std::max(mx, std::fabs(c(k, r) * st.model.lambda[(size_t)r]));
        CHECK(mx < 1e-6);
    }
    // TEST_CASE("wrong batch extents are rejected")
    {
        const DenseTensor full = reconstruct(random_truth({10, 9, 8}, 2, 5));
        StreamState st = init_stream(slice_last(full, 0, 4), desk_config(2, 4, 6, 2, 3));
        CHECK(throws_as<ConfigError>([&] { ingest_batch(st, DenseTensor::zeros({10, 7, 2})); }));
        CHECK(throws_as<ConfigError>([&] { ingest_batch(st, DenseTensor::zeros({10, 9, 8, 2})); }));
        // the stream is still usable after a rejected batch
        ingest_batch(st, slice_last(full, 4, 4));
        CHECK(st.slices_seen == 8);
    }
    // sparse batches (tensor.hpp:66-90, tensor.cpp:87-122): the device COO
    // compression equals compress(to_dense(batch)) done with the dense path,
    // and the SparseTensor errors keep their reference text
    {
        const std::int64_t I = 14, J = 11, t = 5, Q = 4;
        std::vector<Matrix> u, v, w;
        std::uint64_t s = 99;
        auto uni = [&s] {
            s = s * 6364136223846793005ULL + 1442695040888963407ULL;
            return (double)(s >> 11) * 0x1.0p-53;
        };
        for (int r = 0; r < 2; ++r) {
            Matrix a(I, Q), b(J, Q), c(t, Q);
            for (double& x : a.v) x = uni();
            for (double& x : b.v) x = uni();
            for (double& x : c.v) x = uni();
            u.push_back(a);
            v.push_back(b);
            w.push_back(c);
        }
        SparseTensor sp({I, J, t}, {});
        DenseTensor dense = DenseTensor::zeros({I, J, t});
        for (std::int64_t k = 0; k < t; ++k)
            for (std::int64_t i = 0; i < I; i += 3)
                for (std::int64_t j = (i + k) % 2; j < J; j += 2) {
                    const float val = (float)uni();
                    sp.entries.push_back({{i, j, k}, (double)val});
                    dense.data[(size_t)(i + I * j + I * J * k)] = (double)val;
                }
        CooSummaries cs(u, v);
        cs.compress(sp, w);
        const std::vector<DenseTensor> ys = cs.summaries();
        // the same contraction by triple loops (compression.cpp:108-130 on to_dense)
        double err = 0.0, nrm = 0.0;
        for (int r = 0; r < 2; ++r)
            for (std::int64_t a = 0; a < Q; ++a)
                for (std::int64_t b = 0; b < Q; ++b)
                    for (std::int64_t c = 0; c < Q; ++c) {
                        double z = 0.0;
                        for (std::int64_t k = 0; k < t; ++k)
                            for (std::int64_t j = 0; j < J; ++j)
                                for (std::int64_t i = 0; i < I; ++i)
                                    z += dense.data[(size_t)(i + I * j + I * J * k)] * u[r](i, a) * v[r](j, b) *
                                         w[r](k, c);
                        const double y = ys[(size_t)r].data[(size_t)(a + Q * b + Q * Q * c)];
                        err += (y - z) * (y - z);
                        nrm += z * z;
                    }
        CHECK(std::sqrt(err / nrm) < 1e-5);
        SparseTensor oob({I, J, t}, {{{0, 0, 0}, 1.0}, {{I, 0, 0}, 1.0}});
        CHECK(throws_as<ConfigError>([&] { cs.compress(oob, w); }, "SparseTensor: index out of bounds"));
        SparseTensor dup({I, J, t}, {{{1, 2, 3}, 1.0}, {{1, 2, 3}, 2.0}});
        CHECK(throws_as<ConfigError>([&] { cs.compress(dup, w); }, "SparseTensor: duplicate index"));
        SparseTensor nan({I, J, t}, {{{1, 2, 3}, std::nan("")}});
        CHECK(throws_as<NumericError>([&] { cs.compress(nan, w); }, "SparseTensor: non-finite value"));
        // a rejected batch leaves the summaries as they were
        const std::vector<DenseTensor> again = cs.summaries();
        CHECK(again[0].data == ys[0].data && again[1].data == ys[1].data);
    }
    // TEST_CASE("checkpoint round trips") (test_streaming.cpp:205-247)
    {
        const DenseTensor full = reconstruct(random_truth({9, 8, 10}, 2, 71));
        StreamState st = init_stream(slice_last(full, 0, 5), desk_config(2, 3, 6, 2, 53));
        const std::vector<std::uint8_t> bytes = checkpoint_save(st);
        CHECK(checkpoint_save(checkpoint_load(bytes)) == bytes);
        StreamState resumed = checkpoint_load(bytes);
        ingest_batch(st, slice_last(full, 5, 5));
        ingest_batch(resumed, slice_last(full, 5, 5));
        CHECK(checkpoint_save(st) == checkpoint_save(resumed));
        std::vector<std::uint8_t> bad = bytes;
        bad[bad.size() / 2] ^= 0x40;
        CHECK(throws_as<IoError>([&] { checkpoint_load(bad); }, "checksum mismatch"));
        bad = bytes;
        bad.resize(bad.size() - 7);
        CHECK(throws_as<IoError>([&] { checkpoint_load(bad); }, "payload length mismatch"));
    }
    // pipelined ingest == ingest_batch, byte for byte (the checkpoints)
    {
        const DenseTensor full = reconstruct(random_truth({12, 11, 12}, 3, 61));
        const StreamConfig cfg = desk_config(3, 5, 8, 3, 43);
        StreamState a = init_stream(slice_last(full, 0, 6), cfg);
        StreamState b = init_stream(slice_last(full, 0, 6), cfg);
        ingest_batch(a, slice_last(full, 6, 3));
        ingest_batch(a, slice_last(full, 9, 3));
        ingest_batch_async(b, slice_last(full, 6, 3));
        ingest_batch_async(b, slice_last(full, 9, 3));
        sync(b);
        CHECK(b.slices_seen == 12 && b.log.size() == 3);
        CHECK(checkpoint_save(a) == checkpoint_save(b));
    }
    // library-owned NCCL collectives, one rank: the unsharded stream's bits
    {
        const DenseTensor full = reconstruct(random_truth({14, 13, 12}, 2, 81));
        const StreamConfig cfg = desk_config(2, 4, 6, 2, 31);
        StreamState a = init_stream(slice_last(full, 0, 6), cfg);
        ingest_batch(a, slice_last(full, 6, 6));
        ShardedStream sh(cfg, 0, 1, ShardedStream::nccl_unique_id());
        sh.ingest(slice_last(full, 0, 6));
        sh.ingest(slice_last(full, 6, 6));
        CHECK(sh.state().slices_seen == 12);
        for (size_t m = 0; m < 3; ++m) CHECK(sh.state().model.factors[m].v == a.model.factors[m].v);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
