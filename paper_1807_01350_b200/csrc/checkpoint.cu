// OCTS checkpoints of a device-resident stream, in the
// reference's byte format (proj/src/checkpoint.cpp:12-295): "OCTS", u32
// version 1, u64 payload length, u64 CRC-64/ECMA-182 (bit-reflected) of the
// payload, then config, replicas (with the empty temporal window), summaries
// + history accumulators, model, slices seen and the deterministic BatchRecord
// fields, native-endian.  save() reads the device state back; load() rebuilds
// a Stream whose device state holds the loaded values, so a resumed stream
// ingests exactly as the saved one would.  A checkpoint written by the
// reference (or the oracle port) loads here and vice versa.
#include <cuda_runtime.h>

#include <array>
#include <cstring>
#include <string>
#include <vector>

#include "errors.hpp"
#include "stream.hpp"

namespace octen {

namespace {

constexpr std::uint32_t kVersion = 1;
constexpr char kMagic[4] = {'O', 'C', 'T', 'S'};

// CRC-64/ECMA-182, bit-reflected (checkpoint.cpp:17-31)
std::uint64_t crc64(const std::uint8_t* data, std::size_t len) {
    static const std::array<std::uint64_t, 256> table = [] {
        std::array<std::uint64_t, 256> t{};
        constexpr std::uint64_t poly = 0xC96C5795D7870F42ULL;
        for (std::uint32_t i = 0; i < 256; ++i) {
            std::uint64_t c = i;
            for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1) ? poly : 0);
            t[i] = c;
        }
        return t;
    }();
    std::uint64_t c = ~0ULL;
    for (std::size_t i = 0; i < len; ++i) c = table[(c ^ data[i]) & 0xFF] ^ (c >> 8);
    return ~c;
}

struct Out {
    std::vector<std::uint8_t> b;
    void raw(const void* p, size_t n) {
        const auto* q = static_cast<const std::uint8_t*>(p);
        b.insert(b.end(), q, q + n);
    }
    void u8(std::uint8_t v) { b.push_back(v); }
    void u32(std::uint32_t v) { raw(&v, 4); }
    void u64(std::uint64_t v) { raw(&v, 8); }
    void i64(std::int64_t v) { raw(&v, 8); }
    void f64(double v) { raw(&v, 8); }
    // Matrix: i64 rows, i64 cols, column-major doubles
    void matrix(std::int64_t rows, std::int64_t cols, const double* d) {
        i64(rows);
        i64(cols);
        raw(d, sizeof(double) * (size_t)(rows * cols));
    }
};

struct In {
    const std::uint8_t* d;
    size_t n, pos = 0;
    void raw(void* p, size_t k) {
        if (pos + k > n) throw IoError("checkpoint: truncated payload");
        std::memcpy(p, d + pos, k);
        pos += k;
    }
    template <class T>
    T get() {
        T v;
        raw(&v, sizeof v);
        return v;
    }
    std::vector<double> matrix(std::int64_t& rows, std::int64_t& cols) {
        rows = get<std::int64_t>();
        cols = get<std::int64_t>();
        if (rows < 0 || cols < 0) throw IoError("checkpoint: negative matrix extent");
        std::vector<double> v((size_t)(rows * cols));
        raw(v.data(), sizeof(double) * v.size());
        return v;
    }
};

void expect(bool ok, const char* what) {
    if (!ok) throw IoError(std::string("checkpoint: ") + what);
}

}  // namespace

std::vector<std::uint8_t> Stream::checkpoint_save() {
    if (shard_world != 1) throw ConfigError("octen: checkpoints hold every replica (unsharded streams only)");
    if (!initialized) throw ConfigError("octen: stream is not initialised");
    sync();
    const int P = cfg.p, Q = cfg.q, R = cfg.rank, sh = cfg.shared;
    const size_t q3 = (size_t)Q * Q * Q;
    std::vector<double> y = Y.to_host((size_t)P * q3, st);
    std::vector<double> hs = hist.to_host((size_t)P * Q * R, st);
    std::vector<double> a = A.to_host((size_t)I * R, st), b = B.to_host((size_t)J * R, st);
    std::vector<double> c((size_t)K * R), l = lam.to_host((size_t)R, st);
    if (K > 0)
        OCTEN_CUDA(cudaMemcpy2DAsync(c.data(), K * sizeof(double), C.p, capC * sizeof(double), K * sizeof(double), R,
                                     cudaMemcpyDeviceToHost, st));
    OCTEN_CUDA(cudaStreamSynchronize(st));

    Out w;
    // config (checkpoint.cpp:125-143)
    w.u32((std::uint32_t)cfg.rank);
    w.u32((std::uint32_t)cfg.p);
    w.u32((std::uint32_t)cfg.q);
    w.u32((std::uint32_t)cfg.shared);
    w.u32((std::uint32_t)cfg.temporal_mode);
    w.u64(cfg.seed);
    w.u8(cfg.enforce_bounds ? 1 : 0);
    w.u32(0);  // workers: not stream state
    w.u8(cfg.strict ? 1 : 0);
    w.f64(cfg.residual_warning);
    w.u32((std::uint32_t)cfg.rank);  // als.rank (init_stream sets it to the stream rank)
    w.u32((std::uint32_t)cfg.als_max_iters);
    w.f64(cfg.als_rel_tol);
    w.u32((std::uint32_t)cfg.als_n_restarts);
    w.u64(cfg.als_seed);
    // replicas (checkpoint.cpp:168-184): the temporal window is empty at rest
    w.u64(cfg.seed);
    w.u32((std::uint32_t)Q);
    w.u32((std::uint32_t)sh);
    w.u32((std::uint32_t)cfg.temporal_mode);
    w.i64(batches_drawn);
    w.u64(2);
    w.i64(I);
    w.i64(J);
    w.matrix(sh, sh, tgram.data());
    w.u32((std::uint32_t)P);
    for (int p = 0; p < P; ++p) {
        w.u32((std::uint32_t)p);
        w.u64(2);
        w.matrix(I, Q, hU.data() + (size_t)p * I * Q);
        w.matrix(J, Q, hV.data() + (size_t)p * J * Q);
        w.i64(K);  // temporal_window_start
        w.i64(K);  // temporal_rows_total
        w.matrix(0, Q, nullptr);
    }
    // summaries and history (checkpoint.cpp:186-193); history is kept
    // stacked (p Q x R) on the device
    w.i64(batches_seen);
    w.u64((std::uint64_t)P);
    std::vector<double> hb((size_t)Q * R);
    for (int p = 0; p < P; ++p) {
        w.u64(3);
        for (int k = 0; k < 3; ++k) w.i64(Q);
        w.u64(q3);
        w.raw(y.data() + (size_t)p * q3, sizeof(double) * q3);
        for (int r = 0; r < R; ++r)
            for (int a2 = 0; a2 < Q; ++a2) hb[a2 + (size_t)Q * r] = hs[(size_t)p * Q + a2 + (size_t)P * Q * r];
        w.matrix(Q, R, hb.data());
    }
    // model, slices seen, log (checkpoint.cpp:195-211)
    w.u32(3);
    {  // factors in the stream's mode order
        const std::vector<double>* fs[3] = {&a, &b, &c};
        const std::int64_t rows[3] = {I, J, K};
        for (int n = 0; n < 3; ++n) {
            const int sl = factor_slot(n);
            w.matrix(rows[sl], R, fs[sl]->data());
        }
    }
    w.i64(R);
    w.raw(l.data(), sizeof(double) * R);
    w.i64(K);
    w.u64(log.size());
    for (const BatchRecordC& r : log) {
        w.i64(r.batch_index);
        w.i64(r.t_new);
        w.f64(r.temporal_residual);
        w.f64(r.min_match_similarity);
        w.f64(r.max_offdiag_similarity);
        w.u8(r.warned ? 1 : 0);
    }
    std::vector<std::uint8_t> out(kMagic, kMagic + 4);
    Out h;
    h.u32(kVersion);
    h.u64(w.b.size());
    h.u64(crc64(w.b.data(), w.b.size()));
    out.insert(out.end(), h.b.begin(), h.b.end());
    out.insert(out.end(), w.b.begin(), w.b.end());
    return out;
}

std::unique_ptr<Stream> Stream::checkpoint_load(const std::uint8_t* bytes, size_t n, int device) {
    // checkpoint.cpp:222-295: header checks in the reference's order
    if (n < 24 || std::memcmp(bytes, kMagic, 4) != 0) throw IoError("checkpoint: bad magic");
    In head{bytes + 4, 20};
    const std::uint32_t version = head.get<std::uint32_t>();
    if (version != kVersion) throw IoError("checkpoint: unsupported format version " + std::to_string(version));
    const std::uint64_t len = head.get<std::uint64_t>();
    const std::uint64_t crc = head.get<std::uint64_t>();
    if (n != 24 + len) throw IoError("checkpoint: payload length mismatch (corrupt or truncated)");
    if (crc64(bytes + 24, len) != crc) throw IoError("checkpoint: checksum mismatch");
    In r{bytes + 24, (size_t)len};

    StreamCfg c;
    c.rank = (int)r.get<std::uint32_t>();
    c.p = (int)r.get<std::uint32_t>();
    c.q = (int)r.get<std::uint32_t>();
    c.shared = (int)r.get<std::uint32_t>();
    c.temporal_mode = (int)r.get<std::uint32_t>();
    c.seed = r.get<std::uint64_t>();
    c.enforce_bounds = r.get<std::uint8_t>() != 0;
    c.workers = (int)r.get<std::uint32_t>();
    c.strict = r.get<std::uint8_t>() != 0;
    c.residual_warning = r.get<double>();
    (void)r.get<std::uint32_t>();  // als.rank
    c.als_max_iters = (int)r.get<std::uint32_t>();
    c.als_rel_tol = r.get<double>();
    c.als_n_restarts = (int)r.get<std::uint32_t>();
    c.als_seed = r.get<std::uint64_t>();
    c.device = device;

    const std::uint64_t rseed = r.get<std::uint64_t>();
    const int q = (int)r.get<std::uint32_t>(), sh = (int)r.get<std::uint32_t>();
    const int tmode = (int)r.get<std::uint32_t>();
    const std::int64_t drawn = r.get<std::int64_t>();
    const std::uint64_t ndims = r.get<std::uint64_t>();
    expect(ndims == 2 && tmode >= 0 && tmode <= 2 && tmode == c.temporal_mode && q == c.q && sh == c.shared &&
               rseed == c.seed,
           "the device path holds order-3 streams");
    const std::int64_t I = r.get<std::int64_t>(), J = r.get<std::int64_t>();
    std::int64_t rows, cols;
    std::vector<double> tg = r.matrix(rows, cols);
    expect(rows == sh && cols == sh, "temporal shared Gram shape");
    const std::uint32_t P = r.get<std::uint32_t>();
    expect((int)P == c.p, "replica count");
    const int Q = c.q, R = c.rank;
    std::vector<double> hU((size_t)P * I * Q), hV((size_t)P * J * Q);
    std::int64_t K = -1;
    for (std::uint32_t p = 0; p < P; ++p) {
        expect(r.get<std::uint32_t>() == p, "replica order");
        expect(r.get<std::uint64_t>() == 2, "replica projections");
        std::vector<double> u = r.matrix(rows, cols);
        expect(rows == I && cols == Q, "projection shape");
        std::memcpy(hU.data() + (size_t)p * I * Q, u.data(), u.size() * sizeof(double));
        std::vector<double> v = r.matrix(rows, cols);
        expect(rows == J && cols == Q, "projection shape");
        std::memcpy(hV.data() + (size_t)p * J * Q, v.data(), v.size() * sizeof(double));
        const std::int64_t ws = r.get<std::int64_t>(), tot = r.get<std::int64_t>();
        (void)r.matrix(rows, cols);
        expect(rows == 0 && ws == tot, "a stream between batches has an empty temporal window");
        K = tot;
    }
    const std::int64_t seen = r.get<std::int64_t>();
    expect(r.get<std::uint64_t>() == P, "summary count");
    const size_t q3 = (size_t)Q * Q * Q;
    std::vector<double> y((size_t)P * q3), hs((size_t)P * Q * R, 0.0);
    for (std::uint32_t p = 0; p < P; ++p) {
        expect(r.get<std::uint64_t>() == 3, "summary order");
        for (int k = 0; k < 3; ++k) expect(r.get<std::int64_t>() == Q, "summary shape");
        expect(r.get<std::uint64_t>() == q3, "summary size");
        r.raw(y.data() + (size_t)p * q3, sizeof(double) * q3);
        std::vector<double> h = r.matrix(rows, cols);
        expect((rows == Q && cols == R) || (rows * cols == 0), "history shape");
        if (rows * cols)
            for (int rr = 0; rr < R; ++rr)
                for (int a2 = 0; a2 < Q; ++a2) hs[(size_t)p * Q + a2 + (size_t)P * Q * rr] = h[a2 + (size_t)Q * rr];
    }
    expect(r.get<std::uint32_t>() == 3, "model order");
    std::vector<double> fsl[3];  // by slot: A, B, C
    {
        const std::int64_t want[3] = {I, J, K};
        for (int n = 0; n < 3; ++n) {
            const int sl = n == tmode ? 2 : (n < tmode ? n : n - 1);
            fsl[sl] = r.matrix(rows, cols);
            expect(rows == want[sl] && cols == R, "factor shape");
        }
    }
    std::vector<double>& a = fsl[0];
    std::vector<double>& b = fsl[1];
    std::vector<double>& cm = fsl[2];
    expect(r.get<std::int64_t>() == R, "lambda length");
    std::vector<double> l(R);
    r.raw(l.data(), sizeof(double) * R);
    expect(r.get<std::int64_t>() == K, "slices seen");
    const std::uint64_t nlog = r.get<std::uint64_t>();
    std::vector<BatchRecordC> lg(nlog);
    for (auto& rec : lg) {
        rec = BatchRecordC{};
        rec.batch_index = r.get<std::int64_t>();
        rec.t_new = r.get<std::int64_t>();
        rec.temporal_residual = r.get<double>();
        rec.min_match_similarity = r.get<double>();
        rec.max_offdiag_similarity = r.get<double>();
        rec.warned = r.get<std::uint8_t>() != 0;
    }
    if (r.pos != r.n) throw IoError("checkpoint: trailing bytes after payload");

    // a stream whose device state holds the loaded values
    auto s = std::make_unique<Stream>(c);
    s->validate(3);
    s->I = I;
    s->J = J;
    s->hU = std::move(hU);
    s->hV = std::move(hV);
    s->tgram = std::move(tg);
    s->batches_drawn = drawn;
    if (s->pl > 0) {
        s->comp.set_projections(s->pl, Q, sh, I, J, s->hU.data(), s->hV.data(), s->st);
        s->comp.set_temporal_mode(tmode);
    }
    s->merge.set_projections(c.p, Q, sh, R, I, J, s->hU.data(), s->hV.data(), s->st);
    s->set_mode_strides();
    s->Y.upload(y.data(), y.size(), s->st);
    s->hist.upload(hs.data(), hs.size(), s->st);
    s->A.upload(a.data(), a.size(), s->st);
    s->B.upload(b.data(), b.size(), s->st);
    s->lam.upload(l.data(), l.size(), s->st);
    s->K = 0;
    s->ensure_c_capacity(std::max<std::int64_t>(K, 1), s->st);
    if (K > 0)
        OCTEN_CUDA(cudaMemcpy2DAsync(s->C.p, s->capC * sizeof(double), cm.data(), K * sizeof(double),
                                     K * sizeof(double), R, cudaMemcpyHostToDevice, s->st));
    s->K = K;
    s->batches_seen = seen;
    s->log = std::move(lg);
    s->initialized = true;
    OCTEN_CUDA(cudaStreamSynchronize(s->st));
    return s;
}

}  // namespace octen
