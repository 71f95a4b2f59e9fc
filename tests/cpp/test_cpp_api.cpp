// C++ drop-in check: reference-style tests written against include/vqkv/*.hpp
// (the mirror of proj/core/include/vqkv/*.hpp), running on the GPU through
// libvqkv_b200.so.  Each case follows a reference doctest (file:line noted).
// Prints one PASS/FAIL line per case; exit status = number of failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "vqkv/attention.hpp"
#include "vqkv/codebook.hpp"
#include "vqkv/kv_cache.hpp"

using namespace vqkv;

static int g_fail = 0;
static void report(bool ok, const char* name) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", name);
    if (!ok) ++g_fail;
}

static MatrixF rows(std::initializer_list<std::initializer_list<float>> r) {
    MatrixF m(int64_t(r.size()), int64_t(r.begin()->size()));
    int64_t i = 0;
    for (auto& row : r) {
        int64_t j = 0;
        for (float v : row) m(i, j++) = v;
        ++i;
    }
    return m;
}

static CodebookStack stack_from(std::vector<MatrixF> per_stage) {  // test_util.hpp:15-28
    CodebookStack st;
    for (auto& e : per_stage) {
        Codebook cb;
        cb.entries = e;
        cb.projection = MatrixF::Identity(e.cols(), e.cols());
        st.stages.push_back(cb);
    }
    return st;
}

static CodebookStack random_stack(std::mt19937_64& rng, size_t n, uint32_t s, int64_t d) {  // test_util.hpp:30-50
    std::normal_distribution<float> g(0.f, 1.f);
    CodebookStack st;
    const float ps = 1.0f / std::sqrt(float(d));
    for (size_t i = 0; i < n; ++i) {
        Codebook cb;
        cb.entries.resize(s, d);
        for (int64_t k = 0; k < cb.entries.size(); ++k) cb.entries.data()[k] = g(rng);
        cb.projection.resize(d, d);
        for (int64_t k = 0; k < cb.projection.size(); ++k) cb.projection.data()[k] = ps * g(rng);
        st.stages.push_back(cb);
    }
    return st;
}

static MatrixF random_matrix(std::mt19937_64& rng, int64_t r, int64_t c) {
    std::normal_distribution<float> g(0.f, 1.f);
    MatrixF m(r, c);
    for (int64_t k = 0; k < m.size(); ++k) m.data()[k] = g(rng);
    return m;
}

int main() {
    {  // codebook_test.cpp:35-42
        auto st = stack_from({rows({{0, 0}, {1, 0}, {0, 1}})});
        VectorF x{0.9f, 0.1f};
        auto r = nearest_entry(st.stages[0], x);
        report(r.index == 1 && std::fabs(r.distance - 0.14142136f) < 1e-4f, "nearest_entry picks the closest entry");
    }
    {  // codebook_test.cpp:52-57
        auto st = stack_from({rows({{1, 0}, {1, 0}})});
        VectorF x{1.0f, 0.0f};
        report(nearest_entry(st.stages[0], x).index == 0, "nearest_entry ties -> lowest index");
    }
    {  // codebook_test.cpp:90-103
        auto st = stack_from({rows({{1, 0}, {0, 1}}), rows({{0, 0.5f}, {0.5f, 0}})});
        VectorF x{1.2f, 0.4f};
        auto q = quantize(st, x);
        auto rec = reconstruct(st, q.codes);
        report(q.codes == CodeVector{0, 0} && std::fabs(q.final_residual[0] - 0.2f) < 1e-6f &&
                   std::fabs(q.final_residual[1] + 0.1f) < 1e-6f && std::fabs(rec[0] - 1.0f) < 1e-6f &&
                   std::fabs(rec[1] - 0.5f) < 1e-6f,
               "quantize walks the residual through both stages");
    }
    {  // codebook_test.cpp:138-143
        std::mt19937_64 rng(4);
        auto st = random_stack(rng, 2, 4, 3);
        bool ok = false;
        try {
            reconstruct(st, {0, 4});
        } catch (const InvalidCode&) {
            ok = true;
        }
        report(ok, "reconstruct rejects out-of-range codes (InvalidCode)");
    }
    {  // codebook_test.cpp:164-174 at the tensor-core shape (D = 128)
        std::mt19937_64 rng(7);
        auto st = random_stack(rng, 3, 256, 128);
        MatrixF xs = random_matrix(rng, 200, 128);
        auto b = quantize_batch(st, xs);
        bool ok = true;
        for (int64_t r = 0; r < xs.rows() && ok; r += 17) {
            VectorF x(128);
            std::memcpy(x.data(), xs.data() + r * 128, sizeof(float) * 128);
            auto q = quantize(st, x);
            ok = (b.codes.row(size_t(r)) == q.codes) && (b.residual_norms[r] == q.final_residual.norm() ||
                                                         std::fabs(b.residual_norms[r] - q.final_residual.norm()) < 1e-5f);
        }
        report(ok, "quantize_batch matches per-row quantize (D=128)");
        // codebook_test.cpp:188-210 partition invariance
        MatrixF full = reconstruct_block(st, b.codes, 0, 200);
        bool same = true;
        for (size_t beg = 0; beg < 200; beg += 33) {
            size_t end = std::min<size_t>(200, beg + 33);
            MatrixF part = reconstruct_block(st, b.codes, beg, end);
            same &= std::memcmp(part.data(), full.data() + beg * 128, sizeof(float) * (end - beg) * 128) == 0;
        }
        report(same, "reconstruct_block partitions are bit-identical");
    }
    {  // acceptance_test.cpp:184-220 (window accounting, smaller)
        std::mt19937_64 rng(1004);
        auto ks = random_stack(rng, 2, 16, 16);
        auto vs = random_stack(rng, 2, 16, 16);
        vs.cache_kind = CacheKind::value;
        CacheState state(ks, vs, WindowPolicy{4, 64, false});
        state.prefill(random_matrix(rng, 128, 16), random_matrix(rng, 128, 16));
        bool ok = state.total_len() == 128 && state.compressed_rows() == 60 && state.init_rows() == 4 &&
                  state.local_rows() == 64;
        for (size_t t = 0; t < 300; ++t) {
            MatrixF k = random_matrix(rng, 1, 16), v = random_matrix(rng, 1, 16);
            VectorF kk(16), vv(16);
            std::memcpy(kk.data(), k.data(), 64);
            std::memcpy(vv.data(), v.data(), 64);
            state.append_token(kk, vv);
            ok &= state.batched_compressions() == (t + 1) / 64;
        }
        report(ok && state.total_len() == 428, "window-policy accounting (deferred flushes)");
        // attention_test.cpp:54-65 streaming == monolithic over the logical view
        ViewBlock all = state.view_block(0, state.total_len());
        MatrixF qm = random_matrix(rng, 1, 16);
        VectorF q(16);
        std::memcpy(q.data(), qm.data(), 64);
        AttentionConfig cfg;
        VectorF a = attend(state, q, cfg);
        VectorF r = attend_raw(all.keys, all.values, q, cfg);
        float err = 0.f;
        for (int64_t i = 0; i < a.size(); ++i) err = std::max(err, std::fabs(a[i] - r[i]));
        report(err < 1e-4f, "attend over the compressed cache == attention over its logical view");
        AttendStats stats;
        cfg.block_rows = 4;
        attend(state, q, cfg, &stats);
        report(stats.reconstructed_rows == state.compressed_rows() && stats.peak_reconstructed_scalars <= 4 * 32,
               "attend stats follow the reference's block accounting");
    }
    {  // D = 128 cache: attend over the LUT kernel, fidelity (attention.cpp:90-134), VQKS snapshot round trip
        std::mt19937_64 rng(2024);
        auto ks = random_stack(rng, 8, 256, 128);
        auto vs = random_stack(rng, 4, 128, 128);
        vs.cache_kind = CacheKind::value;
        CacheState state(ks, vs, WindowPolicy{4, 32, false});
        MatrixF keys = random_matrix(rng, 300, 128), values = random_matrix(rng, 300, 128);
        state.prefill(keys, values);
        MatrixF qs = random_matrix(rng, 3, 128);
        AttentionConfig cfg;
        FidelityReport fr = fidelity(state, keys, values, qs, cfg);
        ViewBlock all = state.view_block(0, state.total_len());
        VectorF q0 = detail::row_of(qs, 0);
        VectorF a = attend(state, q0, cfg), r = attend_raw(all.keys, all.values, q0, cfg);
        float err = 0.f, mx = 1.f;
        for (int64_t i = 0; i < a.size(); ++i) err = std::max(err, std::fabs(a[i] - r[i])), mx = std::max(mx, std::fabs(r[i]));
        report(err <= mx / 128.f, "attend (G=4 LUT kernel) == attend_raw over the logical view (2^-7 tolerance)");
        {  // attention.cpp:104-115 query by query, from the same public calls
            double err = 0.0, cs = 0.0;
            for (int64_t i = 0; i < qs.rows(); ++i) {
                VectorF qi = detail::row_of(qs, i);
                VectorF c = attend(state, qi, cfg), w = attend_raw(keys, values, qi, cfg);
                double dot = 0.0, nc = 0.0, nw = 0.0;
                for (int64_t d = 0; d < c.size(); ++d) {
                    err = std::max(err, double(std::fabs(c[d] - w[d])));
                    dot += double(c[d]) * w[d];
                    nc += double(c[d]) * c[d];
                    nw += double(w[d]) * w[d];
                }
                cs += dot / (std::sqrt(nc) * std::sqrt(nw));
            }
            cs /= double(qs.rows());
            report(std::fabs(fr.output_max_abs_err - err) < 1e-6 && std::fabs(fr.output_mean_cosine - cs) < 1e-9 &&
                       fr.key_intermediate_mse > 0.0 && fr.value_intermediate_mse > 0.0,
                   "fidelity reports cosine, max error and intermediate MSE");
        }
        bool threw = false;
        try {
            fidelity(state, random_matrix(rng, 5, 128), values, qs, cfg);
        } catch (const InvalidInput&) {
            threw = true;
        }
        report(threw, "fidelity rejects originals of the wrong length (InvalidInput)");
        const std::string path = "/tmp/vqkv_cpp_snapshot.vqks";
        state.save_snapshot(path);
        CacheState back = CacheState::load_snapshot(path, ks, vs);
        ViewBlock all2 = back.view_block(0, back.total_len());
        report(back.total_len() == state.total_len() && back.key_codes() == state.key_codes() &&
                   back.value_codes() == state.value_codes() &&
                   std::memcmp(all2.keys.data(), all.keys.data(), sizeof(float) * size_t(all.keys.size())) == 0,
               "VQKS snapshot round-trips the cache bit for bit");
        auto other = random_stack(rng, 8, 256, 128);
        threw = false;
        try {
            CacheState::load_snapshot(path, other, vs);
        } catch (const InvalidInput&) {
            threw = true;
        }
        report(threw, "load_snapshot rejects a different key stack (content hash)");
        threw = false;
        try {
            throw DivergedError("loss is NaN", 3);
        } catch (const Error& e) {
            threw = std::string(e.what()).find("(epoch 3)") != std::string::npos;
        }
        report(threw, "DivergedError carries the epoch (errors.hpp:44-49)");
    }
    {  // codebook_test.cpp:257-273 RSVQ round trip + hash
        std::mt19937_64 rng(13);
        auto st = random_stack(rng, 3, 9, 6);
        st.cache_kind = CacheKind::value;
        std::ostringstream out(std::ios::binary);
        save_stack(st, out);
        std::istringstream in(out.str(), std::ios::binary);
        auto ld = load_stack(in);
        report(ld.num_stages() == 3 && ld.cache_kind == CacheKind::value &&
                   stack_content_hash(ld) == stack_content_hash(st),
               "stack save/load round-trips with equal content hash");
        std::string bad = out.str();
        bad[0] = 'X';
        std::istringstream in2(bad, std::ios::binary);
        bool ok = false;
        try {
            load_stack(in2);
        } catch (const FormatError& e) {
            ok = e.byte_offset == 0;
        }
        report(ok, "stack loader reports byte offset 0 for bad magic");
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
