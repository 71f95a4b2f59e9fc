// vqkv/attention.hpp -- drop-in for proj/core/include/vqkv/attention.hpp (B200 build).
//
// attend() runs the decode-step attention kernel over the cache's segments
// (init | compressed | pending+local) through vqkv_attend_decode_host: the
// compressed rows are consumed in the dot-product domain (query x codebook
// tables + value histograms) and never materialised.  Accumulation is fp32;
// outputs match the reference's double-precision streaming softmax within the
// documented bf16-level tolerance.  attend_raw runs the attention
// kernel over raw rows only (vqkv_attend_raw_host); fidelity follows
// attention.cpp:90-134 query by query.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>

#include "vqkv/kv_cache.hpp"

namespace vqkv {

struct AttentionConfig {
    size_t block_rows = 128;  // output is invariant to this (kept for API parity)
    double scale = 0.0;       // <= 0 means 1/sqrt(Dk)
    bool causal = true;       // unused, as in the reference (attention.cpp)

    void validate() const {
        if (block_rows < 1) throw InvalidInput("block_rows must be >= 1");
    }
};

struct AttendStats {
    // The reference's accounting of what a block_rows-streaming attend would
    // reconstruct (attention.cpp:46-53); the device path itself materialises
    // no rows.
    size_t peak_reconstructed_scalars = 0;
    size_t reconstructed_rows = 0;
};

struct FidelityReport {
    double output_max_abs_err = 0.0;
    double output_mean_cosine = 1.0;
    double key_intermediate_mse = 0.0;
    double value_intermediate_mse = 0.0;
};

namespace detail {
inline VectorF run_attend(const CodebookStack& ks, const CodebookStack& vs, const float* q, const float* ik,
                          const float* iv, size_t n_init, const CodeMatrix* kc, const CodeMatrix* vc, size_t n_comp,
                          const float* lk, const float* lv, size_t n_local, double scale) {
    const int64_t dk = ks.dim(), dv = vs.dim();
    // One query per call (attention.cpp:26-69).  The decode-attention kernels take G = 4 query
    // heads per KV head; at D = 128 the query is replicated into a group of 4 so the LUT kernel
    // (not the generic reconstruct-per-row one) serves this API too, and row 0 is returned.
    const int group = (dk == 128 && dv == 128 && n_comp > 0) ? 4 : 1;
    std::vector<float> qg(size_t(group * dk));
    for (int g = 0; g < group; ++g) std::memcpy(qg.data() + g * dk, q, sizeof(float) * size_t(dk));
    std::vector<float> og(static_cast<size_t>(group * dv)), lse(static_cast<size_t>(group));
    vqkv_attend_args a{};
    a.n_pairs = 1;
    a.group = uint32_t(group);
    a.q_dev = qg.data();
    a.init_k_dev = ik;
    a.init_v_dev = iv;
    a.n_init = n_init;
    a.kcodes_dev = n_comp ? kc->payload().data() : nullptr;
    a.vcodes_dev = n_comp ? vc->payload().data() : nullptr;
    a.n_comp = n_comp;
    a.local_k_dev = lk;
    a.local_v_dev = lv;
    a.n_local = n_local;
    a.scale = scale;
    a.out_dev = og.data();
    a.lse_dev = lse.data();
    check(vqkv_attend_decode_host(ks.device(), vs.device(), &a));
    VectorF out(dv);
    std::memcpy(out.data(), og.data(), sizeof(float) * size_t(dv));
    return out;
}

template <class Mat>
inline VectorF row_of(const Mat& m, int64_t r) {
    VectorF v(int64_t(m.cols()));
    std::memcpy(v.data(), m.data() + r * int64_t(m.cols()), sizeof(float) * size_t(m.cols()));
    return v;
}
}  // namespace detail

/// softmax(scale q K^T) V over the full logical cache (attention.cpp:26-69).
template <class Vec>
VectorF attend(const CacheState& state, const Vec& query, const AttentionConfig& config, AttendStats* stats = nullptr) {
    config.validate();
    if (state.total_len() < 1) throw InvalidState("cannot attend over an empty cache");
    if (int64_t(query.size()) != state.key_dim()) throw InvalidInput("query dimension does not match key dimension");
    const int64_t kd = state.key_dim(), vd = state.value_dim();
    if (stats) {  // reference block accounting over [init | compressed | ...]
        const size_t len = state.total_len(), c0 = state.init_rows(), c1 = c0 + state.compressed_rows();
        for (size_t b = 0; b < len; b += config.block_rows) {
            const size_t e = std::min(len, b + config.block_rows);
            const size_t lossy = (std::min(e, c1) > std::max(b, c0)) ? std::min(e, c1) - std::max(b, c0) : 0;
            stats->peak_reconstructed_scalars = std::max(stats->peak_reconstructed_scalars, lossy * size_t(kd + vd));
            stats->reconstructed_rows += lossy;
        }
    }
    // pending rows precede the local window in token order
    std::vector<float> lk, lv;
    for (const auto& r : state.pending_keys()) lk.insert(lk.end(), r.begin(), r.end());
    for (const auto& r : state.local_keys()) lk.insert(lk.end(), r.begin(), r.end());
    for (const auto& r : state.pending_values()) lv.insert(lv.end(), r.begin(), r.end());
    for (const auto& r : state.local_values()) lv.insert(lv.end(), r.begin(), r.end());
    const size_t n_local = lk.size() / size_t(kd);
    return detail::run_attend(state.key_stack(), state.value_stack(), query.data(), state.init_keys().data(),
                              state.init_values().data(), state.init_rows(), &state.key_codes(), &state.value_codes(),
                              state.compressed_rows(), lk.data(), lv.data(), n_local, config.scale);
}

/// Same computation over raw matrices (attention.cpp:71-88): keys [L x Dk], values [L x Dv].
template <class Mat, class Vec>
VectorF attend_raw(const Mat& keys, const Mat& values, const Vec& query, const AttentionConfig& config) {
    if (keys.rows() < 1 || keys.rows() != values.rows())
        throw InvalidInput("keys and values must be nonempty and the same length");
    if (int64_t(query.size()) != int64_t(keys.cols())) throw InvalidInput("query dimension does not match key dimension");
    VectorF out(int64_t(values.cols()));
    detail::check(vqkv_attend_raw_host(detail::device_index(), keys.data(), values.data(), uint64_t(keys.rows()),
                               uint32_t(keys.cols()), uint32_t(values.cols()), query.data(), config.scale, out.data()));
    return out;
}

/// Attention over the compressed state vs over the raw originals, one row per query, plus the
/// compressed rows' reconstruction MSE (attention.cpp:90-134).
template <class Mat>
FidelityReport fidelity(const CacheState& state, const Mat& original_keys, const Mat& original_values,
                        const Mat& queries, const AttentionConfig& config) {
    if (size_t(original_keys.rows()) != state.total_len() || size_t(original_values.rows()) != state.total_len())
        throw InvalidInput("originals length does not match cache length");
    if (int64_t(original_keys.cols()) != state.key_dim() || int64_t(original_values.cols()) != state.value_dim())
        throw InvalidInput("originals dimensions do not match the cache");
    if (queries.rows() < 1 || int64_t(queries.cols()) != state.key_dim())
        throw InvalidInput("queries must be nonempty with the key dimension");
    FidelityReport report;
    double cosine_sum = 0.0;
    for (int64_t i = 0; i < int64_t(queries.rows()); ++i) {
        const VectorF q = detail::row_of(queries, i);
        const VectorF compressed = attend(state, q, config);
        const VectorF raw = attend_raw(original_keys, original_values, q, config);
        double err = 0.0, dot = 0.0, nc = 0.0, nr = 0.0;
        for (int64_t d = 0; d < compressed.size(); ++d) {
            err = std::max(err, double(std::fabs(compressed[d] - raw[d])));
            dot += double(compressed[d]) * double(raw[d]);
            nc += double(compressed[d]) * double(compressed[d]);
            nr += double(raw[d]) * double(raw[d]);
        }
        report.output_max_abs_err = std::max(report.output_max_abs_err, err);
        const double denom = std::sqrt(nc) * std::sqrt(nr);
        cosine_sum += denom > 0.0 ? dot / denom : ((nc == 0.0 && nr == 0.0) ? 1.0 : 0.0);
    }
    report.output_mean_cosine = cosine_sum / double(queries.rows());
    const size_t comp = state.compressed_rows();
    if (comp > 0) {
        const size_t first = state.init_rows();
        auto mse = [&](const Mat& orig, const MatrixF& rec) {
            const int64_t d = rec.cols();
            double total = 0.0;
            for (size_t r = 0; r < comp; ++r) {
                double sq = 0.0;
                for (int64_t c = 0; c < d; ++c) {
                    const double x = double(orig.data()[(first + r) * size_t(d) + size_t(c)]) -
                                     double(rec.data()[r * size_t(d) + size_t(c)]);
                    sq += x * x;
                }
                total += sq;
            }
            return total / double(comp);
        };
        report.key_intermediate_mse = mse(original_keys, reconstruct_block(state.key_stack(), state.key_codes(), 0, comp));
        report.value_intermediate_mse =
                mse(original_values, reconstruct_block(state.value_stack(), state.value_codes(), 0, comp));
    }
    return report;
}

}  // namespace vqkv
