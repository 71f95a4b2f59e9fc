// vqkv/attention.hpp -- drop-in for proj/core/include/vqkv/attention.hpp (B200 build).
//
// attend() runs the decode-step attention kernel over the cache's segments
// (init | compressed | pending+local) through vqkv_attend_decode_host: the
// compressed rows are consumed in the dot-product domain (query x codebook
// tables + value histograms) and never materialised.  Accumulation is fp32;
// outputs match the reference's double-precision streaming softmax within the
// documented bf16-level tolerance.  attend_raw runs the same
// kernel over raw rows only.
#pragma once

#include <cmath>

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
    VectorF out(vs.dim());
    float lse = 0.f;
    vqkv_attend_args a{};
    a.n_pairs = 1;
    a.group = 1;
    a.q_dev = q;
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
    a.out_dev = out.data();
    a.lse_dev = &lse;
    check(vqkv_attend_decode_host(ks.device(), vs.device(), &a));
    return out;
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
    (void)vd;
    return detail::run_attend(state.key_stack(), state.value_stack(), query.data(), state.init_keys().data(),
                              state.init_values().data(), state.init_rows(), &state.key_codes(), &state.value_codes(),
                              state.compressed_rows(), lk.data(), lv.data(), n_local, config.scale);
}

/// Same computation over raw matrices (attention.cpp:71-88).  Needs a stack
/// pair only for the device kernel's shapes; any stacks of matching dims work.
template <class Mat, class Vec>
VectorF attend_raw(const CodebookStack& key_stack, const CodebookStack& value_stack, const Mat& keys, const Mat& values,
                   const Vec& query, const AttentionConfig& config) {
    if (keys.rows() < 1 || keys.rows() != values.rows())
        throw InvalidInput("keys and values must be nonempty and the same length");
    if (query.size() != keys.cols()) throw InvalidInput("query dimension does not match key dimension");
    return detail::run_attend(key_stack, value_stack, query.data(), nullptr, nullptr, 0, nullptr, nullptr, 0,
                              keys.data(), values.data(), size_t(keys.rows()), config.scale);
}

}  // namespace vqkv
