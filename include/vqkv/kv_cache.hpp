// vqkv/kv_cache.hpp -- drop-in for proj/core/include/vqkv/kv_cache.hpp (B200 build).
//
// Three-segment KV store for one (layer, head) stream with the reference's
// window policy and accounting (kv_cache.cpp:41-204): raw prompt head,
// compressed middle (CodeMatrix, encoded on the GPU by quantize_batch), raw
// local window; deferred flushes of local_len evicted rows.  Compressed rows
// are reconstructed on the GPU by view_block.  Single writer (kv_cache.hpp:41-44).
#pragma once

#include <cstring>
#include <deque>
#include <fstream>
#include <string>
#include <vector>

#include "vqkv/codebook.hpp"

namespace vqkv {

struct WindowPolicy {
    size_t init_len = 4;      // never-compressed prompt head
    size_t local_len = 1024;  // raw sliding window over recent tokens
    bool eager = false;       // quantize at every eviction instead of batching

    void validate() const {
        if (local_len < 1) throw InvalidInput("local_len must be >= 1");
    }
};

struct MemoryReport {
    size_t raw_bytes_equivalent = 0;
    size_t compressed_payload_bits = 0;
    size_t codebook_overhead_bytes = 0;
    double effective_ratio = 0.0;
};

struct ViewBlock {
    MatrixF keys;    // len x Dk
    MatrixF values;  // len x Dv
    std::vector<bool> exact;
};

class CacheState {
public:
    CacheState(const CodebookStack& key_stack, const CodebookStack& value_stack, WindowPolicy policy)
        : key_stack_(&key_stack), value_stack_(&value_stack), policy_(policy), key_codes_(key_stack.stage_sizes()),
          value_codes_(value_stack.stage_sizes()) {
        policy_.validate();
        key_stack.validate();
        value_stack.validate();
        init_keys_.resize(0, key_stack.dim());
        init_values_.resize(0, value_stack.dim());
    }

    template <class Mat>
    void prefill(const Mat& keys, const Mat& values) {
        if (total_len() != 0 || prefilled_) throw InvalidState("prefill requires an empty cache");
        if (keys.rows() < 1) throw InvalidInput("prefill needs at least one token");
        if (keys.rows() != values.rows()) throw InvalidInput("keys and values must have the same length");
        if (int64_t(keys.cols()) != key_dim() || int64_t(values.cols()) != value_dim())
            throw InvalidInput("key/value dimensions do not match the stacks");
        const size_t len = size_t(keys.rows());
        const size_t n_init = std::min(policy_.init_len, len);
        const size_t n_local = std::min(policy_.local_len, len - n_init);
        const size_t n_mid = len - n_init - n_local;
        const int64_t kd = key_dim(), vd = value_dim();
        init_keys_ = slice(keys, 0, n_init);
        init_values_ = slice(values, 0, n_init);
        if (n_mid > 0) {
            QuantizeBatchResult k = quantize_batch(*key_stack_, slice(keys, n_init, n_init + n_mid));
            QuantizeBatchResult v = quantize_batch(*value_stack_, slice(values, n_init, n_init + n_mid));
            key_codes_ = std::move(k.codes);
            value_codes_ = std::move(v.codes);
            key_residual_norms_.assign(k.residual_norms.data(), k.residual_norms.data() + n_mid);
            value_residual_norms_.assign(v.residual_norms.data(), v.residual_norms.data() + n_mid);
        }
        for (size_t i = len - n_local; i < len; ++i) {
            local_keys_.emplace_back(keys.data() + i * kd, keys.data() + (i + 1) * kd);
            local_values_.emplace_back(values.data() + i * vd, values.data() + (i + 1) * vd);
        }
        prefilled_ = true;
    }

    template <class Vec>
    void append_token(const Vec& key, const Vec& value) {
        if (!prefilled_ && policy_.init_len != 0)
            throw InvalidState("append_token requires a prefilled cache (or init_len == 0)");
        if (int64_t(key.size()) != key_dim() || int64_t(value.size()) != value_dim())
            throw InvalidInput("key/value dimensions do not match the stacks");
        local_keys_.emplace_back(key.data(), key.data() + key.size());
        local_values_.emplace_back(value.data(), value.data() + value.size());
        if (local_keys_.size() > policy_.local_len) {
            pending_keys_.push_back(std::move(local_keys_.front()));
            pending_values_.push_back(std::move(local_values_.front()));
            local_keys_.pop_front();
            local_values_.pop_front();
            if (policy_.eager || pending_keys_.size() >= policy_.local_len) flush_pending();
        }
    }

    ViewBlock view_block(size_t begin, size_t end) const {
        const size_t len = total_len();
        if (begin > end || end > len)
            throw InvalidInput("view range [" + std::to_string(begin) + ", " + std::to_string(end) +
                               ") out of bounds for length " + std::to_string(len));
        ViewBlock out;
        const int64_t kd = key_dim(), vd = value_dim();
        out.keys.resize(int64_t(end - begin), kd);
        out.values.resize(int64_t(end - begin), vd);
        out.exact.assign(end - begin, true);
        const size_t ie = init_rows(), ce = ie + compressed_rows(), pe = ce + pending_rows();
        size_t g = begin;
        while (g < end) {
            const size_t dst = g - begin;
            if (g < ie) {
                const size_t stop = std::min(end, ie);
                copy_rows(out.keys, dst, init_keys_.data() + g * kd, stop - g, kd);
                copy_rows(out.values, dst, init_values_.data() + g * vd, stop - g, vd);
                g = stop;
            } else if (g < ce) {
                const size_t stop = std::min(end, ce);
                MatrixF k = reconstruct_block(*key_stack_, key_codes_, g - ie, stop - ie);
                MatrixF v = reconstruct_block(*value_stack_, value_codes_, g - ie, stop - ie);
                copy_rows(out.keys, dst, k.data(), stop - g, kd);
                copy_rows(out.values, dst, v.data(), stop - g, vd);
                for (size_t i = g; i < stop; ++i) out.exact[i - begin] = false;
                g = stop;
            } else if (g < pe) {
                copy_rows(out.keys, dst, pending_keys_[g - ce].data(), 1, kd);
                copy_rows(out.values, dst, pending_values_[g - ce].data(), 1, vd);
                ++g;
            } else {
                copy_rows(out.keys, dst, local_keys_[g - pe].data(), 1, kd);
                copy_rows(out.values, dst, local_values_[g - pe].data(), 1, vd);
                ++g;
            }
        }
        return out;
    }

    MemoryReport memory_report() const {
        MemoryReport r;
        const size_t spt = size_t(key_dim() + value_dim());
        r.raw_bytes_equivalent = total_len() * spt * 2;
        r.compressed_payload_bits = key_codes_.payload_bits() + value_codes_.payload_bits();
        r.codebook_overhead_bytes = serialized_bytes(*key_stack_) + serialized_bytes(*value_stack_);
        if (compressed_rows() > 0)
            r.effective_ratio = 1.0 - double(r.compressed_payload_bits) / double(compressed_rows() * spt * 16);
        return r;
    }

    size_t total_len() const { return init_rows() + compressed_rows() + pending_rows() + local_rows(); }
    size_t init_rows() const { return size_t(init_keys_.rows()); }
    size_t compressed_rows() const { return key_codes_.rows(); }
    size_t pending_rows() const { return pending_keys_.size(); }
    size_t local_rows() const { return local_keys_.size(); }
    size_t intermediate_rows() const { return compressed_rows() + pending_rows(); }
    size_t batched_compressions() const { return batched_compressions_; }
    const WindowPolicy& policy() const { return policy_; }
    const CodebookStack& key_stack() const { return *key_stack_; }
    const CodebookStack& value_stack() const { return *value_stack_; }
    int64_t key_dim() const { return key_stack_->dim(); }
    int64_t value_dim() const { return value_stack_->dim(); }
    const CodeMatrix& key_codes() const { return key_codes_; }
    const CodeMatrix& value_codes() const { return value_codes_; }
    const std::vector<float>& key_residual_norms() const { return key_residual_norms_; }
    const std::vector<float>& value_residual_norms() const { return value_residual_norms_; }

    /// VQKS snapshot (kv_cache.cpp:206-246): same byte layout as the reference.
    void save_snapshot(const std::string& path) const;
    /// kv_cache.cpp:248-312: rejects foreign stacks (content hash) and inconsistent lengths.
    static CacheState load_snapshot(const std::string& path, const CodebookStack& key_stack,
                                    const CodebookStack& value_stack);

    // raw segment access for the device attention path
    const MatrixF& init_keys() const { return init_keys_; }
    const MatrixF& init_values() const { return init_values_; }
    const std::vector<std::vector<float>>& pending_keys() const { return pending_keys_; }
    const std::vector<std::vector<float>>& pending_values() const { return pending_values_; }
    const std::deque<std::vector<float>>& local_keys() const { return local_keys_; }
    const std::deque<std::vector<float>>& local_values() const { return local_values_; }

private:
    template <class Mat>
    static MatrixF slice(const Mat& m, size_t r0, size_t r1) {
        MatrixF out(int64_t(r1 - r0), int64_t(m.cols()));
        if (r1 > r0) std::memcpy(out.data(), m.data() + r0 * size_t(m.cols()), sizeof(float) * (r1 - r0) * size_t(m.cols()));
        return out;
    }
    static void copy_rows(MatrixF& dst, size_t row, const float* src, size_t n, int64_t d) {
        std::memcpy(dst.data() + row * size_t(d), src, sizeof(float) * n * size_t(d));
    }
    static size_t serialized_bytes(const CodebookStack& s) {
        size_t b = 4 + 4 + 1 + 4;
        for (const auto& st : s.stages) b += 8 + sizeof(float) * size_t(st.entries.size() + st.projection.size());
        return b;
    }
    void flush_pending() {  // kv_cache.cpp:102-120: one batched GPU encode per flush
        const size_t n = pending_keys_.size();
        const int64_t kd = key_dim(), vd = value_dim();
        MatrixF k(int64_t(n), kd), v(int64_t(n), vd);
        for (size_t i = 0; i < n; ++i) {
            std::memcpy(k.data() + i * kd, pending_keys_[i].data(), sizeof(float) * kd);
            std::memcpy(v.data() + i * vd, pending_values_[i].data(), sizeof(float) * vd);
        }
        QuantizeBatchResult kq = quantize_batch(*key_stack_, k);
        QuantizeBatchResult vq = quantize_batch(*value_stack_, v);
        key_codes_.append_rows(kq.codes);
        value_codes_.append_rows(vq.codes);
        for (size_t i = 0; i < n; ++i) {
            key_residual_norms_.push_back(kq.residual_norms[int64_t(i)]);
            value_residual_norms_.push_back(vq.residual_norms[int64_t(i)]);
        }
        pending_keys_.clear();
        pending_values_.clear();
        ++batched_compressions_;
    }

    const CodebookStack* key_stack_;
    const CodebookStack* value_stack_;
    WindowPolicy policy_;
    bool prefilled_ = false;
    MatrixF init_keys_, init_values_;
    CodeMatrix key_codes_, value_codes_;
    std::vector<float> key_residual_norms_, value_residual_norms_;
    std::vector<std::vector<float>> pending_keys_, pending_values_;
    std::deque<std::vector<float>> local_keys_, local_values_;
    size_t batched_compressions_ = 0;
};

namespace detail {
template <class T>
inline void put_scalar(std::ostream& out, T v) {
    out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
inline T get_scalar(std::istream& in, size_t& offset, const char* what) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw FormatError(std::string("truncated file reading ") + what, offset);
    offset += sizeof(T);
    return v;
}
inline void get_bytes(std::istream& in, void* p, size_t n, size_t& offset, const char* what) {
    in.read(static_cast<char*>(p), std::streamsize(n));
    if (!in) throw FormatError(std::string("truncated file reading ") + what, offset);
    offset += n;
}
}  // namespace detail

inline void CacheState::save_snapshot(const std::string& path) const {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path + " for writing");
    using detail::put_scalar;
    out.write("VQKS", 4);
    put_scalar<uint32_t>(out, 1);
    put_scalar<uint64_t>(out, policy_.init_len);
    put_scalar<uint64_t>(out, policy_.local_len);
    put_scalar<uint8_t>(out, policy_.eager ? 1 : 0);
    put_scalar<uint8_t>(out, prefilled_ ? 1 : 0);
    put_scalar<uint64_t>(out, total_len());
    put_scalar<uint32_t>(out, uint32_t(key_dim()));
    put_scalar<uint32_t>(out, uint32_t(value_dim()));
    put_scalar<uint64_t>(out, stack_content_hash(*key_stack_));
    put_scalar<uint64_t>(out, stack_content_hash(*value_stack_));
    put_scalar<uint64_t>(out, batched_compressions_);
    for (const MatrixF* m : {&init_keys_, &init_values_}) {
        put_scalar<uint64_t>(out, uint64_t(m->rows()));
        out.write(reinterpret_cast<const char*>(m->data()), std::streamsize(sizeof(float) * size_t(m->size())));
    }
    key_codes_.save(out);
    value_codes_.save(out);
    out.write(reinterpret_cast<const char*>(key_residual_norms_.data()),
              std::streamsize(sizeof(float) * key_residual_norms_.size()));
    out.write(reinterpret_cast<const char*>(value_residual_norms_.data()),
              std::streamsize(sizeof(float) * value_residual_norms_.size()));
    auto rows = [&](const auto& rs) {
        put_scalar<uint64_t>(out, uint64_t(rs.size()));
        for (const auto& r : rs) out.write(reinterpret_cast<const char*>(r.data()), std::streamsize(sizeof(float) * r.size()));
    };
    rows(pending_keys_);
    rows(pending_values_);
    rows(local_keys_);
    rows(local_values_);
    if (!out) throw IoError("write failed for " + path);
}

inline CacheState CacheState::load_snapshot(const std::string& path, const CodebookStack& key_stack,
                                            const CodebookStack& value_stack) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    size_t off = 0;
    char magic[4] = {};
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "VQKS", 4) != 0) throw FormatError("bad magic, expected VQKS", 0);
    off = 4;
    using detail::get_scalar;
    const auto version = get_scalar<uint32_t>(in, off, "version");
    if (version != 1) throw FormatError("unsupported snapshot version " + std::to_string(version), off - 4);
    WindowPolicy policy;
    policy.init_len = get_scalar<uint64_t>(in, off, "init_len");
    policy.local_len = get_scalar<uint64_t>(in, off, "local_len");
    policy.eager = get_scalar<uint8_t>(in, off, "eager flag") != 0;
    const bool prefilled = get_scalar<uint8_t>(in, off, "prefilled flag") != 0;
    const auto stored_len = get_scalar<uint64_t>(in, off, "total_len");
    const auto dk = get_scalar<uint32_t>(in, off, "key dim");
    const auto dv = get_scalar<uint32_t>(in, off, "value dim");
    if (int64_t(dk) != key_stack.dim() || int64_t(dv) != value_stack.dim())
        throw InvalidInput("snapshot dimensions do not match the supplied stacks");
    const auto kh = get_scalar<uint64_t>(in, off, "key stack hash");
    const auto vh = get_scalar<uint64_t>(in, off, "value stack hash");
    if (kh != stack_content_hash(key_stack) || vh != stack_content_hash(value_stack))
        throw InvalidInput("snapshot was built against different codebook stacks");
    CacheState st(key_stack, value_stack, policy);
    st.prefilled_ = prefilled;
    st.batched_compressions_ = get_scalar<uint64_t>(in, off, "compression count");
    auto matrix = [&](MatrixF& m, int64_t cols, const char* what) {
        const auto r = get_scalar<uint64_t>(in, off, what);
        m.resize(int64_t(r), cols);
        detail::get_bytes(in, m.data(), sizeof(float) * size_t(m.size()), off, what);
    };
    matrix(st.init_keys_, key_stack.dim(), "init keys");
    matrix(st.init_values_, value_stack.dim(), "init values");
    st.key_codes_ = CodeMatrix::load(in, off);
    st.value_codes_ = CodeMatrix::load(in, off);
    st.key_residual_norms_.resize(st.key_codes_.rows());
    detail::get_bytes(in, st.key_residual_norms_.data(), sizeof(float) * st.key_residual_norms_.size(), off,
                      "key residual norms");
    st.value_residual_norms_.resize(st.value_codes_.rows());
    detail::get_bytes(in, st.value_residual_norms_.data(), sizeof(float) * st.value_residual_norms_.size(), off,
                      "value residual norms");
    auto rows = [&](auto& rs, int64_t dim, const char* what) {
        const auto n = get_scalar<uint64_t>(in, off, what);
        for (uint64_t i = 0; i < n; ++i) {
            std::vector<float> r(static_cast<size_t>(dim));
            detail::get_bytes(in, r.data(), sizeof(float) * r.size(), off, what);
            rs.push_back(std::move(r));
        }
    };
    rows(st.pending_keys_, key_stack.dim(), "pending keys");
    rows(st.pending_values_, value_stack.dim(), "pending values");
    rows(st.local_keys_, key_stack.dim(), "local keys");
    rows(st.local_values_, value_stack.dim(), "local values");
    if (st.total_len() != stored_len) throw FormatError("segment lengths do not add up to total_len", off);
    return st;
}

}  // namespace vqkv
