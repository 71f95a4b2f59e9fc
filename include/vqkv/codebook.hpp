// vqkv/codebook.hpp -- drop-in for proj/core/include/vqkv/codebook.hpp (B200 build).
//
// Same names, fields, argument meaning and exceptions as the reference
// (codebook.hpp:18-138); the arithmetic runs in libvqkv_b200.so through the
// C-ABI of include/vqkv_c.h:
//   Codebook::refresh        -> vqkv_stack_create (device refresh, reference fp32 order)
//   nearest_entry            -> vqkv_nearest_host
//   quantize / quantize_batch-> vqkv_quantize_rows_host (tensor-core encoder, D = 128)
//   reconstruct(_block)      -> vqkv_reconstruct_block_host
// Matrices: define VQKV_USE_EIGEN to use the reference's Eigen typedefs
// (codebook.hpp:18-19); otherwise a small row-major stand-in with the subset of
// the Eigen interface these headers need (rows/cols/size/data/operator()).
// Link with -lvqkv_b200 (paper_2603_16435_b200/lib).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iosfwd>
#include <istream>
#include <memory>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include "vqkv/bitpack.hpp"
#include "vqkv/errors.hpp"
#include "vqkv_c.h"

#ifdef VQKV_USE_EIGEN
#include <Eigen/Core>
#endif

namespace vqkv {

#ifdef VQKV_USE_EIGEN
using MatrixF = Eigen::Matrix<float, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
using VectorF = Eigen::VectorXf;
#else
/// Row-major fp32 matrix (stand-in for the reference's Eigen MatrixF).
class MatrixF {
public:
    MatrixF() = default;
    MatrixF(int64_t rows, int64_t cols) : r_(rows), c_(cols), d_(size_t(rows * cols), 0.f) {}
    int64_t rows() const { return r_; }
    int64_t cols() const { return c_; }
    int64_t size() const { return r_ * c_; }
    float* data() { return d_.data(); }
    const float* data() const { return d_.data(); }
    float& operator()(int64_t r, int64_t c) { return d_[size_t(r * c_ + c)]; }
    float operator()(int64_t r, int64_t c) const { return d_[size_t(r * c_ + c)]; }
    void resize(int64_t rows, int64_t cols) {
        r_ = rows;
        c_ = cols;
        d_.assign(size_t(rows * cols), 0.f);
    }
    static MatrixF Zero(int64_t rows, int64_t cols) { return MatrixF(rows, cols); }
    static MatrixF Identity(int64_t rows, int64_t cols) {
        MatrixF m(rows, cols);
        for (int64_t i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.f;
        return m;
    }

private:
    int64_t r_ = 0, c_ = 0;
    std::vector<float> d_;
};

/// fp32 column vector (stand-in for Eigen::VectorXf).
class VectorF {
public:
    VectorF() = default;
    explicit VectorF(int64_t n) : d_(size_t(n), 0.f) {}
    VectorF(std::initializer_list<float> v) : d_(v) {}
    int64_t size() const { return int64_t(d_.size()); }
    float* data() { return d_.data(); }
    const float* data() const { return d_.data(); }
    float& operator[](int64_t i) { return d_[size_t(i)]; }
    float operator[](int64_t i) const { return d_[size_t(i)]; }
    float& operator()(int64_t i) { return d_[size_t(i)]; }
    float operator()(int64_t i) const { return d_[size_t(i)]; }
    void resize(int64_t n) { d_.assign(size_t(n), 0.f); }
    static VectorF Zero(int64_t n) { return VectorF(n); }
    float squaredNorm() const {
        double s = 0;
        for (float v : d_) s += double(v) * v;
        return float(s);
    }
    float norm() const { return std::sqrt(squaredNorm()); }

private:
    std::vector<float> d_;
};
#endif

enum class CacheKind : uint8_t { key = 0, value = 1 };

constexpr size_t kDefaultSearchBlock = 4096;  // codebook.hpp:25

namespace detail {
struct StackHandle {
    vqkv_stack_t h = nullptr;
    ~StackHandle() {
        if (h) vqkv_stack_destroy(h);
    }
};
inline int device_index() {
    const char* e = std::getenv("VQKV_DEVICE");
    return e ? std::atoi(e) : 0;
}
}  // namespace detail

/// One residual stage: raw entries plus a learned projection; effective
/// entries = entries . projection^T are computed on the device (refresh()).
struct Codebook {
    MatrixF entries;     // S x D
    MatrixF projection;  // D x D
    MatrixF effective;   // S x D, row i = projection * entries.row(i)
    VectorF effective_sqnorm;

    int64_t size() const { return entries.rows(); }
    int64_t dim() const { return entries.cols(); }

    /// Recomputes effective entries and their squared norms (on the GPU, in
    /// the reference's fp32 operation order -- bit-identical values).
    void refresh();
    void validate() const;

    // device copy used by nearest_entry (one-stage stack)
    mutable std::shared_ptr<detail::StackHandle> device_;
};

/// Ordered residual stages; immutable once loaded (codebook.hpp:45-56).
struct CodebookStack {
    std::vector<Codebook> stages;
    CacheKind cache_kind = CacheKind::key;

    size_t num_stages() const { return stages.size(); }
    int64_t dim() const { return stages.empty() ? 0 : stages.front().dim(); }
    std::vector<uint32_t> stage_sizes() const {
        std::vector<uint32_t> s;
        for (const auto& c : stages) s.push_back(uint32_t(c.size()));
        return s;
    }
    void validate() const {
        if (stages.empty()) throw InvalidInput("stack must have at least one stage");
        for (const auto& st : stages) {
            st.validate();
            if (st.dim() != dim()) throw InvalidInput("all stages must share one dimension");
        }
    }
    /// The device stack (created on first use; the stack must not change afterwards).
    vqkv_stack_t device() const {
        if (!device_) {
            validate();
            auto h = std::make_shared<detail::StackHandle>();
            std::vector<uint32_t> sizes = stage_sizes();
            std::vector<float> ent, proj;
            for (const auto& c : stages) {
                ent.insert(ent.end(), c.entries.data(), c.entries.data() + c.entries.size());
                proj.insert(proj.end(), c.projection.data(), c.projection.data() + c.projection.size());
            }
            detail::check(vqkv_stack_create(detail::device_index(), int(cache_kind), uint32_t(sizes.size()),
                                            sizes.data(), uint32_t(dim()), ent.data(), proj.data(), &h->h));
            device_ = h;
        }
        return device_->h;
    }

    mutable std::shared_ptr<detail::StackHandle> device_;
};

inline void Codebook::validate() const {
    if (entries.rows() < 1 || entries.cols() < 1) throw InvalidInput("codebook must have S >= 1 and D >= 1");
    if (projection.rows() != entries.cols() || projection.cols() != entries.cols())
        throw InvalidInput("projection must be DxD");
    for (int64_t i = 0; i < entries.size(); ++i)
        if (!std::isfinite(entries.data()[i])) throw InvalidInput("codebook contains non-finite values");
    for (int64_t i = 0; i < projection.size(); ++i)
        if (!std::isfinite(projection.data()[i])) throw InvalidInput("codebook contains non-finite values");
}

inline void Codebook::refresh() {
    validate();
    CodebookStack one;
    one.stages.push_back(*this);
    one.stages.back().device_.reset();
    vqkv_stack_t h = one.device();
    effective.resize(size(), dim());
    effective_sqnorm.resize(size());
    detail::check(vqkv_stack_effective(h, 0, effective.data(), effective_sqnorm.data()));
    device_ = one.device_;
}

using CodeVector = std::vector<uint32_t>;

/// Bit-packed append-only rows (codebook.hpp:63-91); payload bytes are the
/// device kernels' code layout.
class CodeMatrix {
public:
    CodeMatrix() = default;
    explicit CodeMatrix(std::vector<uint32_t> stage_sizes) : stage_sizes_(std::move(stage_sizes)) {
        for (uint32_t s : stage_sizes_) {
            if (s < 1) throw InvalidInput("stage size must be >= 1");
            stage_bit_offset_.push_back(row_bits_);
            unsigned w = index_bit_width(s);
            stage_bits_.push_back(w);
            row_bits_ += w;
        }
    }

    size_t rows() const { return rows_; }
    size_t num_stages() const { return stage_sizes_.size(); }
    const std::vector<uint32_t>& stage_sizes() const { return stage_sizes_; }
    size_t row_bits() const { return row_bits_; }
    size_t payload_bits() const { return rows_ * row_bits_; }
    const std::vector<uint8_t>& payload() const { return payload_; }

    void append(const CodeVector& codes) {
        if (codes.size() != stage_sizes_.size()) throw InvalidInput("code vector has wrong stage count");
        for (size_t i = 0; i < codes.size(); ++i)
            if (codes[i] >= stage_sizes_[i])
                throw InvalidCode("index " + std::to_string(codes[i]) + " out of range for stage " + std::to_string(i));
        const size_t base = rows_ * row_bits_;
        for (size_t i = 0; i < codes.size(); ++i) bit_write(payload_, base + stage_bit_offset_[i], codes[i], stage_bits_[i]);
        ++rows_;
    }
    CodeVector row(size_t r) const {
        if (r >= rows_) throw InvalidInput("row " + std::to_string(r) + " out of range");
        CodeVector c(stage_sizes_.size());
        for (size_t i = 0; i < c.size(); ++i) c[i] = bit_read(payload_, r * row_bits_ + stage_bit_offset_[i], stage_bits_[i]);
        return c;
    }
    uint32_t code_at(size_t r, size_t stage) const {
        if (r >= rows_ || stage >= stage_sizes_.size()) throw InvalidInput("code_at out of range");
        return bit_read(payload_, r * row_bits_ + stage_bit_offset_[stage], stage_bits_[stage]);
    }
    bool operator==(const CodeMatrix& o) const {
        return stage_sizes_ == o.stage_sizes_ && rows_ == o.rows_ && payload_ == o.payload_;
    }

    /// Adopts `rows` rows from a device-produced payload (same layout).
    static CodeMatrix from_payload(std::vector<uint32_t> sizes, const uint8_t* data, size_t rows) {
        CodeMatrix m(std::move(sizes));
        m.rows_ = rows;
        m.payload_.assign(data, data + (rows * m.row_bits_ + 7) / 8);
        return m;
    }
    /// Appends all rows of `other` (same stage sizes), keeping the bit layout.
    void append_rows(const CodeMatrix& other) {
        for (size_t r = 0; r < other.rows(); ++r) append(other.row(r));
    }

    void save(std::ostream& out) const {
        auto put = [&](const void* p, size_t n) { out.write(static_cast<const char*>(p), std::streamsize(n)); };
        uint32_t n = uint32_t(stage_sizes_.size());
        put(&n, 4);
        for (uint32_t s : stage_sizes_) put(&s, 4);
        uint64_t r = rows_;
        put(&r, 8);
        put(payload_.data(), payload_.size());
    }
    static CodeMatrix load(std::istream& in, size_t& offset) {
        auto get = [&](void* p, size_t n, const char* what) {
            in.read(static_cast<char*>(p), std::streamsize(n));
            if (!in) throw FormatError(std::string("truncated file reading ") + what, offset);
            offset += n;
        };
        uint32_t n = 0;
        get(&n, 4, "stage count");
        if (n < 1) throw FormatError("stage count must be >= 1", offset - 4);
        std::vector<uint32_t> sizes(n);
        for (auto& s : sizes) {
            get(&s, 4, "stage size");
            if (s < 1) throw FormatError("stage size must be >= 1", offset - 4);
        }
        CodeMatrix m(std::move(sizes));
        uint64_t rows = 0;
        get(&rows, 8, "row count");
        m.rows_ = rows;
        m.payload_.resize((m.rows_ * m.row_bits_ + 7) / 8);
        get(m.payload_.data(), m.payload_.size(), "code payload");
        return m;
    }

private:
    std::vector<uint32_t> stage_sizes_;
    std::vector<unsigned> stage_bits_;
    std::vector<size_t> stage_bit_offset_;
    size_t row_bits_ = 0;
    size_t rows_ = 0;
    std::vector<uint8_t> payload_;
};

struct NearestResult {
    uint32_t index;
    float distance;
};

/// Argmin over effective entries of ||x - e_i|| (lowest index on ties).
template <class Vec>
NearestResult nearest_entry(const Codebook& codebook, const Vec& x, size_t search_block = kDefaultSearchBlock) {
    if (int64_t(x.size()) != codebook.dim())
        throw InvalidInput("vector dimension " + std::to_string(x.size()) + " does not match codebook dimension " +
                           std::to_string(codebook.dim()));
    for (int64_t i = 0; i < int64_t(x.size()); ++i)
        if (!std::isfinite(x.data()[i])) throw InvalidInput("query vector contains non-finite values");
    if (!codebook.device_) const_cast<Codebook&>(codebook).refresh();
    NearestResult r{0, 0.f};
    detail::check(vqkv_nearest_host(codebook.device_->h, 0, x.data(), search_block, &r.index, &r.distance));
    return r;
}

struct QuantizeResult {
    CodeVector codes;
    VectorF final_residual;
};

inline void check_dim(const CodebookStack& stack, int64_t got) {
    if (got != stack.dim())
        throw InvalidInput("vector dimension " + std::to_string(got) + " does not match stack dimension " +
                           std::to_string(stack.dim()));
}

/// Greedy residual encoding (codebook.cpp:194-206).
template <class Vec>
QuantizeResult quantize(const CodebookStack& stack, const Vec& x, size_t search_block = kDefaultSearchBlock) {
    check_dim(stack, int64_t(x.size()));
    QuantizeResult out;
    const size_t pb = (stack.num_stages() ? vqkv_payload_bytes(stack.device(), 1) : 0);
    std::vector<uint8_t> pay(std::max<size_t>(pb, 1));
    float norm = 0.f;
    out.final_residual.resize(stack.dim());
    detail::check(vqkv_quantize_rows_host(stack.device(), x.data(), 1, search_block, pay.data(), &norm,
                                          out.final_residual.data()));
    out.codes = CodeMatrix::from_payload(stack.stage_sizes(), pay.data(), 1).row(0);
    return out;
}

struct QuantizeBatchResult {
    CodeMatrix codes;
    VectorF residual_norms;
};

/// Row-for-row identical to quantize() on each row (codebook.cpp:225-237).
template <class Mat>
QuantizeBatchResult quantize_batch(const CodebookStack& stack, const Mat& xs, size_t search_block = kDefaultSearchBlock) {
    if (xs.rows() > 0) check_dim(stack, int64_t(xs.cols()));
    QuantizeBatchResult out{CodeMatrix(stack.stage_sizes()), VectorF(int64_t(xs.rows()))};
    if (xs.rows() == 0) return out;
    const uint64_t rows = uint64_t(xs.rows());
    std::vector<uint8_t> pay(std::max<uint64_t>(vqkv_payload_bytes(stack.device(), rows), 1));
    detail::check(vqkv_quantize_rows_host(stack.device(), xs.data(), rows, search_block, pay.data(),
                                          out.residual_norms.data(), nullptr));
    out.codes = CodeMatrix::from_payload(stack.stage_sizes(), pay.data(), rows);
    return out;
}

/// Rows [begin, end); bit-identical for any partition (codebook.cpp:239-250).
inline MatrixF reconstruct_block(const CodebookStack& stack, const CodeMatrix& codes, size_t begin, size_t end) {
    if (begin > end || end > codes.rows())
        throw InvalidInput("row range [" + std::to_string(begin) + ", " + std::to_string(end) + ") out of bounds for " +
                           std::to_string(codes.rows()) + " rows");
    MatrixF out(int64_t(end - begin), stack.dim());
    if (end == begin) return out;
    detail::check(vqkv_reconstruct_block_host(stack.device(), codes.payload().data(), codes.rows(), begin, end,
                                              out.data()));
    return out;
}

/// Sum of the selected effective entries, in stage order (codebook.cpp:208-223).
inline VectorF reconstruct(const CodebookStack& stack, const CodeVector& codes) {
    if (codes.size() != stack.num_stages())
        throw InvalidCode("code vector has " + std::to_string(codes.size()) + " stages, stack has " +
                          std::to_string(stack.num_stages()));
    for (size_t i = 0; i < codes.size(); ++i)
        if (codes[i] >= uint32_t(stack.stages[i].size()))
            throw InvalidCode("index " + std::to_string(codes[i]) + " out of range for stage " + std::to_string(i));
    CodeMatrix m(stack.stage_sizes());
    m.append(codes);
    MatrixF r = reconstruct_block(stack, m, 0, 1);
    VectorF v(stack.dim());
    std::memcpy(v.data(), r.data(), sizeof(float) * size_t(stack.dim()));
    return v;
}

// ---- RSVQ container (codebook.cpp:252-336) ------------------------------------
inline void save_stack(const CodebookStack& stack, std::ostream& out) {
    stack.validate();
    auto put = [&](const void* p, size_t n) { out.write(static_cast<const char*>(p), std::streamsize(n)); };
    put("RSVQ", 4);
    uint32_t version = 1, n = uint32_t(stack.num_stages());
    uint8_t kind = uint8_t(stack.cache_kind);
    put(&version, 4);
    put(&kind, 1);
    put(&n, 4);
    for (const auto& c : stack.stages) {
        uint32_t s = uint32_t(c.size()), d = uint32_t(c.dim());
        put(&s, 4);
        put(&d, 4);
        put(c.entries.data(), sizeof(float) * size_t(c.entries.size()));
        put(c.projection.data(), sizeof(float) * size_t(c.projection.size()));
    }
}

inline void save_stack(const CodebookStack& stack, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path + " for writing");
    save_stack(stack, out);
    if (!out) throw IoError("write failed for " + path);
}

inline CodebookStack load_stack(std::istream& in) {
    size_t off = 0;
    auto get = [&](void* p, size_t n, const char* what) {
        in.read(static_cast<char*>(p), std::streamsize(n));
        if (!in) throw FormatError(std::string("truncated file reading ") + what, off);
        off += n;
    };
    char magic[4] = {};
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "RSVQ", 4) != 0) throw FormatError("bad magic, expected RSVQ", 0);
    off = 4;
    uint32_t version = 0, n = 0;
    uint8_t kind = 0;
    get(&version, 4, "version");
    if (version != 1) throw FormatError("unsupported version " + std::to_string(version), off - 4);
    get(&kind, 1, "cache kind");
    if (kind > 1) throw FormatError("bad cache kind " + std::to_string(kind), off - 1);
    get(&n, 4, "stage count");
    if (n < 1) throw FormatError("stage count must be >= 1", off - 4);
    CodebookStack st;
    st.cache_kind = CacheKind(kind);
    st.stages.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t s = 0, d = 0;
        get(&s, 4, "codebook size");
        get(&d, 4, "dimension");
        if (s < 1 || d < 1) throw FormatError("codebook size and dimension must be >= 1", off - 8);
        const size_t stage_off = off;
        Codebook& cb = st.stages[i];
        cb.entries.resize(s, d);
        get(cb.entries.data(), sizeof(float) * size_t(s) * d, "entries");
        cb.projection.resize(d, d);
        get(cb.projection.data(), sizeof(float) * size_t(d) * d, "projection");
        for (int64_t k = 0; k < cb.entries.size(); ++k)
            if (!std::isfinite(cb.entries.data()[k])) throw FormatError("non-finite values in stage " + std::to_string(i), stage_off);
        for (int64_t k = 0; k < cb.projection.size(); ++k)
            if (!std::isfinite(cb.projection.data()[k]))
                throw FormatError("non-finite values in stage " + std::to_string(i), stage_off);
    }
    st.validate();
    // refresh on load (codebook.cpp:312): one device upload for the whole stack
    vqkv_stack_t h = st.device();
    for (uint32_t i = 0; i < n; ++i) {
        Codebook& cb = st.stages[i];
        cb.effective.resize(cb.size(), cb.dim());
        cb.effective_sqnorm.resize(cb.size());
        detail::check(vqkv_stack_effective(h, i, cb.effective.data(), cb.effective_sqnorm.data()));
    }
    return st;
}

inline CodebookStack load_stack(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    return load_stack(in);
}

/// FNV-1a-64 over the serialized stack (codebook.cpp:326-336).
inline uint64_t stack_content_hash(const CodebookStack& stack) {
    std::ostringstream buf(std::ios::binary);
    save_stack(stack, buf);
    const std::string b = buf.str();
    return vqkv_fnv1a64(reinterpret_cast<const uint8_t*>(b.data()), b.size());
}

}  // namespace vqkv
