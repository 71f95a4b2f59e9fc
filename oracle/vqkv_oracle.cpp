// vqkv_oracle.cpp -- CPU ORACLE for the VQKV hot path.  TEST INFRASTRUCTURE ONLY.
//
// A plain-C++ restatement (no Eigen available in this image) of the reference
// implementation under /root/reference/proj.  Every function cites the
// reference file:line it follows.  The reference itself cannot be built here
// (it needs Eigen 3.4, doctest and CLI11, none of which are present), so the
// arithmetic that Eigen performs is restated explicitly:
//
//  * row-major GEMV (Eigen 3.4 GeneralMatrixVector.h, SSE2 packet of 4 floats,
//    no FMA because the reference CMake passes no -march): per output row, four
//    lane accumulators c[l] += a[j+l]*b[j+l] (multiply, then add), combined by
//    predux = (c0+c2)+(c1+c3), then a scalar tail.              -> gemv_dot()
//  * vectorised reductions (Redux.h LinearVectorizedTraversal, alignedStart=0
//    because cwiseAbs2()/binary products carry no DirectAccessBit): two packet
//    accumulators over 8-float strides, combined, predux, scalar tail.
//                                                                 -> redux_dot()
//  * a GEMV whose matrix has one row falls back to dot() (ProductEvaluators.h,
//    "Fallback to inner product"), so a search block of length 1 scores with
//    redux_dot() instead of gemv_dot().
//
// Build: oracle/Makefile (g++ -O3 -ffp-contract=off, no -march, like
// proj/core/CMakeLists.txt).  Nothing in the product links this file.

#include "vqkv_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <fstream>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---- errors (proj/core/include/vqkv/errors.hpp:12-49) -----------------------
struct Error : std::runtime_error {
    int code;
    uint64_t offset = 0;
    Error(int c, const std::string& m, uint64_t off = 0) : std::runtime_error(m), code(c), offset(off) {}
};
[[noreturn]] void invalid_input(const std::string& m) { throw Error(ORC_INVALID_INPUT, m); }
[[noreturn]] void invalid_state(const std::string& m) { throw Error(ORC_INVALID_STATE, m); }
[[noreturn]] void invalid_code(const std::string& m) { throw Error(ORC_INVALID_CODE, m); }
[[noreturn]] void format_error(const std::string& m, uint64_t off) {
    throw Error(ORC_FORMAT_ERROR, m + " (byte offset " + std::to_string(off) + ")", off);
}

thread_local std::string g_err;
thread_local uint64_t g_err_off = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        return ORC_OK;
    } catch (const Error& e) {
        g_err = e.what();
        g_err_off = e.offset;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ORC_OTHER;
    }
}

// ---- Eigen arithmetic restatements -------------------------------------------
// Row-major GEMV, one output row (GeneralMatrixVector.h, Eigen 3.4, SSE2).
inline float gemv_dot(const float* a, const float* b, int64_t n) {
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    int64_t j = 0;
    for (; j + 4 <= n; j += 4) {
        c0 = c0 + a[j + 0] * b[j + 0];
        c1 = c1 + a[j + 1] * b[j + 1];
        c2 = c2 + a[j + 2] * b[j + 2];
        c3 = c3 + a[j + 3] * b[j + 3];
    }
    float cc = (c0 + c2) + (c1 + c3);
    for (; j < n; ++j) cc += a[j] * b[j];
    return cc;
}

// Redux.h LinearVectorizedTraversal with alignedStart = 0 over p(i) = a[i]*b[i].
inline float redux_dot(const float* a, const float* b, int64_t n) {
    const int64_t aligned = (n / 4) * 4, aligned2 = (n / 8) * 8;
    float res;
    if (aligned) {
        float r0[4], r1[4];
        for (int l = 0; l < 4; ++l) r0[l] = a[l] * b[l];
        if (aligned > 4) {
            for (int l = 0; l < 4; ++l) r1[l] = a[4 + l] * b[4 + l];
            for (int64_t i = 8; i < aligned2; i += 8) {
                for (int l = 0; l < 4; ++l) r0[l] = r0[l] + a[i + l] * b[i + l];
                for (int l = 0; l < 4; ++l) r1[l] = r1[l] + a[i + 4 + l] * b[i + 4 + l];
            }
            for (int l = 0; l < 4; ++l) r0[l] = r0[l] + r1[l];
            if (aligned > aligned2)
                for (int l = 0; l < 4; ++l) r0[l] = r0[l] + a[aligned2 + l] * b[aligned2 + l];
        }
        res = (r0[0] + r0[2]) + (r0[1] + r0[3]);
        for (int64_t i = aligned; i < n; ++i) res = res + a[i] * b[i];
    } else {
        res = a[0] * b[0];
        for (int64_t i = 1; i < n; ++i) res = res + a[i] * b[i];
    }
    return res;
}
inline float squared_norm(const float* a, int64_t n) { return n ? redux_dot(a, a, n) : 0.f; }

// ---- bitpack (proj/core/include/vqkv/bitpack.hpp:14-45) ---------------------
void bit_write(std::vector<uint8_t>& buf, size_t pos0, uint32_t value, unsigned width) {
    size_t need = (pos0 + width + 7) / 8;
    if (buf.size() < need) buf.resize(need, 0);
    for (unsigned b = 0; b < width; ++b) {
        size_t pos = pos0 + b;
        if ((value >> b) & 1u)
            buf[pos / 8] |= uint8_t(1u << (pos % 8));
        else
            buf[pos / 8] &= uint8_t(~(1u << (pos % 8)));
    }
}
uint32_t bit_read(const uint8_t* buf, size_t pos0, unsigned width) {
    uint32_t v = 0;
    for (unsigned b = 0; b < width; ++b) {
        size_t pos = pos0 + b;
        v |= uint32_t((buf[pos / 8] >> (pos % 8)) & 1u) << b;
    }
    return v;
}
unsigned index_bit_width(uint32_t size) {
    unsigned w = 0;
    while ((uint64_t(1) << w) < size) ++w;
    return w;
}

// ---- Codebook / stack (codebook.hpp:30-56, codebook.cpp:30-72) --------------
struct Codebook {
    int64_t S = 0, D = 0;
    std::vector<float> entries, projection, effective, sqnorm;
    // codebook.cpp:30-39: effective.row(i) = entries.row(i) * projection^T,
    // one row at a time (row-major GEMV with the projection as the matrix).
    void refresh() {
        effective.assign(size_t(S * D), 0.f);
        sqnorm.assign(size_t(S), 0.f);
        for (int64_t i = 0; i < S; ++i) {
            const float* e = &entries[size_t(i * D)];
            for (int64_t k = 0; k < D; ++k) {
                const float* p = &projection[size_t(k * D)];
                // D == 1: the 1x1 product takes the dot() fallback; identical value.
                effective[size_t(i * D + k)] = (D == 1) ? redux_dot(p, e, D) : gemv_dot(p, e, D);
            }
            sqnorm[size_t(i)] = squared_norm(&effective[size_t(i * D)], D);
        }
    }
    void validate() const {  // codebook.cpp:41-51
        if (S < 1 || D < 1) invalid_input("codebook must have S >= 1 and D >= 1");
        for (float v : entries)
            if (!std::isfinite(v)) invalid_input("codebook contains non-finite values");
        for (float v : projection)
            if (!std::isfinite(v)) invalid_input("codebook contains non-finite values");
    }
};

}  // namespace orc

struct orc_stack {
    std::vector<orc::Codebook> stages;
    int kind = 0;
    int64_t dim() const { return stages.empty() ? 0 : stages.front().D; }
    std::vector<uint32_t> sizes() const {
        std::vector<uint32_t> s;
        for (auto& c : stages) s.push_back(uint32_t(c.S));
        return s;
    }
    void validate() const {  // codebook.cpp:62-72
        if (stages.empty()) orc::invalid_input("stack must have at least one stage");
        for (auto& st : stages) {
            st.validate();
            if (st.D != dim()) orc::invalid_input("all stages must share one dimension");
        }
    }
};

namespace orc {

// ---- CodeMatrix (codebook.hpp:63-91, codebook.cpp:74-151) -------------------
struct CodeMatrix {
    std::vector<uint32_t> sizes;
    std::vector<unsigned> bits;
    std::vector<size_t> offs;
    size_t row_bits = 0, rows = 0;
    std::vector<uint8_t> payload;
    CodeMatrix() = default;
    explicit CodeMatrix(std::vector<uint32_t> s) : sizes(std::move(s)) {
        for (uint32_t v : sizes) {
            if (v < 1) invalid_input("stage size must be >= 1");
            offs.push_back(row_bits);
            unsigned w = index_bit_width(v);
            bits.push_back(w);
            row_bits += w;
        }
    }
    void append(const std::vector<uint32_t>& codes) {
        if (codes.size() != sizes.size()) invalid_input("code vector has wrong stage count");
        for (size_t i = 0; i < codes.size(); ++i)
            if (codes[i] >= sizes[i])
                invalid_code("index " + std::to_string(codes[i]) + " out of range for stage " +
                             std::to_string(i));
        size_t base = rows * row_bits;
        for (size_t i = 0; i < codes.size(); ++i) bit_write(payload, base + offs[i], codes[i], bits[i]);
        ++rows;
    }
    std::vector<uint32_t> row(size_t r) const {
        if (r >= rows) invalid_input("row " + std::to_string(r) + " out of range");
        std::vector<uint32_t> c(sizes.size());
        for (size_t i = 0; i < c.size(); ++i) c[i] = bit_read(payload.data(), r * row_bits + offs[i], bits[i]);
        return c;
    }
    uint64_t payload_bits() const { return rows * row_bits; }
    void load_payload(const uint8_t* p, size_t n_rows) {
        rows = n_rows;
        payload.assign(p, p + (rows * row_bits + 7) / 8);
    }
};

// ---- search / quantize / reconstruct (codebook.cpp:158-250) -----------------
struct Nearest {
    uint32_t index;
    float score;
};

// codebook.cpp:158-176; optionally reports the second-best score.
Nearest nearest_scored(const Codebook& cb, const float* x, size_t search_block, float* second = nullptr) {
    float best = std::numeric_limits<float>::infinity();
    float sec = std::numeric_limits<float>::infinity();
    uint32_t best_idx = 0;
    const int64_t n = cb.S;
    if (search_block == 0) invalid_input("search_block must be >= 1");
    for (int64_t begin = 0; begin < n; begin += int64_t(search_block)) {
        int64_t len = std::min<int64_t>(int64_t(search_block), n - begin);
        for (int64_t i = 0; i < len; ++i) {
            const float* e = &cb.effective[size_t((begin + i) * cb.D)];
            float dot = (len == 1) ? redux_dot(e, x, cb.D) : gemv_dot(e, x, cb.D);
            float score = cb.sqnorm[size_t(begin + i)] - 2.0f * dot;
            if (score < best) {
                sec = best;
                best = score;
                best_idx = uint32_t(begin + i);
            } else if (score < sec) {
                sec = score;
            }
        }
    }
    if (second) *second = sec;
    return {best_idx, best};
}

void check_dim(const orc_stack& st, int64_t got) {  // codebook.cpp:21-26
    if (got != st.dim())
        invalid_input("vector dimension " + std::to_string(got) + " does not match stack dimension " +
                      std::to_string(st.dim()));
}

// codebook.cpp:194-206
void quantize(const orc_stack& st, const float* x, size_t sb, uint32_t* codes, float* residual,
              float* best = nullptr, float* second = nullptr, float* rnorm = nullptr) {
    const int64_t D = st.dim();
    std::memcpy(residual, x, sizeof(float) * size_t(D));
    for (size_t s = 0; s < st.stages.size(); ++s) {
        const Codebook& cb = st.stages[s];
        if (rnorm) rnorm[s] = std::sqrt(squared_norm(residual, D));
        float sec;
        Nearest n = nearest_scored(cb, residual, sb, &sec);
        if (best) best[s] = n.score;
        if (second) second[s] = sec;
        codes[s] = n.index;
        const float* e = &cb.effective[size_t(n.index) * size_t(D)];
        for (int64_t k = 0; k < D; ++k) residual[k] = residual[k] - e[k];
    }
}

// codebook.cpp:208-223
void reconstruct(const orc_stack& st, const uint32_t* codes, size_t n_codes, float* out) {
    if (n_codes != st.stages.size())
        invalid_code("code vector has " + std::to_string(n_codes) + " stages, stack has " +
                     std::to_string(st.stages.size()));
    const int64_t D = st.dim();
    for (int64_t k = 0; k < D; ++k) out[k] = 0.f;
    for (size_t i = 0; i < n_codes; ++i) {
        const Codebook& cb = st.stages[i];
        if (codes[i] >= uint32_t(cb.S))
            invalid_code("index " + std::to_string(codes[i]) + " out of range for stage " + std::to_string(i));
        const float* e = &cb.effective[size_t(codes[i]) * size_t(D)];
        for (int64_t k = 0; k < D; ++k) out[k] = out[k] + e[k];
    }
}

// codebook.cpp:225-237
CodeMatrix quantize_batch(const orc_stack& st, const float* xs, size_t rows, int64_t xdim, size_t sb,
                          float* norms, float* best = nullptr, float* second = nullptr,
                          float* rnorm = nullptr) {
    if (rows > 0) check_dim(st, xdim);
    CodeMatrix cm(st.sizes());
    const size_t N = st.stages.size();
    const int64_t D = st.dim();
    std::vector<uint32_t> codes(N);
    std::vector<float> r(size_t(std::max<int64_t>(D, 1)));
    for (size_t i = 0; i < rows; ++i) {
        quantize(st, xs + i * size_t(D), sb, codes.data(), r.data(), best ? best + i * N : nullptr,
                 second ? second + i * N : nullptr, rnorm ? rnorm + i * N : nullptr);
        cm.append(codes);
        norms[i] = std::sqrt(squared_norm(r.data(), D));
    }
    return cm;
}

// codebook.cpp:239-250
void reconstruct_block(const orc_stack& st, const CodeMatrix& cm, size_t begin, size_t end, float* out) {
    if (begin > end || end > cm.rows)
        invalid_input("row range [" + std::to_string(begin) + ", " + std::to_string(end) +
                      ") out of bounds for " + std::to_string(cm.rows) + " rows");
    const int64_t D = st.dim();
    for (size_t r = begin; r < end; ++r) {
        std::vector<uint32_t> c = cm.row(r);
        reconstruct(st, c.data(), c.size(), out + (r - begin) * size_t(D));
    }
}

// ---- RSVQ container (codebook.cpp:252-336, io_util.hpp) ----------------------
template <class T>
void put(std::ostream& o, T v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
T get(std::istream& in, uint64_t& off, const char* what) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) format_error(std::string("truncated file reading ") + what, off);
    off += sizeof(T);
    return v;
}
void get_bytes(std::istream& in, void* d, size_t n, uint64_t& off, const char* what) {
    in.read(reinterpret_cast<char*>(d), std::streamsize(n));
    if (!in) format_error(std::string("truncated file reading ") + what, off);
    off += n;
}

void save_stack(const orc_stack& st, std::ostream& out) {
    st.validate();
    out.write("RSVQ", 4);
    put<uint32_t>(out, 1);
    put<uint8_t>(out, uint8_t(st.kind));
    put<uint32_t>(out, uint32_t(st.stages.size()));
    for (auto& cb : st.stages) {
        put<uint32_t>(out, uint32_t(cb.S));
        put<uint32_t>(out, uint32_t(cb.D));
        out.write(reinterpret_cast<const char*>(cb.entries.data()), std::streamsize(4 * cb.entries.size()));
        out.write(reinterpret_cast<const char*>(cb.projection.data()),
                  std::streamsize(4 * cb.projection.size()));
    }
}

orc_stack load_stack(std::istream& in) {
    uint64_t off = 0;
    char magic[4] = {};
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "RSVQ", 4) != 0) format_error("bad magic, expected RSVQ", off);
    off += 4;
    auto version = get<uint32_t>(in, off, "version");
    if (version != 1) format_error("unsupported version " + std::to_string(version), off - 4);
    auto kind = get<uint8_t>(in, off, "cache kind");
    if (kind > 1) format_error("bad cache kind " + std::to_string(kind), off - 1);
    auto n = get<uint32_t>(in, off, "stage count");
    if (n < 1) format_error("stage count must be >= 1", off - 4);
    orc_stack st;
    st.kind = kind;
    st.stages.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        auto s = get<uint32_t>(in, off, "codebook size");
        auto d = get<uint32_t>(in, off, "dimension");
        if (s < 1 || d < 1) format_error("codebook size and dimension must be >= 1", off - 8);
        uint64_t stage_off = off;
        Codebook& cb = st.stages[i];
        cb.S = s;
        cb.D = d;
        cb.entries.resize(size_t(s) * d);
        get_bytes(in, cb.entries.data(), 4 * cb.entries.size(), off, "entries");
        cb.projection.resize(size_t(d) * d);
        get_bytes(in, cb.projection.data(), 4 * cb.projection.size(), off, "projection");
        for (float v : cb.entries)
            if (!std::isfinite(v)) format_error("non-finite values in stage " + std::to_string(i), stage_off);
        for (float v : cb.projection)
            if (!std::isfinite(v)) format_error("non-finite values in stage " + std::to_string(i), stage_off);
        cb.refresh();
    }
    st.validate();
    return st;
}

uint64_t fnv1a(const std::string& bytes) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : bytes) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

// ---- synthetic (synthetic.cpp:11-63) ----------------------------------------
void rope_rotate_row(float* row, int64_t d, int64_t position, double base) {
    for (int64_t i = 0; i < d / 2; ++i) {
        double freq = std::pow(base, -2.0 * double(i) / double(d));
        double angle = double(position) * freq;
        float c = float(std::cos(angle));
        float s = float(std::sin(angle));
        float a = row[2 * i], b = row[2 * i + 1];
        row[2 * i] = a * c - b * s;
        row[2 * i + 1] = a * s + b * c;
    }
}

void generate(int kind, int64_t dim, int64_t count, uint32_t comps, uint64_t seed, double base, float cstd,
              float mscale, float* out) {
    if (dim < 1 || count < 1 || comps < 1) invalid_input("dim, count and component_count must be >= 1");
    if (kind == 1 && dim % 2 != 0) invalid_input("rope_rotated_keys requires an even dimension");
    if (base <= 0.0) invalid_input("rope_base must be positive");
    if (cstd < 0.0f || mscale < 0.0f) invalid_input("component_std and mean_scale must be nonnegative");
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    std::uniform_int_distribution<uint32_t> pick(0, comps - 1);
    std::vector<float> means(size_t(comps) * size_t(dim));
    for (auto& m : means) m = mscale * gauss(rng);
    for (int64_t r = 0; r < count; ++r) {
        uint32_t c = pick(rng);
        float* row = out + size_t(r) * size_t(dim);
        for (int64_t j = 0; j < dim; ++j) row[j] = means[size_t(c) * size_t(dim) + size_t(j)] + cstd * gauss(rng);
        if (kind == 1) rope_rotate_row(row, dim, r, base);
    }
}

// ---- kv cache (kv_cache.hpp:14-108, kv_cache.cpp:41-204) --------------------
struct Cache {
    const orc_stack* ks;
    const orc_stack* vs;
    uint64_t init_len, local_len;
    bool eager;
    bool prefilled = false;
    int64_t kd, vd;
    std::vector<float> init_k, init_v;  // rows x dim
    CodeMatrix kc, vc;
    std::vector<float> kn, vn;
    std::deque<std::vector<float>> pend_k, pend_v, loc_k, loc_v;
    uint64_t batched = 0;

    Cache(const orc_stack* k, const orc_stack* v, uint64_t il, uint64_t ll, bool e)
        : ks(k), vs(v), init_len(il), local_len(ll), eager(e), kd(k->dim()), vd(v->dim()),
          kc(k->sizes()), vc(v->sizes()) {
        if (local_len < 1) invalid_input("local_len must be >= 1");  // kv_cache.cpp:41-45
        k->validate();
        v->validate();
    }
    uint64_t init_rows() const { return init_k.size() / size_t(kd); }
    uint64_t comp_rows() const { return kc.rows; }
    uint64_t total() const { return init_rows() + comp_rows() + pend_k.size() + loc_k.size(); }

    void prefill(const float* keys, const float* values, int64_t rows, int64_t kdim, int64_t vdim) {
        if (total() != 0 || prefilled) invalid_state("prefill requires an empty cache");
        if (rows < 1) invalid_input("prefill needs at least one token");
        if (kdim != kd || vdim != vd) invalid_input("key/value dimensions do not match the stacks");
        const uint64_t len = uint64_t(rows);
        const uint64_t n_init = std::min(init_len, len);
        const uint64_t n_local = std::min(local_len, len - n_init);
        const uint64_t n_mid = len - n_init - n_local;
        init_k.assign(keys, keys + n_init * kd);
        init_v.assign(values, values + n_init * vd);
        if (n_mid > 0) {
            kn.resize(n_mid);
            vn.resize(n_mid);
            kc = quantize_batch(*ks, keys + n_init * kd, n_mid, kd, 4096, kn.data());
            vc = quantize_batch(*vs, values + n_init * vd, n_mid, vd, 4096, vn.data());
        }
        for (uint64_t i = len - n_local; i < len; ++i) {
            loc_k.emplace_back(keys + i * kd, keys + (i + 1) * kd);
            loc_v.emplace_back(values + i * vd, values + (i + 1) * vd);
        }
        prefilled = true;
    }
    void flush() {  // kv_cache.cpp:102-120
        const size_t n = pend_k.size();
        std::vector<float> k(n * kd), v(n * vd), kn2(n), vn2(n);
        for (size_t i = 0; i < n; ++i) {
            std::copy(pend_k[i].begin(), pend_k[i].end(), k.begin() + i * kd);
            std::copy(pend_v[i].begin(), pend_v[i].end(), v.begin() + i * vd);
        }
        CodeMatrix a = quantize_batch(*ks, k.data(), n, kd, 4096, kn2.data());
        CodeMatrix b = quantize_batch(*vs, v.data(), n, vd, 4096, vn2.data());
        for (size_t i = 0; i < n; ++i) {
            kc.append(a.row(i));
            vc.append(b.row(i));
            kn.push_back(kn2[i]);
            vn.push_back(vn2[i]);
        }
        pend_k.clear();
        pend_v.clear();
        ++batched;
    }
    void append(const float* key, int64_t kdim, const float* value, int64_t vdim) {  // :122-141
        if (!prefilled && init_len != 0) invalid_state("append_token requires a prefilled cache (or init_len == 0)");
        if (kdim != kd || vdim != vd) invalid_input("key/value dimensions do not match the stacks");
        loc_k.emplace_back(key, key + kd);
        loc_v.emplace_back(value, value + vd);
        if (loc_k.size() > local_len) {
            pend_k.push_back(std::move(loc_k.front()));
            pend_v.push_back(std::move(loc_v.front()));
            loc_k.pop_front();
            loc_v.pop_front();
            if (eager || pend_k.size() >= local_len) flush();
        }
    }
    // kv_cache.cpp:143-189
    void view_block(uint64_t begin, uint64_t end, float* keys, float* values, uint8_t* exact) const {
        const uint64_t len = total();
        if (begin > end || end > len)
            invalid_input("view range [" + std::to_string(begin) + ", " + std::to_string(end) +
                          ") out of bounds for length " + std::to_string(len));
        const uint64_t ie = init_rows(), ce = ie + comp_rows(), pe = ce + pend_k.size();
        uint64_t g = begin;
        while (g < end) {
            uint64_t dst = g - begin;
            if (g < ie) {
                uint64_t stop = std::min(end, ie);
                std::copy(init_k.begin() + g * kd, init_k.begin() + stop * kd, keys + dst * kd);
                std::copy(init_v.begin() + g * vd, init_v.begin() + stop * vd, values + dst * vd);
                for (uint64_t i = g; i < stop; ++i) exact[i - begin] = 1;
                g = stop;
            } else if (g < ce) {
                uint64_t stop = std::min(end, ce);
                reconstruct_block(*ks, kc, g - ie, stop - ie, keys + dst * kd);
                reconstruct_block(*vs, vc, g - ie, stop - ie, values + dst * vd);
                for (uint64_t i = g; i < stop; ++i) exact[i - begin] = 0;
                g = stop;
            } else if (g < pe) {
                std::copy(pend_k[g - ce].begin(), pend_k[g - ce].end(), keys + dst * kd);
                std::copy(pend_v[g - ce].begin(), pend_v[g - ce].end(), values + dst * vd);
                exact[dst] = 1;
                ++g;
            } else {
                std::copy(loc_k[g - pe].begin(), loc_k[g - pe].end(), keys + dst * kd);
                std::copy(loc_v[g - pe].begin(), loc_v[g - pe].end(), values + dst * vd);
                exact[dst] = 1;
                ++g;
            }
        }
    }
};

// attention.cpp:14-16
double effective_scale(double scale, int64_t kdim) { return scale > 0.0 ? scale : 1.0 / std::sqrt(double(kdim)); }

// Logit of one row: (scale*A)*q with A cast to double; Eigen folds "s*(A*q)"
// into the lhs, and the cast makes the row reduction sequential (non-vector).
inline double logit_row(const float* k, const double* q, int64_t d, double scale) {
    double res = (scale * double(k[0])) * q[0];
    for (int64_t i = 1; i < d; ++i) res = res + (scale * double(k[i])) * q[i];
    return 0.0 + res;
}

// Online-softmax accumulator shared by attend() and attend_segments().
struct Online {
    double running_max = -std::numeric_limits<double>::infinity();
    double normalizer = 0.0;
    std::vector<double> acc;
    explicit Online(int64_t vd) : acc(size_t(vd), 0.0) {}
    // attention.cpp:55-66
    void block(const float* keys, const float* values, size_t n, int64_t kd, int64_t vd, const double* q,
               double scale) {
        std::vector<double> logits(n);
        for (size_t j = 0; j < n; ++j) logits[j] = logit_row(keys + j * kd, q, kd, scale);
        double bmax = logits[0];
        for (size_t j = 1; j < n; ++j) bmax = std::max(bmax, logits[j]);
        double new_max = std::max(running_max, bmax);
        double rescale = std::exp(running_max - new_max);
        normalizer *= rescale;
        for (auto& a : acc) a *= rescale;
        for (size_t j = 0; j < n; ++j) {
            double p = std::exp(logits[j] - new_max);
            normalizer += p;
            for (int64_t d = 0; d < vd; ++d) acc[size_t(d)] = acc[size_t(d)] + p * double(values[j * vd + d]);
        }
        running_max = new_max;
    }
    void finish(float* out) const {
        for (size_t d = 0; d < acc.size(); ++d) out[d] = float(acc[d] / normalizer);
    }
};

// attention.cpp:26-69
void attend(const Cache& c, const float* q, int64_t qdim, uint64_t block_rows, double scale_cfg, float* out,
            uint64_t* peak, uint64_t* nrec) {
    if (block_rows < 1) invalid_input("block_rows must be >= 1");
    if (c.total() < 1) invalid_state("cannot attend over an empty cache");
    if (qdim != c.kd) invalid_input("query dimension does not match key dimension");
    const double scale = effective_scale(scale_cfg, c.kd);
    std::vector<double> qd(static_cast<size_t>(qdim));
    for (int64_t i = 0; i < qdim; ++i) qd[size_t(i)] = double(q[i]);
    Online on(c.vd);
    const uint64_t len = c.total();
    std::vector<float> bk, bv;
    std::vector<uint8_t> ex;
    for (uint64_t begin = 0; begin < len; begin += block_rows) {
        uint64_t stop = std::min(len, begin + block_rows);
        size_t n = size_t(stop - begin);
        bk.resize(n * c.kd);
        bv.resize(n * c.vd);
        ex.resize(n);
        c.view_block(begin, stop, bk.data(), bv.data(), ex.data());
        uint64_t lossy = 0;
        for (auto e : ex) lossy += e ? 0 : 1;
        if (peak) *peak = std::max<uint64_t>(*peak, lossy * uint64_t(c.kd + c.vd));
        if (nrec) *nrec += lossy;
        on.block(bk.data(), bv.data(), n, c.kd, c.vd, qd.data(), scale);
    }
    on.finish(out);
}

// attention.cpp:71-88
void attend_raw(const float* keys, const float* values, int64_t rows, int64_t kd, int64_t vd, const float* q,
                int64_t qdim, double scale_cfg, float* out) {
    if (rows < 1) invalid_input("keys and values must be nonempty and the same length");
    if (qdim != kd) invalid_input("query dimension does not match key dimension");
    const double scale = effective_scale(scale_cfg, kd);
    std::vector<double> qd(static_cast<size_t>(qdim));
    for (int64_t i = 0; i < qdim; ++i) qd[size_t(i)] = double(q[i]);
    std::vector<double> w(static_cast<size_t>(rows));
    for (int64_t j = 0; j < rows; ++j) w[size_t(j)] = logit_row(keys + j * kd, qd.data(), kd, scale);
    double mx = w[0];
    for (auto v : w) mx = std::max(mx, v);
    for (auto& v : w) v = std::exp(v - mx);
    // VectorXd::sum(): Packet2d redux, alignedStart 0.
    const int64_t n = rows, al = (n / 2) * 2, al2 = (n / 4) * 4;
    double sum;
    if (al) {
        double r0[2] = {w[0], w[1]}, r1[2];
        if (al > 2) {
            r1[0] = w[2];
            r1[1] = w[3];
            for (int64_t i = 4; i < al2; i += 4) {
                r0[0] += w[size_t(i)];
                r0[1] += w[size_t(i + 1)];
                r1[0] += w[size_t(i + 2)];
                r1[1] += w[size_t(i + 3)];
            }
            r0[0] += r1[0];
            r0[1] += r1[1];
            if (al > al2) {
                r0[0] += w[size_t(al2)];
                r0[1] += w[size_t(al2 + 1)];
            }
        }
        sum = r0[0] + r0[1];
        for (int64_t i = al; i < n; ++i) sum += w[size_t(i)];
    } else {
        sum = w[0];
    }
    for (auto& v : w) v /= sum;
    std::vector<double> o(static_cast<size_t>(vd), 0.0);
    for (int64_t k = 0; k < rows; ++k)
        for (int64_t d = 0; d < vd; ++d) o[size_t(d)] = o[size_t(d)] + w[size_t(k)] * double(values[k * vd + d]);
    for (int64_t d = 0; d < vd; ++d) out[d] = float(o[size_t(d)]);
}

}  // namespace orc

struct orc_rng {
    std::mt19937_64 g;
};
struct orc_cache {
    orc::Cache c;
};

using namespace orc;

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
uint64_t orc_last_error_offset(void) { return g_err_off; }

orc_rng* orc_rng_new(uint64_t seed) { return new orc_rng{std::mt19937_64(seed)}; }
void orc_rng_free(orc_rng* r) { delete r; }
uint64_t orc_rng_next(orc_rng* r) { return r->g(); }

void orc_random_matrix(orc_rng* r, int64_t rows, int64_t cols, float scale, float* out) {
    std::normal_distribution<float> gauss(0.0f, 1.0f);  // test_util.hpp:51-59
    for (int64_t i = 0; i < rows * cols; ++i) out[i] = scale * gauss(r->g);
}

orc_stack* orc_random_stack(orc_rng* r, uint32_t n, uint32_t size, int64_t dim, int kind) {
    std::normal_distribution<float> gauss(0.0f, 1.0f);  // test_util.hpp:30-50
    auto* st = new orc_stack;
    st->kind = kind;
    float proj_scale = 1.0f / std::sqrt(static_cast<float>(dim));
    for (uint32_t s = 0; s < n; ++s) {
        Codebook cb;
        cb.S = size;
        cb.D = dim;
        cb.entries.resize(size_t(size) * size_t(dim));
        for (auto& v : cb.entries) v = gauss(r->g);
        cb.projection.resize(size_t(dim) * size_t(dim));
        for (auto& v : cb.projection) v = proj_scale * gauss(r->g);
        cb.refresh();
        st->stages.push_back(std::move(cb));
    }
    return st;
}

orc_stack* orc_stack_new(uint32_t n, const uint32_t* sizes, int64_t dim, const float* entries,
                         const float* projections, int kind) {
    auto* st = new orc_stack;
    st->kind = kind;
    size_t eoff = 0;
    for (uint32_t s = 0; s < n; ++s) {
        Codebook cb;
        cb.S = sizes[s];
        cb.D = dim;
        cb.entries.assign(entries + eoff, entries + eoff + size_t(cb.S) * size_t(dim));
        eoff += size_t(cb.S) * size_t(dim);
        cb.projection.assign(size_t(dim) * size_t(dim), 0.f);
        if (projections)
            std::copy(projections + size_t(s) * dim * dim, projections + size_t(s + 1) * dim * dim,
                      cb.projection.begin());
        else
            for (int64_t i = 0; i < dim; ++i) cb.projection[size_t(i * dim + i)] = 1.f;
        cb.refresh();
        st->stages.push_back(std::move(cb));
    }
    return st;
}
void orc_stack_free(orc_stack* s) { delete s; }
uint32_t orc_stack_num_stages(const orc_stack* s) { return uint32_t(s->stages.size()); }
int64_t orc_stack_dim(const orc_stack* s) { return s->dim(); }
uint32_t orc_stack_stage_size(const orc_stack* s, uint32_t i) { return uint32_t(s->stages[i].S); }
int orc_stack_kind(const orc_stack* s) { return s->kind; }
void orc_stack_get_entries(const orc_stack* s, uint32_t i, float* o) {
    std::copy(s->stages[i].entries.begin(), s->stages[i].entries.end(), o);
}
void orc_stack_get_projection(const orc_stack* s, uint32_t i, float* o) {
    std::copy(s->stages[i].projection.begin(), s->stages[i].projection.end(), o);
}
void orc_stack_get_effective(const orc_stack* s, uint32_t i, float* o) {
    std::copy(s->stages[i].effective.begin(), s->stages[i].effective.end(), o);
}
void orc_stack_get_sqnorm(const orc_stack* s, uint32_t i, float* o) {
    std::copy(s->stages[i].sqnorm.begin(), s->stages[i].sqnorm.end(), o);
}
int orc_stack_save(const orc_stack* s, const char* path) {
    return guard([&] {
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error(ORC_IO_ERROR, std::string("cannot open ") + path + " for writing");
        save_stack(*s, out);
        if (!out) throw Error(ORC_IO_ERROR, std::string("write failed for ") + path);
    });
}
uint64_t orc_stack_serialize(const orc_stack* s, uint8_t* buf, uint64_t cap) {
    std::ostringstream o(std::ios::binary);
    if (guard([&] { save_stack(*s, o); }) != ORC_OK) return 0;
    std::string b = o.str();
    if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
    return b.size();
}
orc_stack* orc_stack_load(const char* path) {
    orc_stack* res = nullptr;
    guard([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error(ORC_IO_ERROR, std::string("cannot open ") + path);
        res = new orc_stack(load_stack(in));
    });
    return res;
}
orc_stack* orc_stack_load_bytes(const uint8_t* buf, uint64_t n) {
    orc_stack* res = nullptr;
    guard([&] {
        std::istringstream in(std::string(reinterpret_cast<const char*>(buf), size_t(n)), std::ios::binary);
        res = new orc_stack(load_stack(in));
    });
    return res;
}
uint64_t orc_stack_hash(const orc_stack* s) {
    std::ostringstream o(std::ios::binary);
    save_stack(*s, o);
    return fnv1a(o.str());
}

unsigned orc_index_bit_width(uint32_t size) { return index_bit_width(size); }
uint64_t orc_row_bits(uint32_t n, const uint32_t* sizes) {
    uint64_t b = 0;
    for (uint32_t i = 0; i < n; ++i) b += index_bit_width(sizes[i]);
    return b;
}
uint64_t orc_payload_bytes(uint32_t n, const uint32_t* sizes, uint64_t rows) {
    return (rows * orc_row_bits(n, sizes) + 7) / 8;
}
int orc_codes_pack(uint32_t n, const uint32_t* sizes, const uint32_t* codes, uint64_t rows, uint8_t* payload) {
    return guard([&] {
        CodeMatrix cm(std::vector<uint32_t>(sizes, sizes + n));
        for (uint64_t r = 0; r < rows; ++r) cm.append(std::vector<uint32_t>(codes + r * n, codes + (r + 1) * n));
        std::copy(cm.payload.begin(), cm.payload.end(), payload);
    });
}
int orc_codes_unpack(uint32_t n, const uint32_t* sizes, const uint8_t* payload, uint64_t rows, uint32_t* codes) {
    return guard([&] {
        CodeMatrix cm(std::vector<uint32_t>(sizes, sizes + n));
        cm.load_payload(payload, rows);
        for (uint64_t r = 0; r < rows; ++r) {
            auto c = cm.row(r);
            std::copy(c.begin(), c.end(), codes + r * n);
        }
    });
}

int orc_nearest_entry(const orc_stack* s, uint32_t stage, const float* x, int64_t xdim, uint64_t sb,
                      uint32_t* index, float* distance) {
    return guard([&] {  // codebook.cpp:180-192
        const Codebook& cb = s->stages[stage];
        if (xdim != cb.D)
            invalid_input("vector dimension " + std::to_string(xdim) + " does not match codebook dimension " +
                          std::to_string(cb.D));
        for (int64_t i = 0; i < xdim; ++i)
            if (!std::isfinite(x[i])) invalid_input("query vector contains non-finite values");
        Nearest n = nearest_scored(cb, x, sb);
        *index = n.index;
        *distance = std::sqrt(std::max(0.0f, n.score + squared_norm(x, xdim)));
    });
}
int orc_quantize(const orc_stack* s, const float* x, int64_t xdim, uint64_t sb, uint32_t* codes, float* res) {
    return guard([&] {
        check_dim(*s, xdim);
        quantize(*s, x, sb, codes, res);
    });
}
int orc_reconstruct(const orc_stack* s, const uint32_t* codes, uint64_t n, float* out) {
    return guard([&] { reconstruct(*s, codes, n, out); });
}
int orc_quantize_batch(const orc_stack* s, const float* xs, uint64_t rows, int64_t xdim, uint64_t sb,
                       uint8_t* payload, float* norms, float* best, float* second, float* rnorm) {
    return guard([&] {
        CodeMatrix cm = quantize_batch(*s, xs, rows, xdim, sb, norms, best, second, rnorm);
        std::copy(cm.payload.begin(), cm.payload.end(), payload);
    });
}
int orc_quantize_batch_mt(const orc_stack* s, const float* xs, uint32_t n_streams, uint64_t rps, uint64_t sb,
                          uint8_t* payload, float* norms, int threads) {
    const uint64_t pbytes = orc_payload_bytes(uint32_t(s->stages.size()), s->sizes().data(), rps);
    const int64_t D = s->dim();
    std::vector<int> status(n_streams, ORC_OK);
    auto work = [&](uint32_t first, uint32_t step) {
        for (uint32_t st = first; st < n_streams; st += step) {
            status[st] = guard([&] {
                CodeMatrix cm = quantize_batch(*s, xs + size_t(st) * rps * D, rps, D, sb, norms + size_t(st) * rps);
                std::copy(cm.payload.begin(), cm.payload.end(), payload + size_t(st) * pbytes);
            });
        }
    };
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, uint32_t(t), uint32_t(threads));
    for (auto& t : pool) t.join();
    for (int v : status)
        if (v) return v;
    return ORC_OK;
}
int orc_reconstruct_block(const orc_stack* s, const uint8_t* payload, uint64_t rows, uint64_t begin, uint64_t end,
                          float* out) {
    return guard([&] {
        CodeMatrix cm(s->sizes());
        cm.load_payload(payload, rows);
        reconstruct_block(*s, cm, begin, end, out);
    });
}
void orc_stage_max_norm(const orc_stack* s, float* out) {
    for (size_t i = 0; i < s->stages.size(); ++i) {
        float m = 0.f;
        for (float v : s->stages[i].sqnorm) m = std::max(m, v);
        out[i] = std::sqrt(m);
    }
}

int orc_generate(int kind, int64_t dim, int64_t count, uint32_t comps, uint64_t seed, double base, float cstd,
                 float mscale, float* out) {
    return guard([&] { generate(kind, dim, count, comps, seed, base, cstd, mscale, out); });
}

orc_cache* orc_cache_new(const orc_stack* k, const orc_stack* v, uint64_t il, uint64_t ll, int eager) {
    orc_cache* res = nullptr;
    guard([&] { res = new orc_cache{Cache(k, v, il, ll, eager != 0)}; });
    return res;
}
void orc_cache_free(orc_cache* c) { delete c; }
int orc_cache_prefill(orc_cache* c, const float* k, const float* v, int64_t rows, int64_t kd, int64_t vd) {
    return guard([&] { c->c.prefill(k, v, rows, kd, vd); });
}
int orc_cache_append(orc_cache* c, const float* k, int64_t kd, const float* v, int64_t vd) {
    return guard([&] { c->c.append(k, kd, v, vd); });
}
void orc_cache_counts(const orc_cache* c, uint64_t* o) {
    o[0] = c->c.init_rows();
    o[1] = c->c.comp_rows();
    o[2] = c->c.pend_k.size();
    o[3] = c->c.loc_k.size();
    o[4] = c->c.total();
    o[5] = c->c.batched;
}
int orc_cache_view_block(const orc_cache* c, uint64_t b, uint64_t e, float* k, float* v, uint8_t* ex) {
    return guard([&] { c->c.view_block(b, e, k, v, ex); });
}
void orc_cache_codes(const orc_cache* c, int which, uint8_t* payload, float* norms) {
    const CodeMatrix& cm = which ? c->c.vc : c->c.kc;
    const std::vector<float>& n = which ? c->c.vn : c->c.kn;
    if (payload) std::copy(cm.payload.begin(), cm.payload.end(), payload);
    if (norms) std::copy(n.begin(), n.end(), norms);
}
void orc_cache_memory_report(const orc_cache* cc, uint64_t* raw, uint64_t* bits, uint64_t* over, double* ratio) {
    const Cache& c = cc->c;  // kv_cache.cpp:191-204
    auto sbytes = [](const orc_stack* s) {
        uint64_t b = 4 + 4 + 1 + 4;
        for (auto& st : s->stages) b += 8 + 4 * uint64_t(st.entries.size() + st.projection.size());
        return b;
    };
    const uint64_t spt = uint64_t(c.kd + c.vd);
    *raw = c.total() * spt * 2;
    *bits = c.kc.payload_bits() + c.vc.payload_bits();
    *over = sbytes(c.ks) + sbytes(c.vs);
    *ratio = 0.0;
    if (c.comp_rows() > 0) *ratio = 1.0 - double(*bits) / double(c.comp_rows() * spt * 16);
}
int orc_attend(const orc_cache* c, const float* q, int64_t qd, uint64_t br, double scale, float* out,
               uint64_t* peak, uint64_t* nrec) {
    return guard([&] { attend(c->c, q, qd, br, scale, out, peak, nrec); });
}
int orc_attend_raw(const float* k, const float* v, int64_t rows, int64_t kd, int64_t vd, const float* q,
                   int64_t qd, double scale, float* out) {
    return guard([&] { attend_raw(k, v, rows, kd, vd, q, qd, scale, out); });
}
int orc_attend_segments(const orc_stack* kst, const orc_stack* vst, const float* ik, const float* iv,
                        uint64_t n_init, const uint8_t* kpay, const uint8_t* vpay, uint64_t n_comp,
                        const float* lk, const float* lv, uint64_t n_local, const float* q, double scale_cfg,
                        uint64_t block_rows, float* out, double* lse) {
    return guard([&] {
        const int64_t kd = kst->dim(), vd = vst->dim();
        if (block_rows < 1) invalid_input("block_rows must be >= 1");
        if (n_init + n_comp + n_local < 1) invalid_state("cannot attend over an empty cache");
        CodeMatrix kc(kst->sizes()), vc(vst->sizes());
        kc.load_payload(kpay, n_comp);
        vc.load_payload(vpay, n_comp);
        const double scale = effective_scale(scale_cfg, kd);
        std::vector<double> qd(static_cast<size_t>(kd));
        for (int64_t i = 0; i < kd; ++i) qd[size_t(i)] = double(q[i]);
        Online on(vd);
        const uint64_t len = n_init + n_comp + n_local;
        std::vector<float> bk, bv;
        for (uint64_t begin = 0; begin < len; begin += block_rows) {
            uint64_t stop = std::min(len, begin + block_rows);
            size_t n = size_t(stop - begin);
            bk.resize(n * kd);
            bv.resize(n * vd);
            for (uint64_t g = begin; g < stop; ++g) {
                float* kr = &bk[size_t(g - begin) * kd];
                float* vr = &bv[size_t(g - begin) * vd];
                if (g < n_init) {
                    std::copy(ik + g * kd, ik + (g + 1) * kd, kr);
                    std::copy(iv + g * vd, iv + (g + 1) * vd, vr);
                } else if (g < n_init + n_comp) {
                    reconstruct_block(*kst, kc, g - n_init, g - n_init + 1, kr);
                    reconstruct_block(*vst, vc, g - n_init, g - n_init + 1, vr);
                } else {
                    uint64_t l = g - n_init - n_comp;
                    std::copy(lk + l * kd, lk + (l + 1) * kd, kr);
                    std::copy(lv + l * vd, lv + (l + 1) * vd, vr);
                }
            }
            on.block(bk.data(), bv.data(), n, kd, vd, qd.data(), scale);
        }
        on.finish(out);
        if (lse) *lse = on.running_max + std::log(on.normalizer);
    });
}

}  // extern "C"

// ---- trainer (trainer.cpp:22-248), restated for the checker --------------------------------
namespace orc {
// one row of accumulate_loss (trainer.cpp:43-79): residual chain, loss sums, gradient outer products
void train_row(const orc_stack& st, const float* x, float beta, float gamma, bool sq_commit, double* sums,
               std::vector<float>* grad) {
    const size_t N = st.stages.size();
    const int64_t D = st.dim();
    std::vector<uint32_t> codes(N);
    std::vector<float> tmp(static_cast<size_t>(D));
    quantize(st, x, 4096, codes.data(), tmp.data());  // forward_pass (trainer.cpp:22-34)
    std::vector<std::vector<float>> r(N + 1, std::vector<float>(static_cast<size_t>(D)));
    std::memcpy(r[0].data(), x, sizeof(float) * size_t(D));
    for (size_t i = 0; i < N; ++i) {
        const float* e = &st.stages[i].effective[size_t(codes[i]) * size_t(D)];
        for (int64_t k = 0; k < D; ++k) r[i + 1][size_t(k)] = r[i][size_t(k)] - e[k];
    }
    std::vector<float> sq(N);
    for (size_t i = 0; i < N; ++i) sq[i] = squared_norm(r[i + 1].data(), D);
    sums[0] += double(sq[N - 1]);
    for (size_t i = 0; i < N; ++i) {
        const double s = double(sq[i]);
        sums[1] += s;
        sums[2] += sq_commit ? s : std::sqrt(s);
        sums[3 + i] += s;
    }
    if (!grad) return;
    const std::vector<float>& fin = r[N];
    std::vector<float> suffix(static_cast<size_t>(D), 0.f);
    std::vector<std::vector<float>> gev(N, std::vector<float>(static_cast<size_t>(D)));
    for (size_t i = N; i-- > 0;) {
        const float b2 = 2.0f * beta;
        const float norm = std::sqrt(sq[i]);
        for (int64_t k = 0; k < D; ++k) {
            gev[i][size_t(k)] = (-2.0f * fin[size_t(k)] - b2 * r[i + 1][size_t(k)]) - gamma * suffix[size_t(k)];
            const float step = sq_commit ? 2.0f * r[i + 1][size_t(k)] : (norm > 0.0f ? r[i + 1][size_t(k)] / norm : 0.0f);
            suffix[size_t(k)] = suffix[size_t(k)] + step;
        }
    }
    for (size_t i = 0; i < N; ++i) {
        const float* ent = &st.stages[i].entries[size_t(codes[i]) * size_t(D)];
        float* g = grad[i].data();
        for (int64_t a = 0; a < D; ++a)
            for (int64_t b = 0; b < D; ++b) g[size_t(a * D + b)] = g[size_t(a * D + b)] + gev[i][size_t(a)] * ent[b];
    }
}
}  // namespace orc

extern "C" {
int orc_train_batch(const orc_stack* s, const float* batch, uint64_t rows, float beta, float gamma,
                    int square_commitment, float* grad, double* sums) {
    return guard([&] {
        const size_t N = s->stages.size();
        const int64_t D = s->dim();
        for (size_t i = 0; i < 3 + N; ++i) sums[i] = 0.0;
        std::vector<std::vector<float>> g;
        if (grad) g.assign(N, std::vector<float>(size_t(D * D), 0.f));
        for (uint64_t r = 0; r < rows; ++r)
            orc::train_row(*s, batch + r * uint64_t(D), beta, gamma, square_commitment != 0, sums, grad ? g.data() : nullptr);
        if (grad)
            for (size_t i = 0; i < N; ++i) std::memcpy(grad + i * size_t(D * D), g[i].data(), sizeof(float) * size_t(D * D));
    });
}

orc_stack* orc_train(const float* data, uint64_t count, int64_t dim, uint32_t n_stages, const uint32_t* sizes,
                     const orc_train_config* c, int kind, double* epoch_loss, double* stage_mse) {
    orc_stack* out = nullptr;
    int st = guard([&] {
        if (count < 1 || dim < 1) orc::invalid_input("dataset must have count >= 1 and D >= 1");
        size_t batch = size_t(c->batch_size);
        if (count < 10 * batch) batch = std::min<size_t>(batch, 1024);
        std::mt19937_64 rng(c->seed);
        std::vector<size_t> order(count);
        std::iota(order.begin(), order.end(), size_t{0});
        std::shuffle(order.begin(), order.end(), rng);
        size_t n_hold = 0;
        if (count >= 2) {
            n_hold = std::max<size_t>(1, size_t(std::llround(double(count) * c->holdout_fraction)));
            n_hold = std::min<size_t>(n_hold, count - 1);
        }
        std::vector<size_t> hold(order.end() - ptrdiff_t(n_hold), order.end());
        std::vector<size_t> train_rows(order.begin(), order.end() - ptrdiff_t(n_hold));
        if (hold.empty()) hold = train_rows;
        // init_stack (trainer.cpp:125-148): its own generator on the same seed
        auto s = std::make_unique<orc_stack>();
        s->kind = kind;
        {
            std::mt19937_64 irng(c->seed);
            std::normal_distribution<float> gauss(0.0f, 1.0f);
            for (uint32_t i = 0; i < n_stages; ++i) {
                orc::Codebook cb;
                cb.S = sizes[i];
                cb.D = dim;
                cb.entries.resize(size_t(cb.S * dim));
                for (auto& v : cb.entries) v = c->init_scale * gauss(irng);
                cb.projection.assign(size_t(dim * dim), 0.f);
                for (int64_t k = 0; k < dim; ++k) cb.projection[size_t(k * dim + k)] = 1.f;
                cb.refresh();
                s->stages.push_back(std::move(cb));
            }
        }
        const size_t N = n_stages;
        std::vector<float> buf, grad(N * size_t(dim * dim));
        std::vector<double> sums(3 + N);
        for (uint64_t e = 0; e < c->epochs; ++e) {
            std::shuffle(train_rows.begin(), train_rows.end(), rng);
            double eloss = 0.0;
            size_t seen = 0;
            for (size_t b0 = 0; b0 < train_rows.size(); b0 += batch) {
                const size_t len = std::min(batch, train_rows.size() - b0);
                buf.resize(len * size_t(dim));
                for (size_t i = 0; i < len; ++i)
                    std::memcpy(&buf[i * size_t(dim)], data + train_rows[b0 + i] * uint64_t(dim), sizeof(float) * size_t(dim));
                int r = orc_train_batch(s.get(), buf.data(), len, c->beta, c->gamma, c->square_commitment, grad.data(),
                                        sums.data());
                if (r != ORC_OK) orc::invalid_input(g_err);
                const double recon = sums[0] / double(len), pull = sums[1] / double(len), com = sums[2] / double(len);
                const double total = recon + c->beta * pull + c->gamma * com;
                if (!std::isfinite(total)) orc::invalid_input("training loss became non-finite");
                const float step = c->learning_rate / float(len);
                for (size_t i = 0; i < N; ++i) {
                    auto& p = s->stages[i].projection;
                    for (size_t k = 0; k < p.size(); ++k) p[k] = p[k] - step * grad[i * size_t(dim * dim) + k];
                    s->stages[i].refresh();
                }
                eloss += total * double(len);
                seen += len;
            }
            if (epoch_loss) epoch_loss[e] = eloss / double(seen);
        }
        if (stage_mse) {
            std::vector<double> acc(3 + N, 0.0);
            for (size_t rr : hold) orc::train_row(*s, data + rr * uint64_t(dim), 0.f, 0.f, false, acc.data(), nullptr);
            for (size_t i = 0; i < N; ++i) stage_mse[i] = acc[3 + i] / double(hold.size());
        }
        out = s.release();
    });
    return st == ORC_OK ? out : nullptr;
}
}  // extern "C"
