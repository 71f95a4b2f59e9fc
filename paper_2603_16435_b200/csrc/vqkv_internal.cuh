// vqkv_internal.cuh -- shared definitions of libvqkv_b200.so (not installed).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "vqkv_c.h"

namespace vqkv_dev {

// ---------------------------------------------------------------------------
// Errors: C++ exceptions inside the library, converted to status codes at the
// C-ABI (vqkv_c_api.cu).
struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Err(code, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(VQKV_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define VQKV_CUDA(x) ::vqkv_dev::cuda_check((x), #x)

// Optional event-pair timing of hot kernels (vqkv_profile_enable).
bool prof_enabled();
void prof_record(const char* name, cudaEvent_t start, cudaEvent_t stop);
struct ProfScope {
    const char* name;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(const char* n, cudaStream_t st) : name(n), s(st) {
        if (prof_enabled()) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, s);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, s);
            prof_record(name, a, b);
        }
    }
};

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
inline void launch_check(const char* k) {
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(VQKV_CUDA_ERROR, std::string("launch ") + k + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Per-stage table, mirrored on the device (constant-size POD).
struct StageInfo {
    uint32_t size;     // S_i
    uint32_t bits;     // ceil(log2 S_i)
    uint32_t bit_off;  // offset of this stage's field within a row
    uint32_t pad_size; // S_i rounded up to the tensor-core N chunk (128)
    uint64_t eff_off;  // element offset of stage in eff/sqn (rows of D floats)
    uint64_t eff16_off;// element offset into the fp16 operand copy (chunks of 128 entries x (D + 16))
    uint64_t pad_off;  // row offset of the stage in the padded row space (sqn_pad index)
    float max_norm;    // max_j ||e_j|| (fp32, rounded up)
    float max_sqnorm;  // max_j ||e_j||^2
    float max_abs;     // max_{j,k} |e_jk|
    float pad_;
};

}  // namespace vqkv_dev

struct vqkv_stack_s {
    int device = 0;
    int kind = 0;
    uint32_t n = 0, dim = 0;
    uint64_t row_bits = 0;
    std::vector<vqkv_dev::StageInfo> stages;  // host copy
    vqkv_dev::StageInfo* d_stages = nullptr;  // device copy
    float* d_eff = nullptr;                   // [sum S_i][D] fp32 effective entries
    float* d_raw = nullptr;                   // [sum S_i][D] fp32 raw entries (trainer gradients)
    float* d_sqn = nullptr;                   // [sum S_i]
    __half* d_eff16 = nullptr;                // [sum pad_S_i][D] fp16 operand (D == 128 only)
    __half* d_eff16lo = nullptr;              // fp16(eff - fp16(eff)), same layout (LUT GEMM operand)
    float* d_sqn_pad = nullptr;               // [sum pad_S_i] sqnorm, +inf on padding rows
    uint64_t total_rows = 0, total_pad_rows = 0;
    int* d_error = nullptr;                   // sticky device error flag
    unsigned long long* d_counters = nullptr; // encode diagnostics [4]
    cudaStream_t cp_in = nullptr, cp_out = nullptr;  // host-buffer pipeline copy streams (lazy)
    cudaStream_t cs_alt = nullptr;  // second compute stream: consecutive chunk encodes overlap their tails
    cudaStream_t cs_attn = nullptr;    // decode attention: the raw-row kernel (lowest stream priority)
    cudaStream_t cs_attn_hi = nullptr; // decode attention: the main kernel (highest stream priority)
    // host-buffer calls stage through two persistent device arenas, used alternately: a call waits
    // (host side) for the call two before it, so a host running ahead is held back instead of the
    // stream-ordered pool growing (and mapping memory) inside the timed pipeline
    struct Staging {
        uint8_t* base = nullptr;
        uint64_t bytes = 0;
        cudaEvent_t done = nullptr;
    } staging[2];
    uint32_t staging_next = 0;
    // device scratch of the synchronous *_host entry points (grow-only, freed with the stack;
    // host_mu serialises those calls on this stack)
    uint8_t* host_scratch = nullptr;
    uint64_t host_scratch_bytes = 0;
    std::mutex host_mu;
    std::mutex mu;
};

namespace vqkv_dev {

// ---------------------------------------------------------------------------
// Exact reference arithmetic on the device.  __fmul_rn/__fadd_rn are never
// contracted into FMA, so these reproduce the x86-64 SSE2 results of the
// reference's Eigen 3.4 kernels bit for bit (see oracle/vqkv_oracle.cpp).
__device__ __forceinline__ float gemv_dot_exact(const float* __restrict__ a, const float* __restrict__ b, int n) {
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        c0 = __fadd_rn(c0, __fmul_rn(a[j + 0], b[j + 0]));
        c1 = __fadd_rn(c1, __fmul_rn(a[j + 1], b[j + 1]));
        c2 = __fadd_rn(c2, __fmul_rn(a[j + 2], b[j + 2]));
        c3 = __fadd_rn(c3, __fmul_rn(a[j + 3], b[j + 3]));
    }
    float cc = __fadd_rn(__fadd_rn(c0, c2), __fadd_rn(c1, c3));
    for (; j < n; ++j) cc = __fadd_rn(cc, __fmul_rn(a[j], b[j]));
    return cc;
}

__device__ __forceinline__ float redux_dot_exact(const float* __restrict__ a, const float* __restrict__ b, int n) {
    const int aligned = (n / 4) * 4, aligned2 = (n / 8) * 8;
    float res;
    if (aligned) {
        float r0[4], r1[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) r0[l] = __fmul_rn(a[l], b[l]);
        if (aligned > 4) {
#pragma unroll
            for (int l = 0; l < 4; ++l) r1[l] = __fmul_rn(a[4 + l], b[4 + l]);
            for (int i = 8; i < aligned2; i += 8) {
#pragma unroll
                for (int l = 0; l < 4; ++l) r0[l] = __fadd_rn(r0[l], __fmul_rn(a[i + l], b[i + l]));
#pragma unroll
                for (int l = 0; l < 4; ++l) r1[l] = __fadd_rn(r1[l], __fmul_rn(a[i + 4 + l], b[i + 4 + l]));
            }
#pragma unroll
            for (int l = 0; l < 4; ++l) r0[l] = __fadd_rn(r0[l], r1[l]);
            if (aligned > aligned2) {
#pragma unroll
                for (int l = 0; l < 4; ++l) r0[l] = __fadd_rn(r0[l], __fmul_rn(a[aligned2 + l], b[aligned2 + l]));
            }
        }
        res = __fadd_rn(__fadd_rn(r0[0], r0[2]), __fadd_rn(r0[1], r0[3]));
        for (int i = aligned; i < n; ++i) res = __fadd_rn(res, __fmul_rn(a[i], b[i]));
    } else {
        res = __fmul_rn(a[0], b[0]);
        for (int i = 1; i < n; ++i) res = __fadd_rn(res, __fmul_rn(a[i], b[i]));
    }
    return res;
}

// Score of entry j of a stage under the reference's nearest_scored
// (codebook.cpp:158-176): a search block of length 1 uses the dot() order.
__device__ __forceinline__ float exact_score(const float* __restrict__ e, const float* __restrict__ r, int D,
                                             float sqn, uint32_t j, uint32_t S, uint64_t search_block) {
    uint64_t blk0 = (uint64_t(j) / search_block) * search_block;
    uint64_t len = (uint64_t(S) - blk0 < search_block) ? uint64_t(S) - blk0 : search_block;
    float dot = (len == 1) ? redux_dot_exact(e, r, D) : gemv_dot_exact(e, r, D);
    return __fsub_rn(sqn, __fmul_rn(2.0f, dot));
}

// Reads a `width`-bit field at absolute bit `pos` of an LSB-first stream,
// touching only the bytes the field occupies (bitpack.hpp:29-36).
__device__ __forceinline__ uint32_t read_bits(const uint8_t* __restrict__ p, uint64_t pos, uint32_t width) {
    if (width == 0) return 0;
    uint64_t byte = pos >> 3;
    uint32_t sh = uint32_t(pos & 7);
    uint32_t nbytes = (sh + width + 7) >> 3;
    uint64_t acc = 0;
    for (uint32_t b = 0; b < nbytes; ++b) acc |= uint64_t(__ldg(p + byte + b)) << (8 * b);
    return uint32_t((acc >> sh) & ((width >= 32) ? 0xffffffffull : ((1ull << width) - 1)));
}

inline uint32_t index_bit_width(uint32_t size) {
    uint32_t w = 0;
    while ((uint64_t(1) << w) < size) ++w;
    return w;
}

inline uint64_t payload_bytes(uint64_t row_bits, uint64_t rows) { return (rows * row_bits + 7) / 8; }

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) VQKV_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ---- kernels launched from the C-ABI (defined in the .cu files) -------------
void launch_payload_append(uint8_t* dst, uint64_t dst_stride, uint64_t dst_bits, const uint8_t* src,
                           uint64_t src_stride, uint64_t src_bits, uint32_t n_streams, cudaStream_t s);
void stack_build_device(vqkv_stack_s& st, const float* entries_host, const float* proj_host);
void launch_pack_codes(const uint16_t* codes, uint32_t n_streams, uint64_t rows, uint32_t n_stages,
                       const vqkv_stack_s& st, uint8_t* payload, cudaStream_t s);
void launch_encode_exact(const vqkv_stack_s& st, const float* xs, uint64_t total_rows, uint64_t search_block,
                         uint16_t* codes, float* norms, float* residuals, cudaStream_t s);
void launch_nearest(const vqkv_stack_s& st, uint32_t stage, const float* xs, uint64_t rows, uint64_t search_block,
                    uint32_t* idx, float* dist, cudaStream_t s);
bool encode_tc_supported(const vqkv_stack_s& st);
void launch_encode_tc(const vqkv_stack_s& st, const float* xs, uint32_t n_streams, uint64_t rows_per_stream,
                      uint64_t search_block, uint8_t* payload, float* norms, float* residuals, cudaStream_t s);
void launch_reconstruct(const vqkv_stack_s& st, const uint8_t* payload, uint32_t n_streams, uint64_t rows,
                        uint64_t begin, uint64_t end, float* out, cudaStream_t s,
                        uint64_t stream_stride = 0);
void launch_attend(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a, cudaStream_t s);
int attend_path();
bool attend_lut_supported(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a);
bool gm_supported(const vqkv_stack_s& ks);
uint64_t gm_pair_bytes(const vqkv_stack_s& ks, uint64_t cap);
void launch_keycodes_to_gm(const vqkv_stack_s& ks, const uint8_t* payload, uint64_t payload_stride, uint32_t n_pairs,
                           uint64_t src_row, uint64_t count, uint8_t* gm, uint64_t cap, uint64_t gm_stride,
                           uint64_t dst_row, cudaStream_t s);
void launch_attend_raw(int device, const float* keys, const float* values, uint64_t rows, uint32_t dk, uint32_t dv,
                       const float* q, double scale, float* out, cudaStream_t s);
void launch_keycodes_from_gm(const vqkv_stack_s& ks, const uint8_t* gm, uint64_t cap, uint64_t gm_stride,
                             uint32_t n_pairs, uint64_t count, uint8_t* payload, uint64_t payload_stride,
                             cudaStream_t s);
void launch_lse_combine(const float* o, const float* lse, uint32_t parts, uint64_t rows, uint32_t dv, float* out,
                        float* out_lse, cudaStream_t s);
void train_batch(const vqkv_stack_s& st, const float* batch, uint64_t rows, float beta, float gamma,
                 bool square_commitment, float* grad_proj, double* sums_host, cudaStream_t s);
void nccl_comm_init_all(int ndev, const int* devs, void** comms);
void nccl_comm_destroy(void* comm);
void lse_allgather_combine(void* comm, const float* part_o, const float* part_lse, uint64_t rows, uint32_t dv,
                           float* gather_o, float* gather_lse, float* out, float* out_lse, cudaStream_t s);

}  // namespace vqkv_dev
