// stack.cu -- device-side codebook stack construction (replaces load_stack's
// Codebook::refresh, proj/core/src/codebook.cpp:30-39).
//
// effective[i][k] = dot(projection[k], entries[i]) in the reference's row-major
// GEMV order (4 lane accumulators, mul-then-add, predux (c0+c2)+(c1+c3)), and
// effective_sqnorm[i] = squaredNorm() in Eigen's vectorised-redux order.  The
// same fp32 bits are then used by every kernel; an fp16 copy (rows padded to
// a multiple of 128, pad rows' sqnorm = +inf) feeds the tensor-core encoder.
#include <algorithm>
#include <cmath>

#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

__global__ void refresh_kernel(const float* __restrict__ entries, const float* __restrict__ proj,
                               const StageInfo* __restrict__ stages, uint32_t n_stages, uint32_t D,
                               uint64_t total_rows, float* __restrict__ eff) {
    uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= total_rows * D) return;
    uint64_t row = idx / D;
    uint32_t k = uint32_t(idx % D);
    // find the stage owning this row (n_stages is small; linear scan)
    uint32_t s = 0;
    while (s + 1 < n_stages && stages[s + 1].eff_off / D <= row) ++s;
    const float* e = entries + row * D;
    const float* p = proj + uint64_t(s) * D * D + uint64_t(k) * D;
    eff[idx] = (D == 1) ? redux_dot_exact(p, e, int(D)) : gemv_dot_exact(p, e, int(D));
}

__global__ void sqnorm_kernel(const float* __restrict__ eff, uint32_t D, uint64_t total_rows, float* __restrict__ sqn) {
    uint64_t row = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= total_rows) return;
    const float* e = eff + row * D;
    sqn[row] = redux_dot_exact(e, e, int(D));
}

// fp16 operand copy [pad_S][D] per stage and padded sqnorm (+inf on padding).
__global__ void half_copy_kernel(const float* __restrict__ eff, const float* __restrict__ sqn,
                                 const StageInfo* __restrict__ stages, uint32_t stage, uint32_t D,
                                 __half* __restrict__ eff16, __half* __restrict__ eff16lo, float* __restrict__ sqn_pad) {
    const StageInfo st = stages[stage];
    uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(st.pad_size) * D) return;
    uint32_t j = uint32_t(idx / D);
    uint32_t k = uint32_t(idx % D);
    float v = (j < st.size) ? eff[(st.eff_off) + idx] : 0.f;
    // Pre-swizzled UMMA operand layout (D == 128): 128-entry chunks of 36 KB =
    //  * two K-blocks of [128 rows x 128 B] with the 128B swizzle applied
    //    (16 B granule g of row r stored at g ^ (r % 8)), then
    //  * one 16-wide K-block (no swizzle, 8x16 B core matrices, LBO 128 B,
    //    SBO 256 B) holding ||e_j||^2 split into fp16 hi + lo in columns 0, 1.
    // A single bulk copy of a chunk into 1024 B-aligned smem yields canonical
    // K-major UMMA tiles; the extra K-block lets the MMA add -2^(s-1)||e||^2.
    const uint32_t c = j >> 7, rj = j & 127, kb = k >> 6, kk = k & 63;
    __half* chunk = eff16 + st.eff16_off + uint64_t(c) * 18432;
    const uint64_t off = kb * 8192 + rj * 64 + (((kk >> 3) ^ (rj & 7)) << 3) + (kk & 7);
    const __half hi = __float2half_rn(v);
    chunk[off] = hi;
    // residual fp16(v - hi) in the same layout: hi + lo carries 22 bits of v (the decode-attention
    // LUT GEMM's split-precision operand, attend_lut.cu lut_tc_kernel); v - hi is exact in fp32
    eff16lo[st.eff16_off + uint64_t(c) * 18432 + off] = __float2half_rn(v - __half2float(hi));
    if (k < 16) {
        // ext block: element (rj, k) at (rj/8)*256 B + (k/8)*128 B + (rj%8)*16 B + (k%8)*2 B
        const uint64_t eoff = 16384 + (rj >> 3) * 128 + (k >> 3) * 64 + (rj & 7) * 8 + (k & 7);
        __half hv = __float2half_rn(0.f);
        if (j >= st.size) {
            hv = (k == 0) ? __float2half_rn(INFINITY) : __float2half_rn(0.f);
        } else if (k < 2) {
            const float q = sqn[st.eff_off / D + j];
            const __half hi = __float2half_rn(q);
            hv = (k == 0) ? hi : __float2half_rn(q - __half2float(hi));
        }
        chunk[eoff] = hv;
    }
    if (k == 0) sqn_pad[st.pad_off + j] = (j < st.size) ? sqn[st.eff_off / D + j] : INFINITY;
}

}  // namespace

void stack_build_device(vqkv_stack_s& st, const float* entries_host, const float* proj_host) {
    const uint32_t D = st.dim;
    const uint64_t T = st.total_rows;
    float *d_entries = nullptr, *d_proj = nullptr;
    VQKV_CUDA(cudaMalloc(&d_entries, sizeof(float) * T * D));
    VQKV_CUDA(cudaMalloc(&d_proj, sizeof(float) * uint64_t(st.n) * D * D));
    VQKV_CUDA(cudaMemcpy(d_entries, entries_host, sizeof(float) * T * D, cudaMemcpyHostToDevice));
    if (proj_host) {
        VQKV_CUDA(cudaMemcpy(d_proj, proj_host, sizeof(float) * uint64_t(st.n) * D * D, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> eye(uint64_t(st.n) * D * D, 0.f);
        for (uint32_t s = 0; s < st.n; ++s)
            for (uint32_t i = 0; i < D; ++i) eye[uint64_t(s) * D * D + uint64_t(i) * D + i] = 1.f;
        VQKV_CUDA(cudaMemcpy(d_proj, eye.data(), sizeof(float) * eye.size(), cudaMemcpyHostToDevice));
    }
    VQKV_CUDA(cudaMalloc(&st.d_eff, sizeof(float) * T * D));
    VQKV_CUDA(cudaMalloc(&st.d_sqn, sizeof(float) * T));
    {
        uint64_t n = T * D;
        refresh_kernel<<<unsigned((n + 255) / 256), 256>>>(d_entries, d_proj, st.d_stages, st.n, D, T, st.d_eff);
        launch_check("refresh_kernel");
        sqnorm_kernel<<<unsigned((T + 255) / 256), 256>>>(st.d_eff, D, T, st.d_sqn);
        launch_check("sqnorm_kernel");
    }
    if (D == 128) {
        VQKV_CUDA(cudaMalloc(&st.d_eff16, sizeof(__half) * st.total_pad_rows * (D + 16)));
        VQKV_CUDA(cudaMalloc(&st.d_eff16lo, sizeof(__half) * st.total_pad_rows * (D + 16)));
        VQKV_CUDA(cudaMalloc(&st.d_sqn_pad, sizeof(float) * st.total_pad_rows));
        for (uint32_t s = 0; s < st.n; ++s) {
            uint64_t n = uint64_t(st.stages[s].pad_size) * D;
            half_copy_kernel<<<unsigned((n + 255) / 256), 256>>>(st.d_eff, st.d_sqn, st.d_stages, s, D, st.d_eff16,
                                                                 st.d_eff16lo, st.d_sqn_pad);
            launch_check("half_copy_kernel");
        }
    }
    VQKV_CUDA(cudaDeviceSynchronize());
    // per-stage max norms (host side, from the device's own fp32 sqnorms)
    std::vector<float> sqn(T), effh(T * D);
    VQKV_CUDA(cudaMemcpy(sqn.data(), st.d_sqn, sizeof(float) * T, cudaMemcpyDeviceToHost));
    VQKV_CUDA(cudaMemcpy(effh.data(), st.d_eff, sizeof(float) * T * D, cudaMemcpyDeviceToHost));
    for (uint32_t s = 0; s < st.n; ++s) {
        float m = 0.f;
        const uint64_t off = st.stages[s].eff_off / D;
        for (uint32_t j = 0; j < st.stages[s].size; ++j) {
            float v = sqn[off + j];
            if (!(v <= m)) m = v;  // NaN propagates (non-finite codebooks are rejected earlier)
        }
        st.stages[s].max_sqnorm = m;
        float ma = 0.f;
        for (uint64_t k = off * D; k < (off + st.stages[s].size) * D; ++k) ma = std::max(ma, std::fabs(effh[k]));
        st.stages[s].max_abs = ma;
        // rounded up so that ||e_j|| <= max_norm holds for every entry
        st.stages[s].max_norm = std::nextafter(std::sqrt(m), INFINITY);
    }
    VQKV_CUDA(cudaMemcpy(st.d_stages, st.stages.data(), sizeof(StageInfo) * st.n, cudaMemcpyHostToDevice));
    st.d_raw = d_entries;  // kept: the trainer's straight-through gradients use the raw entries (trainer.cpp:62-67)
    cudaFree(d_proj);
}

}  // namespace vqkv_dev
