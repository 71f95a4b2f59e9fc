// trainer.cu -- one mini-batch of the codebook trainer on the GPU (f4): forward through the
// quantizer, loss terms, and the straight-through gradients of the stage projections.
// Reference: proj/core/src/trainer.cpp:22-86 (forward_pass, accumulate_loss), 166-248 (train).
//
// The forward pass is the library's exact quantizer (encode_exact.cu, the reference's nearest_scored
// order) followed by the per-stage residual chain r_{i+1} = r_i - effective_i[z_i] (fp32, the
// quantizer's own update order).  Gradients follow trainer.cpp:53-67 operation for operation in fp32
// without contraction:
//   ge_i   = (-2 r_N - (2 beta) r_{i+1}) - gamma suffix_i,  suffix_{i-1} = suffix_i + step_i,
//   step_i = 2 r_{i+1} (squared commitment) or r_{i+1} / ||r_{i+1}||,
//   grad_proj_i += ge_i (x) entries_i[z_i]   (outer product, rows accumulated in batch order),
// so the gradients -- and a training run -- reproduce the reference bit for bit.  Loss terms are
// accumulated in double per row (the reference's order within a row; rows are summed atomically).
#include <algorithm>
#include <vector>

#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

constexpr int kTrainThreads = 128;

// one block per row (grid-stride): residual chain in shared memory, per-stage squared norms in the
// reference's squaredNorm order, loss partials, ge_i rows and codes for the gradient GEMM
__global__ void __launch_bounds__(kTrainThreads) train_rows_kernel(
    const StageInfo* __restrict__ stages, uint32_t n, uint32_t D, const float* __restrict__ eff,
    const float* __restrict__ xs, const uint16_t* __restrict__ codes, uint64_t rows, float beta, float gamma,
    int square_commitment, float* __restrict__ G, double* __restrict__ sums) {
    extern __shared__ float tsm[];
    float* res = tsm;                          // [n + 1][D]
    float* suffix = res + uint64_t(n + 1) * D; // [D]
    float* sqf = suffix + D;                   // [n] : ||r_{i+1}||^2 (fp32, reference order)
    double* part = reinterpret_cast<double*>(tsm + ((uint64_t(n + 2) * D + n + 1) & ~uint64_t(1)));  // [3 + n]
    const uint32_t tid = threadIdx.x;
    for (uint32_t i = tid; i < 3 + n; i += blockDim.x) part[i] = 0.0;
    for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        __syncthreads();
        for (uint32_t d = tid; d < D; d += blockDim.x) res[d] = xs[r * D + d];
        for (uint32_t i = 0; i < n; ++i) {
            const float* e = eff + (stages[i].eff_off + uint64_t(codes[r * n + i]) * D);
            for (uint32_t d = tid; d < D; d += blockDim.x)
                res[uint64_t(i + 1) * D + d] = __fsub_rn(res[uint64_t(i) * D + d], e[d]);
        }
        __syncthreads();
        for (uint32_t i = tid; i < n; i += blockDim.x) {
            const float* v = res + uint64_t(i + 1) * D;
            sqf[i] = redux_dot_exact(v, v, int(D));
        }
        __syncthreads();
        if (tid == 0) {
            part[0] += double(sqf[n - 1]);  // reconstruction: ||r_N||^2
            for (uint32_t i = 0; i < n; ++i) {
                const double sq = double(sqf[i]);
                part[1] += sq;  // codebook pull
                part[2] += square_commitment ? sq : sqrt(sq);
                part[3 + i] += sq;  // per-stage (holdout_stage_mse)
            }
        }
        if (!G) continue;
        const float* rN = res + uint64_t(n) * D;
        const float b2 = 2.0f * beta;
        for (uint32_t d = tid; d < D; d += blockDim.x) suffix[d] = 0.f;
        for (uint32_t i = n; i-- > 0;) {
            const float* ri = res + uint64_t(i + 1) * D;
            const float norm = __fsqrt_rn(sqf[i]);
            float* g = G + (r * n + i) * D;
            for (uint32_t d = tid; d < D; d += blockDim.x) {
                const float ge = __fsub_rn(__fsub_rn(__fmul_rn(-2.0f, rN[d]), __fmul_rn(b2, ri[d])), __fmul_rn(gamma, suffix[d]));
                g[d] = ge;
                const float step = square_commitment ? __fmul_rn(2.0f, ri[d]) : (norm > 0.f ? __fdiv_rn(ri[d], norm) : 0.f);
                suffix[d] = __fadd_rn(suffix[d], step);
            }
        }
    }
    __syncthreads();
    for (uint32_t i = tid; i < 3 + n; i += blockDim.x) atomicAdd(sums + i, part[i]);
}

// grad_proj_i[a][b] = sum over rows (in batch order) of G[row][i][a] * entries_i[z_i(row)][b]:
// one output per thread, rows accumulated sequentially with unfused multiply-add (the reference's
// row-by-row outer-product accumulation); rows staged through shared memory in tiles of 32
constexpr int kGT = 16;  // output tile kGT x kGT, 256 threads
__global__ void __launch_bounds__(kGT * kGT) train_grad_kernel(const StageInfo* __restrict__ stages, uint32_t n,
                                                               uint32_t D, const float* __restrict__ raw,
                                                               const float* __restrict__ G,
                                                               const uint16_t* __restrict__ codes, uint64_t rows,
                                                               float* __restrict__ grad) {
    __shared__ float gs[32][kGT + 1], es[32][kGT + 1];
    const uint32_t i = blockIdx.z, a0 = blockIdx.y * kGT, b0 = blockIdx.x * kGT;
    const uint32_t ta = threadIdx.y, tb = threadIdx.x, t = ta * kGT + tb;
    const uint64_t row0 = stages[i].eff_off / D;
    float acc = 0.f;
    for (uint64_t r0 = 0; r0 < rows; r0 += 32) {
        __syncthreads();
        for (uint32_t k = t; k < 32 * kGT; k += kGT * kGT) {
            const uint32_t rr = k / kGT, c = k % kGT;
            const uint64_t r = r0 + rr;
            const bool ok = r < rows;
            gs[rr][c] = (ok && a0 + c < D) ? G[(r * n + i) * D + a0 + c] : 0.f;
            es[rr][c] = (ok && b0 + c < D) ? raw[(row0 + codes[r * n + i]) * D + b0 + c] : 0.f;
        }
        __syncthreads();
        const uint32_t nr = uint32_t(rows - r0 < 32 ? rows - r0 : 32);
        for (uint32_t rr = 0; rr < nr; ++rr) acc = __fadd_rn(acc, __fmul_rn(es[rr][tb], gs[rr][ta]));
    }
    if (a0 + ta < D && b0 + tb < D) grad[(uint64_t(i) * D + a0 + ta) * D + b0 + tb] = acc;
}

}  // namespace

void train_batch(const vqkv_stack_s& st, const float* batch, uint64_t rows, float beta, float gamma,
                 bool square_commitment, float* grad_proj, double* sums_host, cudaStream_t s) {
    const uint32_t n = st.n, D = st.dim;
    const size_t smem = sizeof(float) * ((uint64_t(n + 2) * D + n + 1) & ~uint64_t(1)) + sizeof(double) * (3 + n);
    if (smem > 200 * 1024) fail(VQKV_UNSUPPORTED, "trainer: (stages + 1) x dim too large for one block's residual chain");
    uint16_t* codes = nullptr;
    float *norms = nullptr, *G = nullptr;
    double* sums = nullptr;
    VQKV_CUDA(cudaMallocAsync(&codes, sizeof(uint16_t) * rows * n, s));
    VQKV_CUDA(cudaMallocAsync(&norms, sizeof(float) * rows, s));
    VQKV_CUDA(cudaMallocAsync(&sums, sizeof(double) * (3 + n), s));
    VQKV_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * (3 + n), s));
    if (grad_proj) VQKV_CUDA(cudaMallocAsync(&G, sizeof(float) * rows * n * D, s));
    // forward: the reference's quantize (exact search order) -> codes
    launch_encode_exact(st, batch, rows, 4096, codes, norms, nullptr, s);  // codebook.hpp:25 search_block
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st.device);
    VQKV_CUDA(cudaFuncSetAttribute(train_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const unsigned grid = unsigned(std::min<uint64_t>(rows, uint64_t(sms) * 8));
    train_rows_kernel<<<grid, kTrainThreads, smem, s>>>(st.d_stages, n, D, st.d_eff, batch, codes, rows, beta, gamma,
                                                        square_commitment ? 1 : 0, G, sums);
    launch_check("train_rows_kernel");
    if (grad_proj) {
        dim3 g((D + kGT - 1) / kGT, (D + kGT - 1) / kGT, n);
        train_grad_kernel<<<g, dim3(kGT, kGT), 0, s>>>(st.d_stages, n, D, st.d_raw, G, codes, rows, grad_proj);
        launch_check("train_grad_kernel");
    }
    VQKV_CUDA(cudaMemcpyAsync(sums_host, sums, sizeof(double) * (3 + n), cudaMemcpyDeviceToHost, s));
    VQKV_CUDA(cudaFreeAsync(codes, s));
    VQKV_CUDA(cudaFreeAsync(norms, s));
    VQKV_CUDA(cudaFreeAsync(sums, s));
    if (G) VQKV_CUDA(cudaFreeAsync(G, s));
    VQKV_CUDA(cudaStreamSynchronize(s));
}

}  // namespace vqkv_dev
