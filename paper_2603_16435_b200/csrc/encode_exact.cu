// encode_exact.cu -- exact SIMT residual encoder + CodeMatrix packer.
//
// This path reproduces quantize_batch (proj/core/src/codebook.cpp:158-237)
// operation for operation on CUDA cores: every candidate is scored with the
// reference's fp32 GEMV order (exact_score), argmin keeps the first minimum
// (strict <, lowest index on ties, NaN never wins, index 0 if nothing beats
// +inf), and the residual update / final norm use the reference's fp32 ops.
// It serves any D (the tensor-core encoder covers D == 128) and rows whose
// input is non-finite.  One warp per row; lanes split the codebook entries.
#include <algorithm>
#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

constexpr int kExactWarps = 4;

__global__ void __launch_bounds__(kExactWarps * 32)
encode_exact_kernel(const StageInfo* __restrict__ stages, uint32_t n_stages, uint32_t D, const float* __restrict__ eff,
                    const float* __restrict__ sqn, const float* __restrict__ xs, uint64_t total_rows,
                    uint64_t search_block, uint16_t* __restrict__ codes, float* __restrict__ norms,
                    float* __restrict__ residuals, const uint32_t* __restrict__ row_list,
                    const uint32_t* __restrict__ n_list_dev) {
    extern __shared__ float smem[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    float* r = smem + uint64_t(wib) * D;
    const uint64_t nwork = row_list ? uint64_t(*n_list_dev) : total_rows;
    for (uint64_t w = uint64_t(blockIdx.x) * kExactWarps + wib; w < nwork; w += uint64_t(gridDim.x) * kExactWarps) {
        const uint64_t row = row_list ? row_list[w] : w;
        const float* x = xs + row * D;
        for (uint32_t k = lane; k < D; k += 32) r[k] = x[k];
        __syncwarp();
        for (uint32_t s = 0; s < n_stages; ++s) {
            const StageInfo si = stages[s];
            const float* e0 = eff + si.eff_off;
            const float* q0 = sqn + si.eff_off / D;
            float best = INFINITY;
            uint32_t bidx = 0xffffffffu;
            for (uint32_t j = lane; j < si.size; j += 32) {
                float sc = exact_score(e0 + uint64_t(j) * D, r, int(D), q0[j], j, si.size, search_block);
                if (sc < best) {
                    best = sc;
                    bidx = j;
                }
            }
            // warp argmin: smaller score wins, equal scores -> lower index
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                float ob = __shfl_xor_sync(0xffffffffu, best, off);
                uint32_t oi = __shfl_xor_sync(0xffffffffu, bidx, off);
                if (oi != 0xffffffffu && (bidx == 0xffffffffu || ob < best || (ob == best && oi < bidx))) {
                    best = ob;
                    bidx = oi;
                }
            }
            const uint32_t z = (bidx == 0xffffffffu) ? 0u : bidx;
            if (lane == 0) codes[row * n_stages + s] = uint16_t(z);
            const float* e = e0 + uint64_t(z) * D;
            __syncwarp();
            for (uint32_t k = lane; k < D; k += 32) r[k] = __fsub_rn(r[k], e[k]);
            __syncwarp();
        }
        if (lane == 0) norms[row] = __fsqrt_rn(redux_dot_exact(r, r, int(D)));
        if (residuals)
            for (uint32_t k = lane; k < D; k += 32) residuals[row * D + k] = r[k];
        __syncwarp();
    }
}

// One thread per payload byte: OR of the code fields overlapping the byte
// (bitpack.hpp:14-27 semantics: LSB-first, rows back to back).
__global__ void pack_kernel(const uint16_t* __restrict__ codes, const StageInfo* __restrict__ stages,
                            uint32_t n_stages, uint64_t row_bits, uint32_t n_streams, uint64_t rows,
                            uint64_t stream_bytes, uint8_t* __restrict__ payload) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(n_streams) * stream_bytes) return;
    const uint64_t stream = idx / stream_bytes;
    const uint64_t b = idx % stream_bytes;
    const uint64_t bit0 = b * 8, bit1 = bit0 + 8, limit = rows * row_bits;
    uint32_t byte = 0;
    const uint64_t stop = (bit1 < limit) ? bit1 : limit;
    uint64_t p = bit0;
    while (p < stop) {
        const uint64_t row = p / row_bits;
        const uint64_t q = p - row * row_bits;
        // last stage whose field starts at or before q; it contains q (fields
        // are contiguous, so zero-width stages are skipped automatically)
        uint32_t lo = 0, hi = n_stages;  // invariant: stages[lo].bit_off <= q < stages[hi].bit_off
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (stages[mid].bit_off <= q) lo = mid; else hi = mid;
        }
        const StageInfo si = stages[lo];
        const uint64_t fstart = row * row_bits + si.bit_off;
        const uint64_t fend = fstart + si.bits;
        const uint64_t e = (fend < stop) ? fend : stop;
        const uint32_t code = codes[(stream * rows + row) * n_stages + lo];
        for (uint64_t pp = p; pp < e; ++pp) byte |= ((code >> (pp - fstart)) & 1u) << (pp - bit0);
        p = e;
    }
    payload[idx] = uint8_t(byte);
}

// Fast path for byte-aligned rows (row_bits % 8 == 0, e.g. K 560 bits, V 144):
// a CTA packs 128 rows of one stream.  u16 codes are staged in smem with
// coalesced loads, each thread packs its row LSB-first into a smem byte tile,
// and the tile (contiguous in the payload) is written with coalesced stores.
constexpr int kPackRows = 128;
constexpr int kPackMaxStages = 128;
__global__ void __launch_bounds__(kPackRows) pack_rows_kernel(const uint16_t* __restrict__ codes,
                                                               const StageInfo* __restrict__ stages, uint32_t n_stages,
                                                               uint32_t row_bytes, uint64_t rows,
                                                               uint64_t stream_bytes, uint8_t* __restrict__ payload) {
    extern __shared__ uint8_t psm[];
    uint8_t* sbits = psm;                                                  // [kPackMaxStages]
    uint16_t* sc = reinterpret_cast<uint16_t*>(psm + kPackMaxStages);      // [kPackRows][n_stages]
    uint8_t* so = psm + kPackMaxStages + kPackRows * n_stages * 2;          // [kPackRows][row_bytes]
    const uint64_t stream = blockIdx.y;
    const uint64_t r0 = uint64_t(blockIdx.x) * kPackRows;
    const uint32_t nr = uint32_t((rows - r0 < kPackRows) ? (rows - r0) : kPackRows);
    for (uint32_t i = threadIdx.x; i < n_stages; i += blockDim.x) sbits[i] = uint8_t(stages[i].bits);
    const uint16_t* src = codes + (stream * rows + r0) * n_stages;
    for (uint32_t i = threadIdx.x; i < nr * n_stages; i += blockDim.x) sc[i] = src[i];
    __syncthreads();
    if (threadIdx.x < nr) {
        const uint16_t* c = sc + threadIdx.x * n_stages;
        uint8_t* o = so + threadIdx.x * row_bytes;
        uint64_t acc = 0;
        uint32_t nb = 0, ob = 0;
        for (uint32_t st = 0; st < n_stages; ++st) {
            const uint32_t b = sbits[st];
            acc |= uint64_t(c[st] & ((1u << b) - 1u)) << nb;
            nb += b;
            while (nb >= 8) {
                o[ob++] = uint8_t(acc);
                acc >>= 8;
                nb -= 8;
            }
        }
    }
    __syncthreads();
    uint8_t* dst = payload + stream * stream_bytes + r0 * row_bytes;
    for (uint32_t i = threadIdx.x; i < nr * row_bytes; i += blockDim.x) dst[i] = so[i];
}

// CodeMatrix::append of a whole packed block (codebook.cpp:96-120 semantics for
// many rows): for every stream, the src_bits of src land at bit dst_bits of
// dst; one thread per destination byte, low bits of the first byte kept.
__global__ void payload_append_kernel(uint8_t* __restrict__ dst, uint64_t dst_stride, uint64_t dst_bits,
                                      const uint8_t* __restrict__ src, uint64_t src_stride, uint64_t src_bits,
                                      uint32_t n_streams) {
    const uint64_t b0 = dst_bits >> 3, nb = ((dst_bits + src_bits + 7) >> 3) - b0;
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= nb * n_streams) return;
    const uint64_t stream = idx / nb, k = idx % nb;
    const uint8_t* s = src + stream * src_stride;
    uint8_t* d = dst + stream * dst_stride + b0;
    const uint64_t src_bytes = (src_bits + 7) >> 3;
    const uint32_t sh = uint32_t(dst_bits & 7);
    uint32_t v = (k < src_bytes) ? (uint32_t(s[k]) << sh) : 0u;
    if (k > 0 && sh) v |= uint32_t(s[k - 1]) >> (8 - sh);
    if (k == 0) v |= d[0] & ((1u << sh) - 1u);
    d[k] = uint8_t(v);
}

// nearest_entry (codebook.cpp:180-192) for many vectors against one stage.
__global__ void __launch_bounds__(kExactWarps * 32)
nearest_kernel(StageInfo si, uint32_t D, const float* __restrict__ eff, const float* __restrict__ sqn,
               const float* __restrict__ xs, uint64_t rows, uint64_t search_block, uint32_t* __restrict__ idx_out,
               float* __restrict__ dist_out) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t row = uint64_t(blockIdx.x) * kExactWarps + (threadIdx.x >> 5); row < rows;
         row += uint64_t(gridDim.x) * kExactWarps) {
        const float* x = xs + row * D;
        const float* e0 = eff + si.eff_off;
        const float* q0 = sqn + si.eff_off / D;
        float best = INFINITY;
        uint32_t bidx = 0xffffffffu;
        for (uint32_t j = lane; j < si.size; j += 32) {
            float sc = exact_score(e0 + uint64_t(j) * D, x, int(D), q0[j], j, si.size, search_block);
            if (sc < best) {
                best = sc;
                bidx = j;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            float ob = __shfl_xor_sync(0xffffffffu, best, off);
            uint32_t oi = __shfl_xor_sync(0xffffffffu, bidx, off);
            if (oi != 0xffffffffu && (bidx == 0xffffffffu || ob < best || (ob == best && oi < bidx))) {
                best = ob;
                bidx = oi;
            }
        }
        if (lane == 0) {
            idx_out[row] = (bidx == 0xffffffffu) ? 0u : bidx;
            const float xsq = (D ? redux_dot_exact(x, x, int(D)) : 0.f);
            dist_out[row] = __fsqrt_rn(fmaxf(0.f, __fadd_rn(best, xsq)));
        }
    }
}

}  // namespace

void launch_nearest(const vqkv_stack_s& st, uint32_t stage, const float* xs, uint64_t rows, uint64_t search_block,
                    uint32_t* idx, float* dist, cudaStream_t s) {
    if (rows == 0) return;
    uint64_t blocks = std::min<uint64_t>((rows + kExactWarps - 1) / kExactWarps, 148 * 8);
    nearest_kernel<<<unsigned(blocks), kExactWarps * 32, 0, s>>>(st.stages[stage], st.dim, st.d_eff, st.d_sqn, xs, rows,
                                                                  search_block, idx, dist);
    launch_check("nearest_kernel");
}

void launch_encode_exact(const vqkv_stack_s& st, const float* xs, uint64_t total_rows, uint64_t search_block,
                         uint16_t* codes, float* norms, float* residuals, cudaStream_t s) {
    if (total_rows == 0) return;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st.device);
    uint64_t blocks = std::min<uint64_t>((total_rows + kExactWarps - 1) / kExactWarps, uint64_t(sms) * 8);
    size_t smem = sizeof(float) * st.dim * kExactWarps;
    if (smem > 48 * 1024)
        VQKV_CUDA(cudaFuncSetAttribute(encode_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    ProfScope ps("encode_exact", s);
    encode_exact_kernel<<<unsigned(blocks), kExactWarps * 32, smem, s>>>(
        st.d_stages, st.n, st.dim, st.d_eff, st.d_sqn, xs, total_rows, search_block, codes, norms, residuals, nullptr, nullptr);
    launch_check("encode_exact_kernel");
}

// Exact encoder restricted to a device list of row indices whose length lives
// in device memory (rows the tensor-core encoder hands back: non-finite input).
void launch_encode_exact_rows(const vqkv_stack_s& st, const float* xs, const uint32_t* rows_dev,
                              const uint32_t* n_rows_dev, uint64_t max_rows, uint64_t search_block, uint16_t* codes,
                              float* norms, float* residuals, cudaStream_t s) {
    if (max_rows == 0) return;
    size_t smem = sizeof(float) * st.dim * kExactWarps;
    encode_exact_kernel<<<148, kExactWarps * 32, smem, s>>>(st.d_stages, st.n, st.dim, st.d_eff, st.d_sqn, xs, 0,
                                                             search_block, codes, norms, residuals, rows_dev, n_rows_dev);
    launch_check("encode_exact_kernel(rows)");
}

namespace {
// CodeMatrix rows of a device list of global row indices (stream * rows + row), rows a whole number of
// 16-bit words: one thread per listed row writes its own bytes.
__global__ void pack_listed_rows_kernel(const uint16_t* __restrict__ codes, const uint32_t* __restrict__ list,
                                        const uint32_t* __restrict__ n_list, const StageInfo* __restrict__ stages,
                                        uint32_t n_stages, uint64_t rows, uint64_t stride, uint32_t row_bytes,
                                        uint8_t* __restrict__ payload) {
    const uint32_t n = *n_list;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint64_t g = list[k];
        uint16_t* dst = reinterpret_cast<uint16_t*>(payload + (g / rows) * stride + (g % rows) * row_bytes);
        uint32_t acc = 0, nb = 0;
        for (uint32_t s = 0; s < n_stages; ++s) {
            acc |= uint32_t(codes[g * n_stages + s]) << nb;
            nb += stages[s].bits;
            if (nb >= 16) {
                *dst++ = uint16_t(acc);
                acc >>= 16;
                nb -= 16;
            }
        }
    }
}
}  // namespace

void launch_pack_listed_rows(const uint16_t* codes, const uint32_t* rows_dev, const uint32_t* n_rows_dev,
                             uint64_t max_rows, uint64_t rows, uint32_t n_stages, const vqkv_stack_s& st,
                             uint8_t* payload, cudaStream_t s) {
    if (max_rows == 0) return;
    pack_listed_rows_kernel<<<16, 256, 0, s>>>(codes, rows_dev, n_rows_dev, st.d_stages, n_stages, rows,
                                               payload_bytes(st.row_bits, rows), uint32_t(st.row_bits / 8), payload);
    launch_check("pack_listed_rows_kernel");
}

void launch_pack_codes(const uint16_t* codes, uint32_t n_streams, uint64_t rows, uint32_t n_stages,
                       const vqkv_stack_s& st, uint8_t* payload, cudaStream_t s) {
    const uint64_t sb = payload_bytes(st.row_bits, rows);
    const uint64_t n = sb * n_streams;
    if (n == 0) return;
    ProfScope ps("pack", s);
    uint32_t max_bits = 0;
    for (const auto& si : st.stages) max_bits = std::max(max_bits, si.bits);
    const size_t fsm = kPackMaxStages + size_t(kPackRows) * n_stages * 2 + size_t(kPackRows) * (st.row_bits / 8);
    if (st.row_bits % 8 == 0 && st.row_bits > 0 && n_stages <= uint32_t(kPackMaxStages) && max_bits <= 16 &&
        fsm <= 48 * 1024 && rows > 0) {
        dim3 grid(unsigned((rows + kPackRows - 1) / kPackRows), n_streams);
        pack_rows_kernel<<<grid, kPackRows, fsm, s>>>(codes, st.d_stages, n_stages, uint32_t(st.row_bits / 8), rows, sb,
                                                      payload);
        launch_check("pack_rows_kernel");
        return;
    }
    pack_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(codes, st.d_stages, n_stages, st.row_bits, n_streams, rows,
                                                          sb, payload);
    launch_check("pack_kernel");
}

void launch_payload_append(uint8_t* dst, uint64_t dst_stride, uint64_t dst_bits, const uint8_t* src,
                           uint64_t src_stride, uint64_t src_bits, uint32_t n_streams, cudaStream_t s) {
    if (src_bits == 0 || n_streams == 0) return;
    const uint64_t nb = ((dst_bits + src_bits + 7) >> 3) - (dst_bits >> 3);
    const uint64_t n = nb * n_streams;
    payload_append_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(dst, dst_stride, dst_bits, src, src_stride,
                                                                    src_bits, n_streams);
    launch_check("payload_append_kernel");
}

}  // namespace vqkv_dev
