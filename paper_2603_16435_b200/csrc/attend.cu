// attend.cu -- K3: decode-step attention over the compressed cache
// (replaces attend over CacheState, proj/core/src/attention.cpp:26-69 with
// view_block's segment stitching, proj/core/src/kv_cache.cpp:143-189).
//
// Split-KV: CTA (pair, split) walks a contiguous range of the logical token
// sequence init | compressed | local, keeps an online softmax per query head
// (running max m, normaliser l, unnormalised accumulator) and writes a
// partial (acc, m, l); a combine kernel merges the splits and emits the
// normalised output and the natural-log LSE of scale*logits (the quantity the
// cross-GPU sequence-split merge needs).
//
// This file holds the generic path (any Dk/Dv, any stack shape): keys and
// values are reconstructed row by row in shared memory, exactly as
// view_block does, and never written to HBM.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

constexpr int kAttWarps = 4;

struct SegArgs {
    const float* q;
    const float* init_k;
    const float* init_v;
    uint64_t n_init;
    const uint8_t* kcodes;
    const uint8_t* vcodes;
    uint64_t n_comp;
    const float* local_k;
    const float* local_v;
    uint64_t n_local;
    uint32_t group;
    float scale;
    uint64_t init_stride, local_stride;  // rows between pairs (dense: n_init / n_local)
};

struct StackView {
    const StageInfo* stages;
    uint32_t n;
    uint64_t row_bits;
    const float* eff;
    uint64_t stream_bytes;
};

// Build one logical row (key or value) of token t into dst[0..D) (warp-wide).
__device__ __forceinline__ void build_row(const StackView& sv, const uint8_t* codes, const float* init, const float* local,
                                          uint64_t n_init, uint64_t n_comp, uint64_t t, uint32_t D, float* dst,
                                          uint32_t lane) {
    if (t < n_init) {
        for (uint32_t d = lane; d < D; d += 32) dst[d] = init[t * D + d];
    } else if (t < n_init + n_comp) {
        const uint64_t r = t - n_init;
        for (uint32_t d = lane; d < D; d += 32) dst[d] = 0.f;
        for (uint32_t s0 = 0; s0 < sv.n; s0 += 32) {
            uint32_t my = 0;
            if (s0 + lane < sv.n) {
                const StageInfo si = sv.stages[s0 + lane];
                my = read_bits(codes, r * sv.row_bits + si.bit_off, si.bits);
                if (my >= si.size) my = 0;
            }
            const uint32_t cnt = min(32u, sv.n - s0);
            for (uint32_t k = 0; k < cnt; ++k) {
                const uint32_t z = __shfl_sync(0xffffffffu, my, k);
                const float* e = sv.eff + sv.stages[s0 + k].eff_off + uint64_t(z) * D;
                for (uint32_t d = lane; d < D; d += 32) dst[d] = __fadd_rn(dst[d], __ldg(e + d));
            }
        }
    } else {
        const uint64_t l = t - n_init - n_comp;
        for (uint32_t d = lane; d < D; d += 32) dst[d] = local[l * D + d];
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kAttWarps * 32)
attend_generic_kernel(StackView ksv, StackView vsv, SegArgs a, uint32_t Dk, uint32_t Dv, uint64_t per_split,
                      float* __restrict__ part_acc, float* __restrict__ part_m, float* __restrict__ part_l) {
    extern __shared__ float sm[];
    const uint32_t pair = blockIdx.x, split = blockIdx.y, nsplit = gridDim.y;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t G = a.group;
    float* q = sm;                                               // G*Dk
    float* wbase = q + G * Dk + warp * (Dk + Dv + G * Dv + 2 * G);
    float* kr = wbase;                                           // Dk
    float* vr = kr + Dk;                                         // Dv
    float* acc = vr + Dv;                                        // G*Dv
    float* ml = acc + G * Dv;                                    // m[G], l[G]
    for (uint32_t i = threadIdx.x; i < G * Dk; i += blockDim.x) q[i] = a.q[uint64_t(pair) * G * Dk + i];
    for (uint32_t i = lane; i < G * Dv; i += 32) acc[i] = 0.f;
    for (uint32_t g = lane; g < G; g += 32) {  // any group size
        ml[g] = -INFINITY;
        ml[G + g] = 0.f;
    }
    __syncthreads();
    const uint64_t L = a.n_init + a.n_comp + a.n_local;
    const uint64_t t0 = uint64_t(split) * per_split;
    const uint64_t t1 = min(L, t0 + per_split);
    const float* ik = a.init_k + uint64_t(pair) * a.init_stride * Dk;
    const float* iv = a.init_v + uint64_t(pair) * a.init_stride * Dv;
    const float* lk = a.local_k + uint64_t(pair) * a.local_stride * Dk;
    const float* lv = a.local_v + uint64_t(pair) * a.local_stride * Dv;
    const uint8_t* kc = a.kcodes + uint64_t(pair) * ksv.stream_bytes;
    const uint8_t* vc = a.vcodes + uint64_t(pair) * vsv.stream_bytes;
    for (uint64_t t = t0 + warp; t < t1; t += kAttWarps) {
        build_row(ksv, kc, ik, lk, a.n_init, a.n_comp, t, Dk, kr, lane);
        build_row(vsv, vc, iv, lv, a.n_init, a.n_comp, t, Dv, vr, lane);
        for (uint32_t g = 0; g < G; ++g) {
            float part = 0.f;
            for (uint32_t d = lane; d < Dk; d += 32) part = fmaf(q[g * Dk + d], kr[d], part);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            const float logit = part * a.scale;
            const float m_old = ml[g];
            const float m_new = fmaxf(m_old, logit);
            const float c = __expf(m_old - m_new);
            const float p = __expf(logit - m_new);
            for (uint32_t d = lane; d < Dv; d += 32) acc[g * Dv + d] = fmaf(acc[g * Dv + d], c, p * vr[d]);
            __syncwarp();
            if (lane == 0) {
                ml[g] = m_new;
                ml[G + g] = fmaf(ml[G + g], c, p);
            }
            __syncwarp();
        }
    }
    __syncthreads();
    // merge the warps of this CTA into one partial
    const float* w0 = q + G * Dk;
    const uint32_t stride = Dk + Dv + G * Dv + 2 * G;
    for (uint32_t i = threadIdx.x; i < G * Dv; i += blockDim.x) {
        const uint32_t g = i / Dv;
        float M = -INFINITY;
        for (int w = 0; w < kAttWarps; ++w) M = fmaxf(M, w0[w * stride + Dk + Dv + G * Dv + g]);
        float s = 0.f;
        if (M > -INFINITY)
            for (int w = 0; w < kAttWarps; ++w) {
                const float* ww = w0 + w * stride;
                s += ww[Dk + Dv + i] * __expf(ww[Dk + Dv + G * Dv + g] - M);
            }
        part_acc[((uint64_t(pair) * nsplit + split) * G) * Dv + i] = s;
    }
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) {
        float M = -INFINITY;
        for (int w = 0; w < kAttWarps; ++w) M = fmaxf(M, w0[w * stride + Dk + Dv + G * Dv + g]);
        float l = 0.f;
        if (M > -INFINITY)
            for (int w = 0; w < kAttWarps; ++w) {
                const float* ww = w0 + w * stride;
                l += ww[Dk + Dv + G * Dv + G + g] * __expf(ww[Dk + Dv + G * Dv + g] - M);
            }
        part_m[(uint64_t(pair) * nsplit + split) * G + g] = M;
        part_l[(uint64_t(pair) * nsplit + split) * G + g] = l;
    }
}

// Merge splits: one block per (pair, g).
__global__ void split_combine_kernel(const float* __restrict__ part_acc, const float* __restrict__ part_m,
                                     const float* __restrict__ part_l, uint32_t nsplit, uint32_t G, uint32_t Dv,
                                     float* __restrict__ out, float* __restrict__ lse) {
    const uint32_t pg = blockIdx.x;  // pair*G + g
    const uint32_t pair = pg / G, g = pg % G;
    float M = -INFINITY;
    for (uint32_t s = 0; s < nsplit; ++s) M = fmaxf(M, part_m[(uint64_t(pair) * nsplit + s) * G + g]);
    float Lsum = 0.f;
    for (uint32_t s = 0; s < nsplit; ++s) {
        const float m = part_m[(uint64_t(pair) * nsplit + s) * G + g];
        if (m > -INFINITY) Lsum += part_l[(uint64_t(pair) * nsplit + s) * G + g] * __expf(m - M);
    }
    for (uint32_t d = threadIdx.x; d < Dv; d += blockDim.x) {
        float o = 0.f;
        for (uint32_t s = 0; s < nsplit; ++s) {
            const float m = part_m[(uint64_t(pair) * nsplit + s) * G + g];
            if (m > -INFINITY) o += part_acc[((uint64_t(pair) * nsplit + s) * G + g) * Dv + d] * __expf(m - M);
        }
        out[uint64_t(pg) * Dv + d] = o / Lsum;
    }
    if (threadIdx.x == 0 && lse) lse[pg] = M + logf(Lsum);
}

__global__ void lse_combine_kernel(const float* __restrict__ o, const float* __restrict__ lse, uint32_t parts,
                                   uint64_t rows, uint32_t dv, float* __restrict__ out, float* __restrict__ out_lse) {
    const uint64_t row = blockIdx.x;
    float M = -INFINITY;
    for (uint32_t p = 0; p < parts; ++p) M = fmaxf(M, lse[uint64_t(p) * rows + row]);
    float S = 0.f;
    for (uint32_t p = 0; p < parts; ++p) {
        const float v = lse[uint64_t(p) * rows + row];
        if (v > -INFINITY) S += __expf(v - M);
    }
    for (uint32_t d = threadIdx.x; d < dv; d += blockDim.x) {
        float acc = 0.f;
        for (uint32_t p = 0; p < parts; ++p) {
            const float v = lse[uint64_t(p) * rows + row];
            if (v > -INFINITY) acc = fmaf(__expf(v - M) / S, o[(uint64_t(p) * rows + row) * dv + d], acc);
        }
        out[row * dv + d] = acc;
    }
    if (threadIdx.x == 0 && out_lse) out_lse[row] = M + logf(S);
}

}  // namespace

int attend_path() {
    const char* e = getenv("VQKV_ATTEND_PATH");  // 1 = force the generic kernel (tests)
    return e ? atoi(e) : 0;
}

bool attend_lut_supported(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a);
void launch_attend_lut(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a, cudaStream_t s);

// Group sizes other than the LUT kernel's 4 query heads per KV head: the heads run through the LUT
// path in groups of 4 (the last group padded by repeating its last head), each from a compact
// [pair][4][Dk] copy of its queries, the outputs copied back into [pair][group][Dv].  Each group
// re-reads the codes, which still beats the generic per-token kernel by a wide margin.
bool attend_lut_grouped(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a, cudaStream_t s) {
    constexpr uint32_t kLutG = 4;
    if (a.group == kLutG || a.group == 0 || a.n_pairs == 0) return false;
    vqkv_attend_args a4 = a;
    a4.group = kLutG;
    if (!attend_lut_supported(ks, vs, a4)) return false;
    const uint32_t G = a.group, Dk = ks.dim, Dv = vs.dim, P = a.n_pairs;
    float *q4 = nullptr, *o4 = nullptr, *l4 = nullptr;
    VQKV_CUDA(cudaMallocAsync(&q4, sizeof(float) * P * kLutG * Dk, s));
    VQKV_CUDA(cudaMallocAsync(&o4, sizeof(float) * P * kLutG * Dv, s));
    VQKV_CUDA(cudaMallocAsync(&l4, sizeof(float) * P * kLutG, s));
    for (uint32_t h0 = 0; h0 < G; h0 += kLutG) {
        const uint32_t nh = std::min(kLutG, G - h0);
        for (uint32_t j = 0; j < kLutG; ++j) {  // head h0 + j (the last one repeated as padding)
            const uint32_t h = h0 + std::min(j, nh - 1);
            VQKV_CUDA(cudaMemcpy2DAsync(q4 + j * Dk, sizeof(float) * kLutG * Dk, a.q_dev + size_t(h) * Dk,
                                        sizeof(float) * G * Dk, sizeof(float) * Dk, P, cudaMemcpyDeviceToDevice, s));
        }
        a4.q_dev = q4;
        a4.out_dev = o4;
        a4.lse_dev = a.lse_dev ? l4 : nullptr;
        launch_attend_lut(ks, vs, a4, s);
        VQKV_CUDA(cudaMemcpy2DAsync(a.out_dev + size_t(h0) * Dv, sizeof(float) * G * Dv, o4, sizeof(float) * kLutG * Dv,
                                    sizeof(float) * nh * Dv, P, cudaMemcpyDeviceToDevice, s));
        if (a.lse_dev)
            VQKV_CUDA(cudaMemcpy2DAsync(a.lse_dev + h0, sizeof(float) * G, l4, sizeof(float) * kLutG, sizeof(float) * nh, P,
                                        cudaMemcpyDeviceToDevice, s));
    }
    VQKV_CUDA(cudaFreeAsync(q4, s));
    VQKV_CUDA(cudaFreeAsync(o4, s));
    VQKV_CUDA(cudaFreeAsync(l4, s));
    return true;
}

void launch_attend(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a, cudaStream_t s) {
    if (attend_path() != 1 && attend_lut_supported(ks, vs, a)) {
        launch_attend_lut(ks, vs, a, s);
        return;
    }
    if (attend_path() != 1 && attend_lut_grouped(ks, vs, a, s)) return;
    const uint32_t Dk = ks.dim, Dv = vs.dim, G = a.group;
    const uint64_t L = a.n_init + a.n_comp + a.n_local;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ks.device);
    // enough splits for ~4 CTAs per SM, at least 64 tokens each
    uint64_t want = std::max<uint64_t>(1, (uint64_t(sms) * 4 + a.n_pairs - 1) / a.n_pairs);
    uint64_t nsplit = std::min<uint64_t>(want, std::max<uint64_t>(1, (L + 63) / 64));
    nsplit = std::min<uint64_t>(nsplit, 65535);
    const uint64_t per_split = (L + nsplit - 1) / nsplit;
    nsplit = (L + per_split - 1) / per_split;
    float *pacc = nullptr, *pm = nullptr, *pl = nullptr;
    VQKV_CUDA(cudaMallocAsync(&pacc, sizeof(float) * a.n_pairs * nsplit * G * Dv, s));
    VQKV_CUDA(cudaMallocAsync(&pm, sizeof(float) * a.n_pairs * nsplit * G, s));
    VQKV_CUDA(cudaMallocAsync(&pl, sizeof(float) * a.n_pairs * nsplit * G, s));
    StackView ksv{ks.d_stages, ks.n, ks.row_bits, ks.d_eff,
                  a.kcodes_stride ? a.kcodes_stride : payload_bytes(ks.row_bits, a.n_comp)};
    StackView vsv{vs.d_stages, vs.n, vs.row_bits, vs.d_eff,
                  a.vcodes_stride ? a.vcodes_stride : payload_bytes(vs.row_bits, a.n_comp)};
    const double scale = a.scale > 0.0 ? a.scale : 1.0 / std::sqrt(double(Dk));
    SegArgs sa{a.q_dev, a.init_k_dev, a.init_v_dev, a.n_init, a.kcodes_dev, a.vcodes_dev, a.n_comp,
               a.local_k_dev, a.local_v_dev, a.n_local, G, float(scale),
               a.init_stride ? a.init_stride : a.n_init, a.local_stride ? a.local_stride : a.n_local};
    const size_t smem = sizeof(float) * (G * Dk + kAttWarps * (Dk + Dv + G * Dv + 2 * G));
    if (smem > 227 * 1024) fail(VQKV_UNSUPPORTED, "attention head shape too large for shared memory");
    if (smem > 48 * 1024)
        VQKV_CUDA(cudaFuncSetAttribute(attend_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 grid(a.n_pairs, unsigned(nsplit));
    {
    ProfScope ps("attend", s);
    attend_generic_kernel<<<grid, kAttWarps * 32, smem, s>>>(ksv, vsv, sa, Dk, Dv, per_split, pacc, pm, pl);
    launch_check("attend_generic_kernel");
    }
    {
    ProfScope ps2("attend_combine", s);
    split_combine_kernel<<<a.n_pairs * G, 128, 0, s>>>(pacc, pm, pl, unsigned(nsplit), G, Dv, a.out_dev, a.lse_dev);
    launch_check("split_combine_kernel");
    }
    VQKV_CUDA(cudaFreeAsync(pacc, s));
    VQKV_CUDA(cudaFreeAsync(pm, s));
    VQKV_CUDA(cudaFreeAsync(pl, s));
}

// attend_raw (attention.cpp:71-88): softmax(scale q K^T) V over raw rows only, one query --
// the generic kernel with every row in the "local" segment (no codebooks are touched).
void launch_attend_raw(int device, const float* keys, const float* values, uint64_t rows, uint32_t dk, uint32_t dv,
                       const float* q, double scale, float* out, cudaStream_t s) {
    vqkv_stack_s ks, vs;  // shape-only views: n_comp = 0, so no stage table is read
    ks.device = vs.device = device;
    ks.dim = dk;
    vs.dim = dv;
    vqkv_attend_args a{};
    a.n_pairs = 1;
    a.group = 1;
    a.q_dev = q;
    a.local_k_dev = keys;
    a.local_v_dev = values;
    a.n_local = rows;
    a.scale = scale;
    a.out_dev = out;
    launch_attend(ks, vs, a, s);
}

void launch_lse_combine(const float* o, const float* lse, uint32_t parts, uint64_t rows, uint32_t dv, float* out,
                        float* out_lse, cudaStream_t s) {
    lse_combine_kernel<<<unsigned(rows), 128, 0, s>>>(o, lse, parts, rows, dv, out, out_lse);
    launch_check("lse_combine_kernel");
}

}  // namespace vqkv_dev
