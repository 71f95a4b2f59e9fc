// attend_lut.cu -- K3 fast path: decode-step attention over the compressed
// cache in the dot-product domain (D = 128, G = 4 query heads per KV head).
//
// Reference: attend (proj/core/src/attention.cpp:26-69) over
// CacheState::view_block (kv_cache.cpp:143-189), whose compressed rows are
// reconstruct() sums (codebook.cpp:208-223).  Because reconstruction is a sum
// of codebook rows, for every query q_g
//     scale * q_g . k_t = sum_s LUT_s[z_s,t][g],   LUT_s[j][g] = scale * q_g . e_s[j]
//     sum_t p_t,g v_t   = sum_s sum_j H_s[j][g] e_s[j],  H_s[j][g] = sum_{t: z_s,t = j} p_t,g
// so keys cost one table lookup per (token, stage) and values one histogram
// update per (token, stage); neither K nor V rows are ever materialised.
//
// Kernels (one launch each, all on the caller's stream):
//   lut_kernel      LUT[pair][s][j] = float4 over g, fp32 (FFMA from the
//                   fp32 effective entries; the table stays L2-hot per pair)
//   attend_lut      CTA = (pair, split of <= 8192 compressed tokens):
//                   keys: 4-stage LUT groups double-buffered into smem by bulk
//                   copy (TMA engine), one LDS.128 + 4 FADD per (token, stage);
//                   split max; p = exp(logit - max); values: int32 fixed-point
//                   (2^-18) smem histograms via native shared atomics;
//                   writes (H as fp32, m, l).  One extra CTA per pair handles
//                   the raw init/local rows directly (o_acc, m, l).
//   lut_combine     per pair: merge splits by LSE weights, contract H with the
//                   value codebooks, add the raw part, normalise, emit lse.
#include <algorithm>
#include <cmath>
#include <vector>

#include "tc_ptx.cuh"
#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

constexpr int kG = 4;              // query heads per KV head on this path
constexpr int kD = 128;            // head dim
constexpr int kAttThreads = 512;
constexpr int kTokPerThread = 16;
constexpr int kSplitTokens = kAttThreads * kTokPerThread;  // 8192
constexpr int kMaxVStages = 64;    // value stages supported by the LUT path
constexpr int kKeyBatch = 4;
constexpr uint32_t kQueueCap = 64;                       // per-warp value-token queue entries
constexpr uint32_t kQueueOff = 131072 + 1024;             // smem offset of the queues (after the control area)
constexpr uint32_t kMainSmem = kQueueOff + (kAttThreads / 32) * kQueueCap * (1 + 4) * 4;      // key tokens whose code loads are in flight together
constexpr int kGroupStages = 4;    // LUT stages per smem buffer (4 x 16 KB)
constexpr uint32_t kGmCodeOff = 131072 + 1024;               // == kQueueOff: queues are used after the keys
constexpr uint32_t kGmCodeBuf = 5 * kSplitTokens;              // one group's records of a split (40 KB)
constexpr uint32_t kAlignSlack = 16384 - 1024;                 // 1 KB-aligned window start -> 16 KB alignment
constexpr uint32_t kGmSmem = kGmCodeOff + 2 * kGmCodeBuf;
constexpr float kHistScale = 262144.0f;  // 2^18 fixed point for p in [0, 1]

struct LutArgs {
    const float* q;        // [pairs][G][D]
    const float* keff;     // key effective entries
    const StageInfo* kst;
    uint32_t kn;
    uint64_t kentries;     // total key entries (sum S)
    float scale;
    float4* lut;           // [pairs][kentries]
};

// LUT[pair][e] = scale * q_g . E[e] for all key entries e (stage-concatenated).
// CTA: 128 entries x 8 pairs, 256 threads; thread = 4 entries x 4 queries of one pair.
constexpr int kLutEntries = 128;
constexpr int kLutStride = kD + 2;  // even row stride: 8 B-aligned float2 reads, 2 wavefronts per warp load
__global__ void __launch_bounds__(256) lut_kernel(LutArgs a, uint32_t n_pairs) {
    extern __shared__ float lsm[];
    float4* qs = reinterpret_cast<float4*>(lsm);  // [8 pairs][D] x float4 over g: one LDS.128 per dim
    float* es = lsm + 8 * kG * kD;                // [128 entries][kLutStride]
    const uint32_t e0 = blockIdx.x * kLutEntries, p0 = blockIdx.y * 8;
    for (uint32_t i = threadIdx.x; i < 8 * kD; i += blockDim.x) {
        const uint32_t p = i / kD, c = i % kD;
        const float* qp = a.q + uint64_t(p0 + p) * kG * kD + c;
        qs[i] = (p0 + p < n_pairs) ? make_float4(qp[0], qp[kD], qp[2 * kD], qp[3 * kD]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (uint32_t i = threadIdx.x; i < kLutEntries * kD / 4; i += blockDim.x) {
        const uint32_t r = (4 * i) / kD, c = (4 * i) % kD;
        const float4 v = (e0 + r < a.kentries) ? __ldg(reinterpret_cast<const float4*>(a.keff + uint64_t(e0 + r) * kD + c))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float2*>(es + r * kLutStride + c) = make_float2(v.x, v.y);
        *reinterpret_cast<float2*>(es + r * kLutStride + c + 2) = make_float2(v.z, v.w);
    }
    __syncthreads();
    const uint32_t eg = threadIdx.x & 31, p = threadIdx.x >> 5;
    __align__(8) float acc[4][kG];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int g = 0; g < kG; ++g) acc[i][g] = 0.f;
    const float4* qp = qs + p * kD;
#pragma unroll 4
    for (int c = 0; c < kD; c += 2) {
        const float4 q0 = qp[c], q1 = qp[c + 1];  // broadcast within the warp
        float2 ev[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) ev[i] = *reinterpret_cast<const float2*>(es + (eg + 32 * i) * kLutStride + c);
        // packed FFMA2 over head pairs: per lane the same fmaf sequence as scalar code
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2* a2 = reinterpret_cast<float2*>(acc[i]);
            const float2 ex = make_float2(ev[i].x, ev[i].x), ey = make_float2(ev[i].y, ev[i].y);
            a2[0] = ptx::fma2(make_float2(q0.x, q0.y), ex, a2[0]);
            a2[1] = ptx::fma2(make_float2(q0.z, q0.w), ex, a2[1]);
            a2[0] = ptx::fma2(make_float2(q1.x, q1.y), ey, a2[0]);
            a2[1] = ptx::fma2(make_float2(q1.z, q1.w), ey, a2[1]);
        }
    }
    if (p0 + p < n_pairs)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t e = e0 + eg + 32 * i;
            if (e < a.kentries)
                a.lut[uint64_t(p0 + p) * a.kentries + e] = make_float4(acc[i][0] * a.scale, acc[i][1] * a.scale,
                                                                        acc[i][2] * a.scale, acc[i][3] * a.scale);
        }
}

// ---- LUT build on the tensor cores --------------------------------------------------------
// The LUT is a GEMM: LUT[pair][e][g] = scale * E[e] . q[pair][g], i.e. [entries x 128] x
// [128 x (pairs * G)].  fp16 split precision: E = E_hi + E_lo (stack operands, the encoder's
// pre-swizzled chunks), q 2^sigma = Q_hi + Q_lo (per row power-of-two scale, exact), and
// E_hi Q_lo + E_lo Q_hi + E_hi Q_hi accumulate in fp32 in TMEM; the dropped E_lo Q_lo and the
// lo roundings are ~2^-22 relative to sum_k |E_k q_k|, the fp32 FFMA LUT's own error level.
// q_prep_kernel: one warp per (pair, g) row -> Q_hi / Q_lo in 128-row SW128 K-major tiles
// (the half_copy_kernel layout) and qscl[row] = scale * 2^-sigma.
__global__ void q_prep_kernel(const float* __restrict__ q, uint32_t n_rows, uint32_t n_rows_pad, float scale,
                              __half* __restrict__ qhi, __half* __restrict__ qlo, float* __restrict__ qscl) {
    const uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= n_rows_pad) return;
    float4 v = (r < n_rows) ? reinterpret_cast<const float4*>(q + uint64_t(r) * kD)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    float m = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    int sig = 0;
    if (m > 0.f && isfinite(m)) {
        int e;
        frexpf(m, &e);  // m in [2^(e-1), 2^e): m 2^sig < 2^14
        sig = min(100, max(-100, 14 - e));
    }
    const float sc = ldexpf(1.0f, sig);
    const float x[4] = {v.x * sc, v.y * sc, v.z * sc, v.w * sc};
    const uint32_t t = r >> 7, rr = r & 127;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t k = lane * 4 + i, kb = k >> 6, kk = k & 63;
        const uint64_t off = uint64_t(t) * 16384 + kb * 8192 + rr * 64 + (((kk >> 3) ^ (rr & 7)) << 3) + (kk & 7);
        const __half h = __float2half_rn(x[i]);
        qhi[off] = h;
        qlo[off] = __float2half_rn(x[i] - __half2float(h));
    }
    if (lane == 0) qscl[r] = (r < n_rows) ? ldexpf(scale, -sig) : 0.f;
}

// CTA = 128-entry chunk c of key stage s, looping over the 128-row tiles of (pair, g) query
// rows.  Warp 4 (one thread) loads the chunk's E_hi / E_lo once and double-buffers the Q tiles
// by bulk copy, and issues 24 MMAs M128 N128 K16 per tile into one of two TMEM accumulators;
// warps 0-3 (thread = entry row = TMEM lane) drain the other accumulator meanwhile: 32 pairs'
// float4 per thread and tile, coalesced across lanes.
constexpr uint32_t kLutTcSmem = 6 * 32768 + 1024;
__global__ void __launch_bounds__(160) lut_tc_kernel(const __half* __restrict__ eff16, const __half* __restrict__ eff16lo,
                                                     const StageInfo* __restrict__ kst, const __half* __restrict__ qhi,
                                                     const __half* __restrict__ qlo, const float* __restrict__ qscl,
                                                     uint32_t n_pairs, uint32_t n_qtiles, uint64_t kentries,
                                                     float4* __restrict__ lut) {
    extern __shared__ uint8_t lsm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_e, bar_q[2], bar_mma[2], bar_epi[2];
    __shared__ uint32_t tmem_base;
    const StageInfo si = kst[blockIdx.y];
    const uint32_t c = blockIdx.x;
    if (c * 128 >= si.size) return;  // uniform per CTA
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar_e), 1);
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(ptx::smem_u32(&bar_q[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&bar_mma[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&bar_epi[b]), 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 256);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t s_ehi = ptx::smem_u32(sm), s_elo = s_ehi + 32768;
    auto s_qhi = [&](uint32_t b) { return s_ehi + 65536 + b * 65536; };
    if (warp == 4) {
        if (lane == 0) {
            const uint64_t eo = si.eff16_off + uint64_t(c) * 18432;
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar_e), 2 * 32768);
            ptx::bulk_g2s(s_ehi, eff16 + eo, 32768, ptx::smem_u32(&bar_e));
            ptx::bulk_g2s(s_elo, eff16lo + eo, 32768, ptx::smem_u32(&bar_e));
            auto load_q = [&](uint32_t tq) {
                const uint32_t b = tq & 1, bar = ptx::smem_u32(&bar_q[b]);
                ptx::mbar_arrive_expect_tx(bar, 2 * 32768);
                ptx::bulk_g2s(s_qhi(b), qhi + uint64_t(tq) * 16384, 32768, bar);
                ptx::bulk_g2s(s_qhi(b) + 32768, qlo + uint64_t(tq) * 16384, 32768, bar);
            };
            load_q(0);
            if (n_qtiles > 1) load_q(1);
            ptx::mbar_wait(ptx::smem_u32(&bar_e), 0);
            constexpr uint32_t idesc = ptx::idesc_f16_f32(128, 128);
            for (uint32_t tq = 0; tq < n_qtiles; ++tq) {
                const uint32_t b = tq & 1, use = tq >> 1;
                ptx::mbar_wait(ptx::smem_u32(&bar_q[b]), use & 1);
                if (tq >= 2) ptx::mbar_wait(ptx::smem_u32(&bar_epi[b]), (use - 1) & 1);  // accumulator b drained
                ptx::tc_fence_after();
                const uint32_t qh = s_qhi(b), ql = qh + 32768;
                const uint32_t A[3] = {s_ehi, s_elo, s_ehi}, B[3] = {ql, qh, qh};  // small terms first
#pragma unroll
                for (int part = 0; part < 3; ++part)
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t koff = (k >> 2) * 16384 + (k & 3) * 32;
                        ptx::mma_f16_ss(tmem + 128u * b, ptx::umma_desc_sw128(A[part] + koff),
                                        ptx::umma_desc_sw128(B[part] + koff), idesc, (part | k) ? 1u : 0u);
                    }
                ptx::mma_commit(ptx::smem_u32(&bar_mma[b]));
                if (tq + 2 < n_qtiles) {
                    // Q buffer b is free once these MMAs complete
                    ptx::mbar_wait(ptx::smem_u32(&bar_mma[b]), use & 1);
                    load_q(tq + 2);
                }
            }
        }
    } else {
        const uint32_t j = c * 128 + warp * 32 + lane;  // entry within the stage
        const uint64_t e = si.eff_off / kD + j;
        for (uint32_t tq = 0; tq < n_qtiles; ++tq) {
            const uint32_t b = tq & 1, use = tq >> 1;
            ptx::mbar_wait(ptx::smem_u32(&bar_mma[b]), use & 1);
            ptx::tc_fence_after();
            const float* sclp = qscl + uint64_t(tq) * 128;
            float v[4][32];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) ptx::tmem_ld32(tmem + ((warp * 32u) << 16) + 128u * b + 32u * c4, v[c4]);
            ptx::tc_wait_ld();
            ptx::tc_fence_before();
            ptx::mbar_arrive(ptx::smem_u32(&bar_epi[b]));
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)
#pragma unroll
                for (int pp = 0; pp < 8; ++pp) {
                    const uint32_t pair = tq * 32 + c4 * 8 + pp;
                    if (j < si.size && pair < n_pairs) {
                        const float4 sc = __ldg(reinterpret_cast<const float4*>(sclp) + c4 * 8 + pp);
                        lut[uint64_t(pair) * kentries + e] = (
                               make_float4(v[c4][4 * pp] * sc.x, v[c4][4 * pp + 1] * sc.y, v[c4][4 * pp + 2] * sc.z,
                                           v[c4][4 * pp + 3] * sc.w));
                    }
                }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}

// ---- int16 LUT (opt-in, VQKV_ATTEND_INT16=1) -------------------------------------------
// One scale per (pair, head): Δ = max_e |LUT[e][g]| / 32767, entries stored as biased u16
// (round(L / Δ) + 32768, 4 heads in 8 B) and summed exactly in int32 by the main kernel (GM = 2):
// per-logit error ≤ n_stages · Δ / 2 against the fp32 LUT.
// CTA = pair: max_e |LUT[e][g]| over the pair's fp32 LUT, then the quantised copy (the second
// read of the pair's 0.9 MB hits L2).
__global__ void __launch_bounds__(1024) lut_int16_kernel(const float4* __restrict__ lut, uint64_t kentries,
                                                         uint2* __restrict__ lut16, float* __restrict__ dq) {
    __shared__ float red[32][kG];
    __shared__ float smax[kG];
    const uint32_t pair = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float4* L = lut + uint64_t(pair) * kentries;
    constexpr int kU = 8;  // loads in flight per thread
    float m[kG] = {0.f, 0.f, 0.f, 0.f};
    for (uint64_t e0 = threadIdx.x; e0 < kentries; e0 += uint64_t(kU) * blockDim.x) {
        float4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t e = e0 + uint64_t(u) * blockDim.x;
            v[u] = e < kentries ? __ldg(L + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const float x[kG] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int g = 0; g < kG; ++g) m[g] = fmaxf(m[g], isfinite(x[g]) ? fabsf(x[g]) : INFINITY);  // non-finite -> NaN logits
        }
    }
#pragma unroll
    for (int g = 0; g < kG; ++g) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m[g] = fmaxf(m[g], __shfl_xor_sync(0xffffffffu, m[g], o));
        if (lane == 0) red[warp][g] = m[g];
    }
    __syncthreads();
    if (threadIdx.x < kG) {
        float r = 0.f;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) r = fmaxf(r, red[w][threadIdx.x]);
        smax[threadIdx.x] = r;
        dq[pair * kG + threadIdx.x] = r / 32767.0f;
    }
    __syncthreads();
    float inv[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) inv[g] = smax[g] > 0.f ? 32767.0f / smax[g] : 0.f;
    uint2* Q = lut16 + uint64_t(pair) * kentries;
    for (uint64_t e0 = threadIdx.x; e0 < kentries; e0 += uint64_t(kU) * blockDim.x) {
        float4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t e = e0 + uint64_t(u) * blockDim.x;
            v[u] = e < kentries ? __ldg(L + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t e = e0 + uint64_t(u) * blockDim.x;
            const float x[kG] = {v[u].x, v[u].y, v[u].z, v[u].w};
            uint32_t q[kG];
#pragma unroll
            for (int g = 0; g < kG; ++g) q[g] = uint32_t(max(-32767, min(32767, __float2int_rn(x[g] * inv[g]))) + 32768);
            if (e < kentries) Q[e] = make_uint2(q[0] | q[1] << 16, q[2] | q[3] << 16);
        }
    }
}

// Reads 64 bits starting at bit `pos` of a byte stream: two aligned 64-bit
// loads when they stay inside [.., end), byte loads otherwise (buffer tails).
__device__ __forceinline__ uint64_t read_bits64(const uint8_t* base, uint64_t pos, const uint8_t* end) {
    const uint8_t* p = base + (pos >> 3);
    const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(7);
    const uint32_t sh = uint32_t((reinterpret_cast<uintptr_t>(p) - a) * 8 + (pos & 7));
    if (a + 16 <= reinterpret_cast<uintptr_t>(end)) {
        const uint64_t* q = reinterpret_cast<const uint64_t*>(a);
        const uint64_t lo = __ldg(q), hi = __ldg(q + 1);
        return sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
    }
    uint64_t v = 0;
    const uint32_t bsh = uint32_t(pos & 7);
    for (int b = 0; b < 8 && p + b < end; ++b) v |= uint64_t(p[b]) << (8 * b);
    uint64_t extra = (p + 8 < end) ? uint64_t(p[8]) : 0ull;
    return bsh ? ((v >> bsh) | (extra << (64 - bsh))) : v;
}

// always-valid 16 bytes: the target of clamped (ignored) loads in the batched key loop
__device__ const uint64_t g_zero16[2] = {0ull, 0ull};

struct MainArgs {
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
    const StageInfo* kst;
    uint32_t kn;
    uint64_t krow_bits, kstream_bytes, kentries;
    const StageInfo* vst;
    uint32_t vn;
    uint64_t vrow_bits, vstream_bytes, ventries;
    const float4* lut;
    const uint8_t* kend;
    const uint8_t* vend;
    float scale;
    uint32_t n_splits;  // compressed splits per pair (+1 raw CTA)
    float* part_h;      // [pairs][splits][ventries][G]
    float* part_o;      // [pairs][G][D]  (raw CTA)
    float* part_m;      // [pairs][splits+1][G]
    float* part_l;      // [pairs][splits+1][G]
    uint64_t init_stride, local_stride;  // rows between pairs
    uint64_t gm_cap;                     // group-major key codes: token capacity per group segment
    const uint2* lut16;                  // GM = 2: int16 LUT (biased u16, 4 heads)
    const float* dq;                     // GM = 2: [pairs][G] scale of the int16 LUT
};

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = -INFINITY;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
    return r;
}
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float r = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) r += red[w];
    return r;
}

// raw init/local rows of one pair: direct fp32 attention (no codebooks).  Latency matters
// here (one CTA per pair runs beside the split CTAs): rows are read in batches with all
// their loads in flight, and every value load feeds the 4 heads.
__device__ void raw_rows(const MainArgs& a, uint32_t pair, float* smem) {
    constexpr int kRowBatch = 8;
    float* red = smem;                 // 64
    float* qs = smem + 64;             // G*D
    float* ls = qs + kG * kD;          // logits / weights [n_raw][G] (n_raw <= 8192)
    float* po = ls + kSplitTokens * kG;  // [4 row groups][G][D] partial outputs
    for (uint32_t i = threadIdx.x; i < kG * kD; i += blockDim.x) qs[i] = a.q[uint64_t(pair) * kG * kD + i];
    __syncthreads();
    const uint32_t n_raw = uint32_t(a.n_init + a.n_local);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    auto krow = [&](uint32_t r) -> const float4* {
        return reinterpret_cast<const float4*>(
            (r < a.n_init) ? a.init_k + (uint64_t(pair) * a.init_stride + r) * kD
                           : a.local_k + (uint64_t(pair) * a.local_stride + (r - a.n_init)) * kD);
    };
    float4 qv[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) qv[g] = reinterpret_cast<const float4*>(qs + g * kD)[lane];
    const bool up = lane & 16u, b3 = lane & 8u;
    for (uint32_t r0 = warp; r0 < n_raw; r0 += nw * kRowBatch) {
        float4 kv[kRowBatch];
#pragma unroll
        for (int u = 0; u < kRowBatch; ++u) {
            const uint32_t r = r0 + u * nw;
            kv[u] = (r < n_raw) ? __ldg(krow(r) + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kRowBatch; ++u) {
            float d[kG];
#pragma unroll
            for (int g = 0; g < kG; ++g)
                d[g] = kv[u].x * qv[g].x + kv[u].y * qv[g].y + kv[u].z * qv[g].z + kv[u].w * qv[g].w;
            // 4-value butterfly: 6 shuffles leave head 2*bit4 + bit3 summed over the warp
            float k0 = up ? d[2] : d[0], k1 = up ? d[3] : d[1];
            k0 += __shfl_xor_sync(0xffffffffu, up ? d[0] : d[2], 16);
            k1 += __shfl_xor_sync(0xffffffffu, up ? d[1] : d[3], 16);
            float k = b3 ? k1 : k0;
            k += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
            k += __shfl_xor_sync(0xffffffffu, k, 4);
            k += __shfl_xor_sync(0xffffffffu, k, 2);
            k += __shfl_xor_sync(0xffffffffu, k, 1);
            const uint32_t r = r0 + u * nw;
            if ((lane & 7u) == 0 && r < n_raw) ls[r * kG + (lane >> 3)] = k * a.scale;
        }
    }
    __syncthreads();
    for (int g = 0; g < kG; ++g) {
        float m = -INFINITY;
        for (uint32_t r = threadIdx.x; r < n_raw; r += blockDim.x) m = fmaxf(m, ls[r * kG + g]);
        m = block_max(m, red);
        float l = 0.f;
        for (uint32_t r = threadIdx.x; r < n_raw; r += blockDim.x) {
            const float p = __expf(ls[r * kG + g] - m);
            ls[r * kG + g] = p;
            l += p;
        }
        l = block_sum(l, red);
        if (threadIdx.x == 0) {
            a.part_m[(uint64_t(pair) * (a.n_splits + 1) + a.n_splits) * kG + g] = m;
            a.part_l[(uint64_t(pair) * (a.n_splits + 1) + a.n_splits) * kG + g] = l;
        }
    }
    __syncthreads();
    // o[g][d] = sum_r p[r][g] v_r[d]: thread = (row group rg, d) over rows rg, rg + 4, ...;
    // each value load feeds the 4 heads, kRowBatch loads in flight
    {
        const uint32_t d = threadIdx.x % kD, rg = threadIdx.x / kD, nrg = blockDim.x / kD;
        const float* iv = a.init_v + uint64_t(pair) * a.init_stride * kD + d;
        const float* lv = a.local_v + uint64_t(pair) * a.local_stride * kD + d;
        const float4* p4 = reinterpret_cast<const float4*>(ls);
        float acc[kG] = {0.f, 0.f, 0.f, 0.f};
        for (uint32_t r0 = rg; r0 < n_raw; r0 += nrg * kRowBatch) {
            float x[kRowBatch];
#pragma unroll
            for (int u = 0; u < kRowBatch; ++u) {
                const uint32_t r = r0 + u * nrg;
                x[u] = (r >= n_raw) ? 0.f : (r < a.n_init) ? __ldg(iv + uint64_t(r) * kD) : __ldg(lv + uint64_t(r - a.n_init) * kD);
            }
#pragma unroll
            for (int u = 0; u < kRowBatch; ++u) {
                const uint32_t r = r0 + u * nrg;
                if (r < n_raw) {
                    const float4 p = p4[r];
                    acc[0] = fmaf(p.x, x[u], acc[0]);
                    acc[1] = fmaf(p.y, x[u], acc[1]);
                    acc[2] = fmaf(p.z, x[u], acc[2]);
                    acc[3] = fmaf(p.w, x[u], acc[3]);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < kG; ++g) po[(rg * kG + g) * kD + d] = acc[g];
    }
    __syncthreads();
    const uint32_t nrg = blockDim.x / kD;
    for (uint32_t gd = threadIdx.x; gd < kG * kD; gd += blockDim.x) {
        float o = 0.f;
        for (uint32_t rg = 0; rg < nrg; ++rg) o += po[rg * kG * kD + gd];
        a.part_o[uint64_t(pair) * kG * kD + gd] = o;
    }
}

__device__ __forceinline__ void lds128(uint32_t addr, float2& a, float2& b) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y) : "r"(addr));
}

__device__ __forceinline__ void lds64(uint32_t addr, uint2& w) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "r"(addr));
}

// GM = 1: key codes in the group-major layout (attend_lut.cu, "group-major key codes"):
// per LUT group one bulk copy of the split's 5-byte records lands next to the LUT group,
// so every code byte crosses L2 -> SM once, and a lookup is SHF + LOP3 + LDS.128 + 2 FADD2
// (slot address = 16 KB-aligned stage slot | code << 4).  GM = 0: reference CodeMatrix rows,
// re-read per LUT group through L1/L2 (any geometry the LUT path supports).
template <int GM>
__global__ void __launch_bounds__(kAttThreads, 1) attend_lut_kernel(MainArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pair = blockIdx.y, split = blockIdx.x;
    float* fsm = reinterpret_cast<float*>(smem_raw);
    if (split == a.n_splits) {
        if (a.n_init + a.n_local > 0) {
            raw_rows(a, pair, fsm);
        } else if (threadIdx.x < kG) {
            a.part_m[(uint64_t(pair) * (a.n_splits + 1) + a.n_splits) * kG + threadIdx.x] = -INFINITY;
            a.part_l[(uint64_t(pair) * (a.n_splits + 1) + a.n_splits) * kG + threadIdx.x] = 0.f;
        }
        return;
    }
    // smem: [0, 128K) two LUT group buffers (2 x 4 stages x 1024 x 16 B) / value histograms
    //       then mbarriers and reduction scratch
    // the layout below starts at the first 16 KB-aligned shared address (the window
    // starts after the 1 KB system reservation), so a LUT slot address is base | code << 4
    uint8_t* const sm = smem_raw + ((16384u - (ptx::smem_u32(smem_raw) & 16383u)) & 16383u);
    uint8_t* lut_buf = sm;
    uint8_t* code_buf = sm + kGmCodeOff;  // GM: two record buffers (the value queues reuse them later)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 131072);
    float* red = reinterpret_cast<float*>(sm + 131072 + 64);
    const uint64_t t0 = uint64_t(split) * kSplitTokens;
    const uint64_t nt = (a.n_comp - t0 < uint64_t(kSplitTokens)) ? (a.n_comp - t0) : uint64_t(kSplitTokens);
    const uint8_t* kc = a.kcodes + uint64_t(pair) * a.kstream_bytes;
    const uint8_t* vc = a.vcodes + uint64_t(pair) * a.vstream_bytes;
    const float4* lutp = a.lut + uint64_t(pair) * a.kentries;
    // 32-bit key-code addressing: bit positions relative to the 8 B-aligned start of the
    // pair's stream (stream bit counts < 2^32 are checked on the host)
    const uint64_t* kc64 = reinterpret_cast<const uint64_t*>(reinterpret_cast<uintptr_t>(kc) & ~uintptr_t(7));
    const uint32_t kbase_bits = uint32_t((reinterpret_cast<uintptr_t>(kc) & 7u) * 8u);
    const uint32_t kwords = uint32_t((reinterpret_cast<uintptr_t>(a.kend) - reinterpret_cast<uintptr_t>(kc64)) >> 3 > 0xffffffffull
                                         ? 0xffffffffu
                                         : (reinterpret_cast<uintptr_t>(a.kend) - reinterpret_cast<uintptr_t>(kc64)) >> 3);
    const uint32_t krow32 = uint32_t(a.krow_bits);
    const uint64_t* vc64 = reinterpret_cast<const uint64_t*>(reinterpret_cast<uintptr_t>(vc) & ~uintptr_t(7));
    const uint32_t vbase_bits = uint32_t((reinterpret_cast<uintptr_t>(vc) & 7u) * 8u);
    const uint32_t vwords = uint32_t((reinterpret_cast<uintptr_t>(a.vend) - reinterpret_cast<uintptr_t>(vc64)) >> 3 > 0xffffffffull
                                         ? 0xffffffffu
                                         : (reinterpret_cast<uintptr_t>(a.vend) - reinterpret_cast<uintptr_t>(vc64)) >> 3);
    const uint32_t vrow32 = uint32_t(a.vrow_bits);
    const uint32_t nvwin = (a.vn + 5u) / 6u;

    float lg[kTokPerThread][kG];
#pragma unroll
    for (int k = 0; k < kTokPerThread; ++k)
#pragma unroll
        for (int g = 0; g < kG; ++g) lg[k][g] = 0.f;
    // the key logits accumulate as head pairs with packed FADD2 (2 instructions per lookup)
    float2 (*lg2)[2] = reinterpret_cast<float2 (*)[2]>(lg);
    uint32_t il[GM == 2 ? kTokPerThread : 1][kG];  // GM = 2: exact sums of the biased int16 entries
#pragma unroll
    for (int k = 0; k < (GM == 2 ? kTokPerThread : 1); ++k)
#pragma unroll
        for (int g = 0; g < kG; ++g) il[k][g] = 0u;

    // ---- keys: LUT groups of kGroupStages stages, double-buffered bulk copies
    const uint32_t ngroups = (a.kn + kGroupStages - 1) / kGroupStages;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bars[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&bars[1]), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](uint32_t grp) {
        const uint32_t b = grp & 1;
        const uint32_t s0 = grp * kGroupStages;
        const uint32_t s1 = min(a.kn, s0 + kGroupStages);
        uint32_t bytes = 0;
        for (uint32_t s = s0; s < s1; ++s) bytes += a.kst[s].size * 16u;
        const uint32_t bar = ptx::smem_u32(&bars[b]);
        if constexpr (GM == 2) {
            // int16 LUT: stage q -> 8 KB slot q (entry = 4 biased u16); missing stages as in GM = 1
            uint32_t hb = 0;
            for (uint32_t st = s0; st < s1; ++st) hb += a.kst[st].size * 8u;
            const uint32_t clo = uint32_t((nt * 4 + 15) & ~uint64_t(15)), chi = uint32_t((nt + 15) & ~uint64_t(15));
            ptx::mbar_arrive_expect_tx(bar, hb + (kGroupStages - (s1 - s0)) * 16u + clo + chi);
            const uint2* l16 = a.lut16 + uint64_t(pair) * a.kentries;
            for (uint32_t st = s0; st < s0 + kGroupStages; ++st) {
                uint8_t* dst = lut_buf + b * 65536 + (st - s0) * 8192;
                if (st < s1)
                    ptx::bulk_g2s(ptx::smem_u32(dst), l16 + a.kst[st].eff_off / kD, a.kst[st].size * 8u, bar);
                else
                    ptx::bulk_g2s(ptx::smem_u32(dst), g_zero16, 16u, bar);
            }
            const uint8_t* seg = kc + uint64_t(grp) * a.gm_cap * 5;
            ptx::bulk_g2s(ptx::smem_u32(code_buf + b * kGmCodeBuf), seg + t0 * 4, clo, bar);
            ptx::bulk_g2s(ptx::smem_u32(code_buf + b * kGmCodeBuf + 4 * kSplitTokens), seg + a.gm_cap * 4 + t0, chi, bar);
        } else if constexpr (GM == 1) {
            // stage q -> 16 KB slot q; a missing stage (partial last group) has code 0 and
            // a zero entry 0; the split's records: lo32 words, then the high bytes
            const uint32_t clo = uint32_t((nt * 4 + 15) & ~uint64_t(15)), chi = uint32_t((nt + 15) & ~uint64_t(15));
            ptx::mbar_arrive_expect_tx(bar, bytes + (kGroupStages - (s1 - s0)) * 16u + clo + chi);
            for (uint32_t s = s0; s < s0 + kGroupStages; ++s) {
                uint8_t* dst = lut_buf + b * 65536 + (s - s0) * 16384;
                if (s < s1)
                    ptx::bulk_g2s(ptx::smem_u32(dst), lutp + a.kst[s].eff_off / kD, a.kst[s].size * 16u, bar);
                else
                    ptx::bulk_g2s(ptx::smem_u32(dst), g_zero16, 16u, bar);
            }
            const uint8_t* seg = kc + uint64_t(grp) * a.gm_cap * 5;
            ptx::bulk_g2s(ptx::smem_u32(code_buf + b * kGmCodeBuf), seg + t0 * 4, clo, bar);
            ptx::bulk_g2s(ptx::smem_u32(code_buf + b * kGmCodeBuf + 4 * kSplitTokens), seg + a.gm_cap * 4 + t0, chi, bar);
        } else {
            ptx::mbar_arrive_expect_tx(bar, bytes);
            uint32_t off = 0;
            for (uint32_t s = s0; s < s1; ++s) {
                const uint32_t nb = a.kst[s].size * 16u;
                ptx::bulk_g2s(ptx::smem_u32(lut_buf + b * 65536 + off), lutp + a.kst[s].eff_off / kD, nb, bar);
                off += nb;
            }
        }
    };
    if (threadIdx.x == 0) issue(0);
    for (uint32_t grp = 0; grp < ngroups; ++grp) {
        if (threadIdx.x == 0 && grp + 1 < ngroups) issue(grp + 1);
        ptx::mbar_wait(ptx::smem_u32(&bars[grp & 1]), (grp >> 1) & 1);
        if constexpr (GM == 2) {
            const uint32_t Lb = ptx::smem_u32(lut_buf) + (grp & 1) * 65536u;
            const uint32_t* clo = reinterpret_cast<const uint32_t*>(code_buf + (grp & 1) * kGmCodeBuf);
            const uint8_t* chi = code_buf + (grp & 1) * kGmCodeBuf + 4 * kSplitTokens;
            uint32_t off[kGroupStages], msk[kGroupStages];
#pragma unroll
            for (int q = 0; q < kGroupStages; ++q) {
                const uint32_t st = grp * kGroupStages + q;
                off[q] = (st < a.kn) ? a.kst[st].bit_off - a.kst[grp * kGroupStages].bit_off : 0u;
                msk[q] = (st < a.kn) ? ((1u << a.kst[st].bits) - 1u) << 3 : 0u;
            }
#pragma unroll
            for (int k = 0; k < kTokPerThread; ++k) {
                const uint32_t lt = threadIdx.x + uint32_t(k) * kAttThreads;
                const uint32_t lo = clo[lt], hi = chi[lt];
                const uint32_t xl = lo << 3, xh = __funnelshift_l(lo, hi, 3);
                uint2 w[4];
                lds64(Lb | (xl & msk[0]), w[0]);
                lds64((Lb + 8192u) | (__funnelshift_r(xl, xh, off[1]) & msk[1]), w[1]);
                lds64((Lb + 16384u) | (__funnelshift_r(xl, xh, off[2]) & msk[2]), w[2]);
                lds64((Lb + 24576u) | (__funnelshift_r(xl, xh, off[3]) & msk[3]), w[3]);
                // per 32-bit word: the whole word and its high half accumulate; the low-half sum is
                // recovered exactly afterwards (full - (high << 16), mod 2^32: it stays below 2^22)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    il[k][0] += w[q].x;
                    il[k][1] += w[q].x >> 16;
                    il[k][2] += w[q].y;
                    il[k][3] += w[q].y >> 16;
                }
            }
            __syncthreads();  // buffers (grp & 1) are refilled two groups later
            continue;
        }
        if constexpr (GM == 1) {
            const uint32_t Lb = ptx::smem_u32(lut_buf) + (grp & 1) * 65536u;
            const uint32_t* clo = reinterpret_cast<const uint32_t*>(code_buf + (grp & 1) * kGmCodeBuf);
            const uint8_t* chi = code_buf + (grp & 1) * kGmCodeBuf + 4 * kSplitTokens;
            // field q of the record x = rec << 4 sits at bit off_q: (x >> off_q) & (mask_q << 4)
            uint32_t off[kGroupStages], msk[kGroupStages];
#pragma unroll
            for (int q = 0; q < kGroupStages; ++q) {
                const uint32_t s = grp * kGroupStages + q;
                off[q] = (s < a.kn) ? a.kst[s].bit_off - a.kst[grp * kGroupStages].bit_off : 0u;
                msk[q] = (s < a.kn) ? ((1u << a.kst[s].bits) - 1u) << 4 : 0u;
            }
#pragma unroll
            for (int k = 0; k < kTokPerThread; ++k) {
                // tokens past nt read stale records (valid slots; their logits are masked below)
                const uint32_t lt = threadIdx.x + uint32_t(k) * kAttThreads;
                const uint32_t lo = clo[lt], hi = chi[lt];
                const uint32_t xl = lo << 4, xh = __funnelshift_l(lo, hi, 4);
                float2 v[4][2];
                lds128(Lb | (xl & msk[0]), v[0][0], v[0][1]);
                lds128((Lb + 16384u) | (__funnelshift_r(xl, xh, off[1]) & msk[1]), v[1][0], v[1][1]);
                lds128((Lb + 32768u) | (__funnelshift_r(xl, xh, off[2]) & msk[2]), v[2][0], v[2][1]);
                lds128((Lb + 49152u) | (__funnelshift_r(xl, xh, off[3]) & msk[3]), v[3][0], v[3][1]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    lg2[k][0] = ptx::add2(lg2[k][0], v[q][0]);
                    lg2[k][1] = ptx::add2(lg2[k][1], v[q][1]);
                }
            }
            __syncthreads();  // buffers (grp & 1) are refilled two groups later
            continue;
        }
        const uint32_t s0 = grp * kGroupStages;
        const uint32_t s1 = min(a.kn, s0 + kGroupStages);
        const float4* L = reinterpret_cast<const float4*>(lut_buf + (grp & 1) * 65536);
        const uint32_t gbit = a.kst[s0].bit_off;
        uint32_t loff[kGroupStages], lbits[kGroupStages], lofs[kGroupStages];
        uint32_t acc_off = 0;
#pragma unroll
        for (int q = 0; q < kGroupStages; ++q) {
            const uint32_t s = s0 + q;
            lbits[q] = (s < s1) ? a.kst[s].bits : 0u;
            loff[q] = (s < s1) ? a.kst[s].bit_off - gbit : 0u;
            lofs[q] = acc_off;
            acc_off += (s < s1) ? a.kst[s].size : 0u;
        }
        // kKeyBatch tokens per batch: all their code-word loads are issued before any
        // is used (branch-free: out-of-range tokens and the last words of the buffer
        // read a dummy word; the rare buffer-tail tokens take read_bits64's careful path).
        // Bit positions are 32-bit, relative to the 8 B-aligned start of the pair's stream.
#pragma unroll
        for (int kb = 0; kb < kTokPerThread; kb += kKeyBatch) {
            uint2 lo[kKeyBatch], hi[kKeyBatch];
            uint32_t sh[kKeyBatch];
            bool fast[kKeyBatch];
#pragma unroll
            for (int k = 0; k < kKeyBatch; ++k) {
                const uint32_t t = threadIdx.x + uint32_t(kb + k) * kAttThreads;
                const uint32_t pos = (uint32_t(t0) + t) * krow32 + gbit + kbase_bits;
                const uint32_t wi = pos >> 6;
                sh[k] = pos & 63u;
                fast[k] = (t < nt) && (wi + 2u <= kwords);
                const uint2* q = reinterpret_cast<const uint2*>(fast[k] ? kc64 + wi : g_zero16);
                lo[k] = __ldg(q);
                hi[k] = __ldg(q + 1);
            }
#pragma unroll
            for (int k = 0; k < kKeyBatch; ++k) {
                const uint32_t t = threadIdx.x + uint32_t(kb + k) * kAttThreads;
                if (t < nt) {
                    // 64-bit window starting at bit sh of (lo, hi) as two 32-bit words
                    const bool low = sh[k] < 32u;
                    const uint32_t s5 = sh[k] & 31u;
                    const uint32_t wa = low ? lo[k].x : lo[k].y, wb = low ? lo[k].y : hi[k].x;
                    const uint32_t wc = low ? hi[k].x : hi[k].y;
                    uint32_t w0 = __funnelshift_r(wa, wb, s5), w1 = __funnelshift_r(wb, wc, s5);
                    if (!fast[k]) {
                        const uint64_t w = read_bits64(kc, (t0 + t) * a.krow_bits + gbit, a.kend);
                        w0 = uint32_t(w);
                        w1 = uint32_t(w >> 32);
                    }
#pragma unroll
                    for (int q = 0; q < kGroupStages; ++q) {
                        if (lbits[q]) {
                            const uint32_t z = (loff[q] < 32u ? __funnelshift_r(w0, w1, loff[q]) : (w1 >> (loff[q] - 32u))) &
                                               ((1u << lbits[q]) - 1u);
                            const float4 v = L[lofs[q] + z];
                            lg2[kb + k][0] = ptx::add2(lg2[kb + k][0], make_float2(v.x, v.y));
                            lg2[kb + k][1] = ptx::add2(lg2[kb + k][1], make_float2(v.z, v.w));
                        }
                    }
                }
            }
        }
        __syncthreads();  // buffer (grp & 1) is refilled two groups later
    }

    if constexpr (GM == 2) {
        const float* dqp = a.dq + uint64_t(pair) * kG;
        const int bias = int(a.kn) * 32768;
#pragma unroll
        for (int k = 0; k < kTokPerThread; ++k) {
            il[k][0] -= il[k][1] << 16;
            il[k][2] -= il[k][3] << 16;
        }
#pragma unroll
        for (int g = 0; g < kG; ++g) {
            const float d = __ldg(dqp + g);
#pragma unroll
            for (int k = 0; k < kTokPerThread; ++k) lg[k][g] = float(int(il[k][g]) - bias) * d;
        }
    }

    // ---- split max / p / l
    float mg[kG], lsum[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < kTokPerThread; ++k)
            if (threadIdx.x + uint64_t(k) * kAttThreads < nt) m = fmaxf(m, lg[k][g]);
        mg[g] = block_max(m, red);
    }
#pragma unroll
    for (int g = 0; g < kG; ++g) {
        float l = 0.f;
#pragma unroll
        for (int k = 0; k < kTokPerThread; ++k) {
            const bool ok = threadIdx.x + uint64_t(k) * kAttThreads < nt;
            const float p = ok ? __expf(lg[k][g] - mg[g]) : 0.f;
            lg[k][g] = p;
            l += p;
        }
        lsum[g] = block_sum(l, red);
    }

    // ---- values: int32 fixed-point histograms H[s][j][g] in smem (reuses the LUT area)
    uint32_t* H = reinterpret_cast<uint32_t*>(sm);
    const uint32_t hsz = uint32_t(a.ventries) * kG;
    // value-stage descriptors, read once per CTA: entry offset << 16 | bit offset
    // within the stage's 6-stage window << 5 | bits; window start bits per group
    uint32_t* vd = reinterpret_cast<uint32_t*>(sm + 131072 + 64 + 256);
    uint32_t* vgb = vd + kMaxVStages;
    for (uint32_t i = threadIdx.x; i < hsz; i += blockDim.x) H[i] = 0u;
    if (threadIdx.x < a.vn) {
        const StageInfo si = a.vst[threadIdx.x];
        const uint32_t first = (threadIdx.x / 6u) * 6u;
        vd[threadIdx.x] = uint32_t(si.eff_off / kD) << 16 | (si.bit_off - a.vst[first].bit_off) << 5 | si.bits;
        if (threadIdx.x == first) vgb[threadIdx.x / 6u] = si.bit_off;
    }
    __syncthreads();
    // Histogram updates of one token: its <= 6-field value-code windows, then one shared
    // atomic per (stage, head) with a nonzero weight.
    auto hist_token = [&](uint32_t t, const uint32_t (&P)[kG]) {
        const uint32_t rb = (uint32_t(t0) + t) * vrow32 + vbase_bits;
        // windows of the common case (<= 3, i.e. up to 18 value stages) load together
        uint32_t w0[3], w1[3];
        bool ok3 = nvwin <= 3u;
        if (ok3) {
#pragma unroll
            for (int wdw = 0; wdw < 3; ++wdw) {
                const uint32_t pos = rb + vgb[wdw < int(nvwin) ? wdw : 0];
                const uint32_t wi = pos >> 6;
                const bool f = wi + 2u <= vwords;
                ok3 = ok3 && (f || wdw >= int(nvwin));
                const uint2* q = reinterpret_cast<const uint2*>(f ? vc64 + wi : g_zero16);
                const uint2 lo = __ldg(q), hi = __ldg(q + 1);
                const uint32_t sh = pos & 63u, s5 = sh & 31u;
                const bool low = sh < 32u;
                const uint32_t wa = low ? lo.x : lo.y, wb = low ? lo.y : hi.x, wc = low ? hi.x : hi.y;
                w0[wdw] = __funnelshift_r(wa, wb, s5);
                w1[wdw] = __funnelshift_r(wb, wc, s5);
            }
        }
        for (uint32_t s0 = 0, wdw = 0; s0 < a.vn; s0 += 6, ++wdw) {
            uint32_t x0, x1;
            if (ok3) {
                x0 = wdw == 0 ? w0[0] : (wdw == 1 ? w0[1] : w0[2]);
                x1 = wdw == 0 ? w1[0] : (wdw == 1 ? w1[1] : w1[2]);
            } else {  // many value stages or the buffer tail: careful 64-bit reads
                const uint64_t w = read_bits64(vc, (t0 + t) * a.vrow_bits + vgb[wdw], a.vend);
                x0 = uint32_t(w);
                x1 = uint32_t(w >> 32);
            }
            const uint32_t s1 = min(a.vn, s0 + 6u);
            for (uint32_t st = s0; st < s1; ++st) {
                const uint32_t d = vd[st];
                const uint32_t lo5 = (d >> 5) & 63u;
                const uint32_t z = (lo5 < 32u ? __funnelshift_r(x0, x1, lo5) : (x1 >> (lo5 - 32u))) &
                                   ((1u << (d & 31u)) - 1u);
                uint32_t* h = H + ((d >> 16) + z) * kG;
#pragma unroll
                for (int g = 0; g < kG; ++g)
                    if (P[g]) atomicAdd(h + g, P[g]);
            }
        }
    };
    // Tokens whose weights all round to 0 in the 2^-18 fixed point add nothing; the others
    // are compacted into a per-warp queue and processed 32 at a time, so the histogram
    // loop runs with full warps instead of the few lanes that happen to contribute.
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t* qt = reinterpret_cast<uint32_t*>(sm + kQueueOff) + (threadIdx.x >> 5) * (kQueueCap * (1 + kG));
    uint32_t* qP = qt + kQueueCap;
    uint32_t qlen = 0;
    auto flush = [&](uint32_t n) {
        if (lane < n) {
            uint32_t P[kG];
#pragma unroll
            for (int g = 0; g < kG; ++g) P[g] = qP[lane * kG + g];
            hist_token(qt[lane], P);
        }
    };
#pragma unroll
    for (int k = 0; k < kTokPerThread; ++k) {
        const uint32_t t = threadIdx.x + uint32_t(k) * kAttThreads;
        uint32_t P[kG];
#pragma unroll
        for (int g = 0; g < kG; ++g) P[g] = __float2uint_rn(lg[k][g] * kHistScale);
        const bool act = t < nt && (P[0] | P[1] | P[2] | P[3]) != 0u;
        const uint32_t mask = __ballot_sync(0xffffffffu, act);
        if (act) {
            const uint32_t pos = qlen + __popc(mask & ((1u << lane) - 1u));
            qt[pos] = t;
#pragma unroll
            for (int g = 0; g < kG; ++g) qP[pos * kG + g] = P[g];
        }
        qlen += __popc(mask);
        if (qlen >= 32u) {
            __syncwarp();
            flush(32u);
            __syncwarp();
            if (lane + 32u < qlen) {  // keep the overflow for the next batch
                qt[lane] = qt[lane + 32u];
#pragma unroll
                for (int g = 0; g < kG; ++g) qP[lane * kG + g] = qP[(lane + 32u) * kG + g];
            }
            __syncwarp();
            qlen -= 32u;
        }
    }
    __syncwarp();
    flush(qlen);
    __syncthreads();
    float* ph = a.part_h + (uint64_t(pair) * a.n_splits + split) * hsz;
    for (uint32_t i = threadIdx.x; i < hsz; i += blockDim.x) ph[i] = float(H[i]) * (1.0f / kHistScale);
    if (threadIdx.x < kG) {
        a.part_m[(uint64_t(pair) * (a.n_splits + 1) + split) * kG + threadIdx.x] = mg[threadIdx.x];
        a.part_l[(uint64_t(pair) * (a.n_splits + 1) + split) * kG + threadIdx.x] = lsum[threadIdx.x];
    }
}

// Split weights: w[pair][s][g] = exp(m_s - M), L = sum_s w l_s, M = max_s m_s.
__global__ void lut_weights_kernel(const float* __restrict__ part_m, const float* __restrict__ part_l,
                                   uint32_t n_splits, uint32_t n_pairs, float* __restrict__ w, float* __restrict__ ML) {
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;  // pair * G + g
    if (idx >= n_pairs * kG) return;
    const uint32_t pair = idx / kG, g = idx % kG, ns = n_splits + 1;
    float M = -INFINITY;
    for (uint32_t s = 0; s < ns; ++s) M = fmaxf(M, part_m[(uint64_t(pair) * ns + s) * kG + g]);
    float L = 0.f;
    for (uint32_t s = 0; s < ns; ++s) {
        const float m = part_m[(uint64_t(pair) * ns + s) * kG + g];
        const float ww = (m > -INFINITY) ? __expf(m - M) : 0.f;
        w[(uint64_t(pair) * ns + s) * kG + g] = ww;
        L += ww * part_l[(uint64_t(pair) * ns + s) * kG + g];
    }
    ML[idx * 2] = M;
    ML[idx * 2 + 1] = L;
}

// CTA = (pair, 256-entry chunk of the value codebooks): merge the split
// histograms of the chunk, contract with the chunk's codebook rows and add the
// partial output into acc[pair][g][d] (fp32 atomics in L2).  Merge: every split's
// load is in flight at once.  Contraction: thread = (d, quarter of the chunk), one
// codebook load feeds the 4 heads.
__global__ void __launch_bounds__(512) lut_contract_kernel(const float* __restrict__ part_h, const float* __restrict__ w,
                                                           uint32_t n_splits, const float* __restrict__ veff,
                                                           uint64_t ventries, float* __restrict__ acc) {
    constexpr int kChunk = 256, kMerge = 16;
    __shared__ float4 hs[kChunk];
    __shared__ float4 po[4][kD];
    const uint32_t pair = blockIdx.y;
    const uint64_t e0 = uint64_t(blockIdx.x) * kChunk;
    const uint32_t ne = uint32_t((ventries - e0 < kChunk) ? (ventries - e0) : kChunk);
    const uint32_t ns = n_splits + 1;
    float* hsf = reinterpret_cast<float*>(hs);
    for (uint32_t i = threadIdx.x; i < kChunk * kG; i += blockDim.x) {
        const uint32_t e = i / kG, g = i % kG;
        float v = 0.f;
        if (e < ne) {
            const float* src = part_h + (uint64_t(pair) * n_splits * ventries + e0) * kG + i;
            const float* wp = w + uint64_t(pair) * ns * kG + g;
            for (uint32_t s0 = 0; s0 < n_splits; s0 += kMerge) {
                float x[kMerge];
#pragma unroll
                for (int k = 0; k < kMerge; ++k)
                    x[k] = (s0 + k < n_splits) ? __ldg(src + uint64_t(s0 + k) * ventries * kG) : 0.f;
#pragma unroll
                for (int k = 0; k < kMerge; ++k)
                    if (s0 + k < n_splits) v = fmaf(wp[(s0 + k) * kG], x[k], v);
            }
        }
        hsf[i] = v;
    }
    __syncthreads();
    const uint32_t d = threadIdx.x % kD, qt = threadIdx.x / kD;  // quarter qt: entries qt, qt + 4, ...
    float o[kG] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (uint32_t e = qt; e < ne; e += 4) {
        const float x = __ldg(veff + (e0 + e) * kD + d);
        const float4 h = hs[e];
        o[0] = fmaf(h.x, x, o[0]);
        o[1] = fmaf(h.y, x, o[1]);
        o[2] = fmaf(h.z, x, o[2]);
        o[3] = fmaf(h.w, x, o[3]);
    }
    po[qt][d] = make_float4(o[0], o[1], o[2], o[3]);
    __syncthreads();
    if (threadIdx.x < kG * kD) {
        const uint32_t g = threadIdx.x / kD, dd = threadIdx.x % kD;
        const float* pf = reinterpret_cast<const float*>(po);
        const float r = (pf[(0 * kD + dd) * kG + g] + pf[(1 * kD + dd) * kG + g]) +
                        (pf[(2 * kD + dd) * kG + g] + pf[(3 * kD + dd) * kG + g]);
        atomicAdd(acc + (uint64_t(pair) * kG + g) * kD + dd, r);
    }
}

// out = (acc + w_raw * o_raw) / L, lse = M + log L
__global__ void lut_finish_kernel(const float* __restrict__ acc, const float* __restrict__ part_o,
                                  const float* __restrict__ w, const float* __restrict__ ML, uint32_t n_splits,
                                  uint32_t n_pairs, float* __restrict__ out, float* __restrict__ lse) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // (pair, g, d)
    if (idx >= uint64_t(n_pairs) * kG * kD) return;
    const uint32_t pg = uint32_t(idx / kD), pair = pg / kG, g = pg % kG;
    const float wr = w[(uint64_t(pair) * (n_splits + 1) + n_splits) * kG + g];
    float v = acc[idx];
    if (wr > 0.f) v = fmaf(wr, part_o[idx], v);
    out[idx] = v / ML[pg * 2 + 1];
    if (idx % kD == 0 && lse) lse[pg] = ML[pg * 2] + logf(ML[pg * 2 + 1]);
}

}  // namespace

// tensor-core LUT build: D = 128 stacks carry the fp16 hi/lo operand chunks
static bool lut_tc_ok(const vqkv_stack_s& ks) {
    const char* e = getenv("VQKV_LUT_FFMA");
    if ((e && e[0] == '1') || ks.dim != kD || !ks.d_eff16 || !ks.d_eff16lo) return false;
    // E_hi = fp16(e) must be finite with headroom (the FFMA kernel covers larger entries)
    for (const auto& st : ks.stages)
        if (!(st.max_abs < 32768.f)) return false;
    return true;
}

bool attend_lut_supported(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a) {
    if (ks.dim != kD || vs.dim != kD || a.group != kG) return false;
    if (a.n_init + a.n_local > kSplitTokens) return false;
    // 32-bit bit positions inside one pair's key-code stream (+ alignment slack)
    if (uint64_t(a.n_comp) * ks.row_bits + 64 >= (1ull << 32)) return false;
    if (uint64_t(a.n_comp) * vs.row_bits + 64 >= (1ull << 32)) return false;
    for (const auto& s : ks.stages)
        if (s.size > 1024 || s.bits > 10) return false;
    // 4 key stages per 64-bit read and LUT group (<= 64 KB)
    for (uint32_t s0 = 0; s0 < ks.n; s0 += kGroupStages) {
        uint32_t bits = 0, bytes = 0;
        for (uint32_t s = s0; s < std::min(ks.n, s0 + kGroupStages); ++s) {
            bits += ks.stages[s].bits;
            bytes += ks.stages[s].size * 16u;
        }
        if (bits > 56 || bytes > 65536) return false;
    }
    uint32_t ventries = 0;
    for (uint32_t s0 = 0; s0 < vs.n; s0 += 6) {
        uint32_t bits = 0;
        for (uint32_t s = s0; s < std::min(vs.n, s0 + 6u); ++s) bits += vs.stages[s].bits;
        if (bits > 56) return false;
    }
    if (vs.n > uint32_t(kMaxVStages)) return false;
    for (const auto& s : vs.stages) ventries += s.size;
    if (ventries > 65535) return false;
    if (uint64_t(ventries) * kG * 4 > 131072) return false;
    return true;
}

// ---- group-major key codes ------------------------------------------------------------
// Per pair, per LUT group g (stages 4g..4g+3): a segment of cap 5-byte records, stored as
// cap little-endian u32 words (record bits 0-31) followed by cap bytes (bits 32-39).  A
// record holds the group's fields in stage order at their CodeMatrix offsets relative to
// the group's first field (codebook.cpp:96-120 row layout), missing stages as zeros.
__global__ void gm_pack_kernel(const uint8_t* __restrict__ payload, uint64_t payload_stride, uint64_t row_bits,
                               const uint8_t* payload_end, const uint32_t* __restrict__ gbit, const uint32_t* __restrict__ gwidth,
                               uint32_t n_groups, uint64_t src_row, uint64_t count, uint8_t* __restrict__ gm, uint64_t cap,
                               uint64_t gm_stride, uint64_t dst_row) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint32_t g = blockIdx.y, pair = blockIdx.z;
    if (t >= count) return;
    const uint8_t* src = payload + pair * payload_stride;
    const uint64_t w = read_bits64(src, (src_row + t) * row_bits + gbit[g], payload_end);
    const uint64_t rec = gwidth[g] >= 64 ? w : (w & ((1ull << gwidth[g]) - 1ull));
    uint8_t* seg = gm + pair * gm_stride + uint64_t(g) * cap * 5;
    reinterpret_cast<uint32_t*>(seg)[dst_row + t] = uint32_t(rec);
    seg[cap * 4 + dst_row + t] = uint8_t(rec >> 32);
}

bool gm_supported(const vqkv_stack_s& ks) {
    if (ks.dim != kD) return false;
    for (const auto& st : ks.stages)
        if (st.size > 1024 || st.bits > 10) return false;
    return true;
}

// int16 LUT (opt-in: VQKV_ATTEND_INT16=1): group-major codes, even key stage sizes (8 B entries
// keep every stage slot a multiple of 16 B for the bulk copies), at most 64 stages (exact int32 sums)
static bool int16_lut_ok(const vqkv_stack_s& ks) {
    const char* e = getenv("VQKV_ATTEND_INT16");
    if (!(e && e[0] == '1') || !gm_supported(ks) || ks.n > 64) return false;
    for (const auto& st : ks.stages)
        if (st.size & 1u) return false;
    return true;
}

uint64_t gm_pair_bytes(const vqkv_stack_s& ks, uint64_t cap) {
    return uint64_t((ks.n + kGroupStages - 1) / kGroupStages) * cap * 5;
}

void launch_keycodes_to_gm(const vqkv_stack_s& ks, const uint8_t* payload, uint64_t payload_stride, uint32_t n_pairs,
                           uint64_t src_row, uint64_t count, uint8_t* gm, uint64_t cap, uint64_t gm_stride,
                           uint64_t dst_row, cudaStream_t s) {
    const uint32_t ng = (ks.n + kGroupStages - 1) / kGroupStages;
    std::vector<uint32_t> h(2 * ng);
    for (uint32_t g = 0; g < ng; ++g) {
        const uint32_t s0 = g * kGroupStages, s1 = std::min(ks.n, s0 + kGroupStages);
        h[g] = ks.stages[s0].bit_off;
        h[ng + g] = ks.stages[s1 - 1].bit_off + ks.stages[s1 - 1].bits - ks.stages[s0].bit_off;
    }
    uint32_t* d = nullptr;
    VQKV_CUDA(cudaMallocAsync(&d, sizeof(uint32_t) * 2 * ng, s));
    VQKV_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(uint32_t) * 2 * ng, cudaMemcpyHostToDevice, s));
    const uint64_t pb = payload_bytes(ks.row_bits, src_row + count);
    const uint8_t* end = payload + uint64_t(n_pairs - 1) * payload_stride + pb;
    dim3 grid(unsigned((count + 255) / 256), ng, n_pairs);
    gm_pack_kernel<<<grid, 256, 0, s>>>(payload, payload_stride, ks.row_bits, end, d, d + ng, ng, src_row, count, gm, cap,
                                        gm_stride, dst_row);
    launch_check("gm_pack_kernel");
    VQKV_CUDA(cudaFreeAsync(d, s));
}

void launch_attend_lut(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a, cudaStream_t s) {
    const uint64_t kent = ks.total_rows, vent = vs.total_rows;
    const uint32_t n_splits = uint32_t((a.n_comp + kSplitTokens - 1) / kSplitTokens);
    const double scale = a.scale > 0.0 ? a.scale : 1.0 / std::sqrt(double(kD));
    float4* lut = nullptr;
    float *ph = nullptr, *po = nullptr, *pm = nullptr, *pl = nullptr;
    const bool i16 = a.kcodes_layout == VQKV_KEYCODES_GROUP_MAJOR && int16_lut_ok(ks);
    uint2* lut16 = nullptr;
    float* dq = nullptr;
    VQKV_CUDA(cudaMallocAsync(&lut, sizeof(float4) * a.n_pairs * kent, s));
    VQKV_CUDA(cudaMallocAsync(&ph, sizeof(float) * std::max<uint64_t>(1, uint64_t(a.n_pairs) * n_splits * vent * kG), s));
    VQKV_CUDA(cudaMallocAsync(&po, sizeof(float) * a.n_pairs * kG * kD, s));
    VQKV_CUDA(cudaMallocAsync(&pm, sizeof(float) * a.n_pairs * (n_splits + 1) * kG, s));
    VQKV_CUDA(cudaMallocAsync(&pl, sizeof(float) * a.n_pairs * (n_splits + 1) * kG, s));
    {
        ProfScope ps("attend_lut_build", s);
        if (lut_tc_ok(ks)) {
            // tensor-core LUT GEMM (VQKV_LUT_FFMA=1 selects the FFMA kernel below)
            const uint32_t rows = a.n_pairs * kG, rows_pad = (rows + 127) / 128 * 128, qt = rows_pad / 128;
            __half *qh = nullptr, *ql = nullptr;
            float* qs = nullptr;
            VQKV_CUDA(cudaMallocAsync(&qh, sizeof(__half) * rows_pad * kD, s));
            VQKV_CUDA(cudaMallocAsync(&ql, sizeof(__half) * rows_pad * kD, s));
            VQKV_CUDA(cudaMallocAsync(&qs, sizeof(float) * rows_pad, s));
            q_prep_kernel<<<rows_pad / 8, 256, 0, s>>>(a.q_dev, rows, rows_pad, float(scale), qh, ql, qs);
            launch_check("q_prep_kernel");
            VQKV_CUDA(cudaFuncSetAttribute(lut_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLutTcSmem)));
            uint32_t maxch = 0;
            for (const auto& st : ks.stages) maxch = std::max(maxch, (st.size + 127) / 128);
            lut_tc_kernel<<<dim3(maxch, ks.n), 160, kLutTcSmem, s>>>(ks.d_eff16, ks.d_eff16lo, ks.d_stages, qh, ql, qs,
                                                                    a.n_pairs, qt, kent, lut);
            launch_check("lut_tc_kernel");
            VQKV_CUDA(cudaFreeAsync(qh, s));
            VQKV_CUDA(cudaFreeAsync(ql, s));
            VQKV_CUDA(cudaFreeAsync(qs, s));
        } else {
        LutArgs la{a.q_dev, ks.d_eff, ks.d_stages, ks.n, kent, float(scale), lut};
        dim3 grid(unsigned((kent + kLutEntries - 1) / kLutEntries), (a.n_pairs + 7) / 8);
        const int lsmem = int(sizeof(float) * (8 * kG * kD + kLutEntries * kLutStride));
        VQKV_CUDA(cudaFuncSetAttribute(lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem));
        lut_kernel<<<grid, 256, lsmem, s>>>(la, a.n_pairs);
        launch_check("lut_kernel");
        }
        if (i16) {
            VQKV_CUDA(cudaMallocAsync(&lut16, sizeof(uint2) * a.n_pairs * kent, s));
            VQKV_CUDA(cudaMallocAsync(&dq, sizeof(float) * a.n_pairs * kG, s));
            lut_int16_kernel<<<a.n_pairs, 1024, 0, s>>>(lut, kent, lut16, dq);
            launch_check("lut_int16_kernel");
        }
    }
    {
        ProfScope ps("attend", s);
        const uint64_t kpb = payload_bytes(ks.row_bits, a.n_comp), vpb = payload_bytes(vs.row_bits, a.n_comp);
        const uint64_t kstr = a.kcodes_stride ? a.kcodes_stride : kpb, vstr = a.vcodes_stride ? a.vcodes_stride : vpb;
        MainArgs ma{a.q_dev, a.init_k_dev, a.init_v_dev, a.n_init, a.kcodes_dev, a.vcodes_dev, a.n_comp,
                    a.local_k_dev, a.local_v_dev, a.n_local, ks.d_stages, ks.n, ks.row_bits, kstr, kent,
                    vs.d_stages, vs.n, vs.row_bits, vstr, vent, lut,
                    // end of the last pair's payload: reads stop here (earlier pairs may read into the next)
                    a.kcodes_dev + uint64_t(a.n_pairs - 1) * kstr + kpb,
                    a.vcodes_dev + uint64_t(a.n_pairs - 1) * vstr + vpb, float(scale), n_splits,
                    ph, po, pm, pl, a.init_stride ? a.init_stride : a.n_init,
                    a.local_stride ? a.local_stride : a.n_local, a.kcodes_cap, lut16, dq};
        {  // per launch (per-device attribute)
            VQKV_CUDA(cudaFuncSetAttribute(attend_lut_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kMainSmem + kAlignSlack)));
            VQKV_CUDA(cudaFuncSetAttribute(attend_lut_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kGmSmem + kAlignSlack)));
            VQKV_CUDA(cudaFuncSetAttribute(attend_lut_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kGmSmem + kAlignSlack)));
        }
        dim3 grid(n_splits + 1, a.n_pairs);
        if (i16)
            attend_lut_kernel<2><<<grid, kAttThreads, kGmSmem + kAlignSlack, s>>>(ma);
        else if (a.kcodes_layout == VQKV_KEYCODES_GROUP_MAJOR)
            attend_lut_kernel<1><<<grid, kAttThreads, kGmSmem + kAlignSlack, s>>>(ma);
        else
            attend_lut_kernel<0><<<grid, kAttThreads, kMainSmem + kAlignSlack, s>>>(ma);
        launch_check("attend_lut_kernel");
    }
    {
        ProfScope ps("attend_combine", s);
        float *w = nullptr, *ML = nullptr, *acc = nullptr;
        VQKV_CUDA(cudaMallocAsync(&w, sizeof(float) * a.n_pairs * (n_splits + 1) * kG, s));
        VQKV_CUDA(cudaMallocAsync(&ML, sizeof(float) * a.n_pairs * kG * 2, s));
        VQKV_CUDA(cudaMallocAsync(&acc, sizeof(float) * a.n_pairs * kG * kD, s));
        VQKV_CUDA(cudaMemsetAsync(acc, 0, sizeof(float) * a.n_pairs * kG * kD, s));
        lut_weights_kernel<<<(a.n_pairs * kG + 127) / 128, 128, 0, s>>>(pm, pl, n_splits, a.n_pairs, w, ML);
        launch_check("lut_weights_kernel");
        if (n_splits > 0) {
            dim3 g2(unsigned((vent + 255) / 256), a.n_pairs);
            lut_contract_kernel<<<g2, 512, 0, s>>>(ph, w, n_splits, vs.d_eff, vent, acc);
            launch_check("lut_contract_kernel");
        }
        const uint64_t n = uint64_t(a.n_pairs) * kG * kD;
        lut_finish_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(acc, po, w, ML, n_splits, a.n_pairs, a.out_dev,
                                                                   a.lse_dev);
        launch_check("lut_finish_kernel");
        VQKV_CUDA(cudaFreeAsync(w, s));
        VQKV_CUDA(cudaFreeAsync(ML, s));
        VQKV_CUDA(cudaFreeAsync(acc, s));
    }
    VQKV_CUDA(cudaFreeAsync(lut, s));
    if (i16) {
        VQKV_CUDA(cudaFreeAsync(lut16, s));
        VQKV_CUDA(cudaFreeAsync(dq, s));
    }
    VQKV_CUDA(cudaFreeAsync(ph, s));
    VQKV_CUDA(cudaFreeAsync(po, s));
    VQKV_CUDA(cudaFreeAsync(pm, s));
    VQKV_CUDA(cudaFreeAsync(pl, s));
}

}  // namespace vqkv_dev
