// attend_lut.cu -- K3: decode-step attention over the compressed cache in the
// dot-product domain (D = 128, G = 4 query heads per KV head).
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
// Layouts (all per (sequence, KV head) pair):
//   LUT      fp32, key stages in groups of 8: [group][j < R][slot 8][head 4] -- one
//            128 B row per code value j holds the 8 stages' float4 entries.
//   key codes ("attention records", vqkv_keycodes_to_gm): per group of 8 key stages
//            and token t an 80-bit record of eight 10-bit fields, ROTATED: field k
//            holds the code of stage slot (t & 7) ^ k.  Stored as two planes per group,
//            cap x u64 (record bits 0-63) then cap x u16 (bits 64-79): 10 B per token
//            and group, the CodeMatrix row's 70 B at the paper geometry.
//   value codes: the reference CodeMatrix rows (codebook.cpp:74-151), unchanged.
//
// Why the rotation: the lanes of a warp hold consecutive tokens, so in one LDS.128
// the 8 lanes of a quarter-warp read slots (lane & 7) ^ k -- 8 distinct 16 B bank
// groups of the 128 B rows whatever the codes are.  Every key lookup is a
// conflict-free wavefront (the round-1 layout lost 56 % of its wavefronts to bank
// conflicts of random LDS.128 gathers).
//
// Kernels (one launch each, on the caller's stream):
//   q_prep + lut_tc  the LUT GEMM on tcgen05 (split fp16, fp32 accumulate) -> fp32 LUT
//   attend_atr       CTA = (pair, contiguous token range), 512 threads, chunks of 8192
//                    tokens (16 per thread, logits in registers):
//                      keys   - per LUT group: one 128 KB bulk copy (TMA engine) of the
//                               group's rows into smem; per token 8 x (SHF, LOP3,
//                               LDS.128, 2 FADD2) from the thread's 10 B record;
//                      softmax- chunk max m_c, p = exp(l - m_c), l_c = sum p (fp32);
//                      values - p in fixed point with quantum u_c = l_c 2^-28 (a
//                               RELATIVE quantum: see the bound below); per token with a
//                               nonzero weight the warp updates the 16 stages x 4 heads
//                               of int32 smem histograms, lane = (stage slot, head), so
//                               each ATOMS hits 32 distinct banks;
//                      fold   - H into the CTA's fp32 accumulator (global, L2-resident)
//                               rescaled to the running max (online softmax);
//                    after the last chunk the CTA contracts its accumulator with the
//                    value codebooks (o = sum H e) and writes (o, m, l).
//                    One more CTA per pair attends the raw init/local rows directly.
//   combine          per pair: LSE merge of its CTAs' partials, normalise, emit lse.
//
// Value-path error bound (rigorous).  In a chunk of n_c <= 8192 tokens the histogram
// rounds each p_t to a multiple of u_c = l_c 2^-28 (round to nearest, |err| <= u_c/2;
// tokens below u_c/2 round to 0 and are skipped).  The normaliser uses the exact fp32
// l.  With chunk weights exp(m_c - M) and L = sum_c l_c exp(m_c - M):
//     |o' - o|_inf <= sum_c n_c (u_c/2) exp(m_c - M) max_t|v_t|_inf / L
//                  <= 8192 * 2^-29 * max_t|v_t|_inf = 2^-16 max_t|v_t|_inf,
// independent of how flat or peaked the attention is (no absolute cut).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "tc_ptx.cuh"
#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

constexpr int kG = 4;                          // query heads per KV head on this path
constexpr int kD = 128;                        // head dim
constexpr int kThreads = 512;
#ifndef VQKV_ATTN_KB
#define VQKV_ATTN_KB 2  // key records loaded per batch, one batch ahead of the lookups
#endif
#ifndef VQKV_ATTN_HANDOFF
#define VQKV_ATTN_HANDOFF 1  // pairs split between two CTAs are contracted once (accumulator hand-off)
#endif
#ifndef VQKV_ATTN_TOK
#define VQKV_ATTN_TOK 16
#endif
constexpr int kTok = VQKV_ATTN_TOK;            // tokens per thread per chunk
constexpr int kChunk = kThreads * kTok;        // 8192 tokens per chunk
constexpr int kGS = 8;                         // key stages per LUT group (one 128 B row)
constexpr uint32_t kRowBytes = kGS * 16;       // 8 slots x float4
constexpr uint32_t kLutBytes = 1024 * kRowBytes;  // 128 KB: one group, up to 1024 code values
constexpr uint32_t kMaxVStages = 64;
constexpr uint32_t kSmemCtl = 2048;            // barrier, TMEM address, reductions, value descriptors
constexpr uint32_t kQueueCap = 32 + 32 * 4;    // per-warp queue of (token, head) entries with a nonzero weight
constexpr uint32_t kQueueBytes = (kThreads / 32) * kQueueCap * 8;
constexpr uint32_t kSlabTok = 4 * kThreads;      // value rows staged per slab (4 tokens per thread)
constexpr uint32_t kSlabBytes = 38400;           // per slab buffer: rows of up to 149 bits + alignment slack
constexpr uint32_t kMaxSlabRowBits = ((kSlabBytes - 48) * 8) / kSlabTok;
constexpr uint32_t kMainSmem = kLutBytes + kSmemCtl + kQueueBytes + 2 * kSlabBytes;
constexpr float kQuantum = 268435456.0f;       // 2^28: p / u_c = p * 2^28 / l_c

// LUT element offset (in float4) of (pair, stage s, code j)
__host__ __device__ __forceinline__ uint64_t lut_off(uint64_t pair, uint32_t ng, uint32_t R, uint32_t s, uint32_t j) {
    return ((pair * ng + (s >> 3)) * R + j) * kGS + (s & 7u);
}

struct LutArgs {
    const float* q;        // [pairs][G][D]
    const float* keff;     // key effective entries
    const StageInfo* kst;
    uint32_t kn;
    uint64_t kentries;     // total key entries (sum S)
    float scale;
    float4* lut;           // grouped layout (lut_off)
    uint32_t ng, R;
};

// FFMA fallback of the LUT build (entries too large for the fp16 split operands).
// CTA: 128 entries (stage-concatenated) x 8 pairs, 256 threads; thread = 4 entries x 4 queries.
constexpr int kLutEntries = 128;
constexpr int kLutStride = kD + 2;  // even row stride: 8 B-aligned float2 reads
__global__ void __launch_bounds__(256) lut_kernel(LutArgs a, uint32_t n_pairs) {
    extern __shared__ float lsm[];
    float4* qs = reinterpret_cast<float4*>(lsm);  // [8 pairs][D] x float4 over g
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
        const float4 q0 = qp[c], q1 = qp[c + 1];
        float2 ev[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) ev[i] = *reinterpret_cast<const float2*>(es + (eg + 32 * i) * kLutStride + c);
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
            if (e < a.kentries) {
                uint32_t s = 0;  // stage of entry e (stages are few; scan)
                while (s + 1 < a.kn && e >= uint32_t(a.kst[s + 1].eff_off / kD)) ++s;
                const uint32_t j = e - uint32_t(a.kst[s].eff_off / kD);
                a.lut[lut_off(p0 + p, a.ng, a.R, s, j)] = make_float4(acc[i][0] * a.scale, acc[i][1] * a.scale,
                                                                      acc[i][2] * a.scale, acc[i][3] * a.scale);
            }
        }
}

// slots of a partial last group (stages that do not exist) are read with code 0: zero row 0
__global__ void lut_zero_missing_kernel(float4* lut, uint32_t ng, uint32_t R, uint32_t kn) {
    const uint32_t pair = blockIdx.x, slot = threadIdx.x;
    const uint32_t s = (ng - 1) * kGS + slot;
    if (slot < kGS && s >= kn) lut[lut_off(pair, ng, R, s, 0)] = make_float4(0.f, 0.f, 0.f, 0.f);
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
                                                     uint32_t n_pairs, uint32_t n_qtiles, uint32_t ng, uint32_t R,
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
        __shared__ __align__(16) float sc_s[2][128];     // the q-tile's row scales (one load per thread)
        for (uint32_t tq = 0; tq < n_qtiles; ++tq) {
            const uint32_t b = tq & 1, use = tq >> 1;
            sc_s[b][threadIdx.x] = qscl[uint64_t(tq) * 128 + threadIdx.x];
            asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps: scales in, tile tq - 2's reads done
            ptx::mbar_wait(ptx::smem_u32(&bar_mma[b]), use & 1);
            ptx::tc_fence_after();
            const float* sclp = sc_s[b];
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
                        const float4 sc = reinterpret_cast<const float4*>(sclp)[c4 * 8 + pp];
                        lut[lut_off(pair, ng, R, blockIdx.y, j)] = (
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

// Persistent, query-tile stationary LUT GEMM (the default; lut_tc_kernel above is the per-chunk
// version).  CTA = (query tile tq, replica r of cpq): it keeps its 128 (pair, g) query rows (Q_hi /
// Q_lo, 64 KB) in shared memory and streams the key chunks (s, c) = items r, r + cpq, ... through a
// two-slot ring (E_hi / E_lo, 64 KB per slot) by bulk copy; 24 MMAs per item into one of two TMEM
// accumulators while warps 0-3 drain the other.  One wave over the SMs instead of one CTA per
// (stage, chunk), and the query tile is read once per CTA instead of once per chunk.
constexpr uint32_t kLutTc2Smem = 6 * 32768 + 1024;
constexpr uint32_t kLutTc2MaxStages = 128;
// (register budget for 3 x 192 threads: leaves room for a raw-row CTA of the side stream on the SM)
__global__ void __launch_bounds__(192, 3) lut_tc2_kernel(const __half* __restrict__ eff16, const __half* __restrict__ eff16lo,
                                                          const StageInfo* __restrict__ kst, uint32_t n_stages,
                                                          const __half* __restrict__ qhi, const __half* __restrict__ qlo,
                                                          const float* __restrict__ qscl, uint32_t n_pairs, uint32_t cpq,
                                                          uint32_t ng, uint32_t R, float4* __restrict__ lut) {
    extern __shared__ uint8_t lsm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_q, e_full[2], e_empty[2], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base;
    __shared__ uint32_t pre[kLutTc2MaxStages + 1];  // chunk prefix over the stages
    __shared__ __align__(16) float sc_s[128];        // the query tile's row scales
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tq = blockIdx.x / cpq, rep = blockIdx.x % cpq;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar_q), 1);
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(ptx::smem_u32(&e_full[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&e_empty[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&acc_full[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&acc_empty[b]), 128);
        }
        ptx::fence_mbar_init();
        uint32_t acc = 0;
        for (uint32_t st = 0; st < n_stages; ++st) {
            pre[st] = acc;
            acc += (kst[st].size + 127u) / 128u;
        }
        pre[n_stages] = acc;
    }
    if (threadIdx.x < 128) sc_s[threadIdx.x] = qscl[uint64_t(tq) * 128 + threadIdx.x];
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 256);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t n_items = pre[n_stages];
    const uint32_t s_q = ptx::smem_u32(sm);  // Q_hi, Q_lo at + 32 KB
    auto s_e = [&](uint32_t b) { return s_q + 65536u + b * 65536u; };  // E_hi, E_lo at + 32 KB
    // item -> (stage, chunk): the stage whose chunk range holds it
    auto item_sc = [&](uint32_t it, uint32_t& st, uint32_t& c) {
        uint32_t lo = 0, hi = n_stages - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= it) lo = mid; else hi = mid - 1;
        }
        st = lo;
        c = it - pre[lo];
    };
    if (warp == 4) {
        if (lane == 0) {  // producer: the query tile once, then the key chunks
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar_q), 65536);
            ptx::bulk_g2s(s_q, qhi + uint64_t(tq) * 16384, 32768, ptx::smem_u32(&bar_q));
            ptx::bulk_g2s(s_q + 32768, qlo + uint64_t(tq) * 16384, 32768, ptx::smem_u32(&bar_q));
            uint32_t k = 0;
            for (uint32_t it = rep; it < n_items; it += cpq, ++k) {
                const uint32_t b = k & 1u, u = k >> 1;
                ptx::mbar_wait(ptx::smem_u32(&e_empty[b]), (u & 1u) ^ 1u);
                uint32_t st, c;
                item_sc(it, st, c);
                const uint64_t eo = kst[st].eff16_off + uint64_t(c) * 18432;
                ptx::mbar_arrive_expect_tx(ptx::smem_u32(&e_full[b]), 65536);
                ptx::bulk_g2s(s_e(b), eff16 + eo, 32768, ptx::smem_u32(&e_full[b]));
                ptx::bulk_g2s(s_e(b) + 32768, eff16lo + eo, 32768, ptx::smem_u32(&e_full[b]));
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = ptx::idesc_f16_f32(128, 128);
            ptx::mbar_wait(ptx::smem_u32(&bar_q), 0);
            uint32_t k = 0;
            for (uint32_t it = rep; it < n_items; it += cpq, ++k) {
                const uint32_t b = k & 1u, u = k >> 1;
                ptx::mbar_wait(ptx::smem_u32(&e_full[b]), u & 1u);
                ptx::mbar_wait(ptx::smem_u32(&acc_empty[b]), (u & 1u) ^ 1u);
                ptx::tc_fence_after();
                const uint32_t eh = s_e(b), el = eh + 32768, qh = s_q, ql = s_q + 32768;
                const uint32_t A[3] = {eh, el, eh}, B[3] = {ql, qh, qh};  // small terms first
#pragma unroll
                for (int part = 0; part < 3; ++part)
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t koff = (kk >> 2) * 16384 + (kk & 3) * 32;
                        ptx::mma_f16_ss(tmem + 128u * b, ptx::umma_desc_sw128(A[part] + koff),
                                        ptx::umma_desc_sw128(B[part] + koff), idesc, (part | kk) ? 1u : 0u);
                    }
                ptx::mma_commit(ptx::smem_u32(&acc_full[b]));
                ptx::mma_commit(ptx::smem_u32(&e_empty[b]));
            }
        }
    } else {
        // epilogue: thread = entry row of the chunk = TMEM lane; 32 pairs' float4 per item
        uint32_t k = 0;
        for (uint32_t it = rep; it < n_items; it += cpq, ++k) {
            const uint32_t b = k & 1u, u = k >> 1;
            uint32_t st, c;
            item_sc(it, st, c);
            const uint32_t size = kst[st].size, j = c * 128u + warp * 32u + lane;
            ptx::mbar_wait(ptx::smem_u32(&acc_full[b]), u & 1u);
            ptx::tc_fence_after();
            // two halves of 64 columns (16 pairs each): fewer live registers
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
                float v[2][32];
#pragma unroll
                for (int c4 = 0; c4 < 2; ++c4)
                    ptx::tmem_ld32(tmem + ((warp * 32u) << 16) + 128u * b + 64u * hh + 32u * c4, v[c4]);
                ptx::tc_wait_ld();
                if (hh == 1) {
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(ptx::smem_u32(&acc_empty[b]));
                }
#pragma unroll
                for (int c4 = 0; c4 < 2; ++c4)
#pragma unroll
                    for (int pp = 0; pp < 8; ++pp) {
                        const uint32_t pair = tq * 32 + (2 * hh + c4) * 8 + pp;
                        if (j < size && pair < n_pairs) {
                            const float4 sc = reinterpret_cast<const float4*>(sc_s)[(2 * hh + c4) * 8 + pp];
                            lut[lut_off(pair, ng, R, st, j)] =
                                make_float4(v[c4][4 * pp] * sc.x, v[c4][4 * pp + 1] * sc.y, v[c4][4 * pp + 2] * sc.z,
                                            v[c4][4 * pp + 3] * sc.w);
                        }
                    }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}

// LUT GEMM over stage pairs (the default): like lut_tc2_kernel (persistent, query-tile stationary), but
// an item is (stage pair sp, chunk c): stages 2 sp and 2 sp + 1 accumulate into the two halves of a
// 256-column TMEM buffer (double-buffered per item), so each (pair, code) gets its two adjacent LUT slots
// as one 32-byte store -- a full L2 sector, half the store instructions of one 16 B store per stage.
__global__ void __launch_bounds__(192, 3) lut_tc4_kernel(const __half* __restrict__ eff16, const __half* __restrict__ eff16lo,
                                                          const StageInfo* __restrict__ kst, uint32_t n_stages,
                                                          const __half* __restrict__ qhi, const __half* __restrict__ qlo,
                                                          const float* __restrict__ qscl, uint32_t n_pairs, uint32_t cpq,
                                                          uint32_t maxch, uint32_t ng, uint32_t R, float4* __restrict__ lut) {
    extern __shared__ uint8_t lsm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(lsm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar_q, e_full[2], e_empty[2], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(16) float sc_s[128];  // the query tile's row scales
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tq = blockIdx.x / cpq, rep = blockIdx.x % cpq;
    const uint32_t nsp = (n_stages + 1) / 2, n_items = nsp * maxch;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar_q), 1);
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(ptx::smem_u32(&e_full[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&e_empty[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&acc_full[b]), 1);
            ptx::mbar_init(ptx::smem_u32(&acc_empty[b]), 128);
        }
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 128) sc_s[threadIdx.x] = qscl[uint64_t(tq) * 128 + threadIdx.x];
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(&tmem_base), 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t s_q = ptx::smem_u32(sm);  // Q_hi, Q_lo at + 32 KB
    auto s_e = [&](uint32_t b) { return s_q + 65536u + b * 65536u; };  // E_hi, E_lo at + 32 KB
    auto has = [&](uint32_t st, uint32_t c) { return st < n_stages && c * 128u < kst[st].size; };
    if (warp == 4) {
        if (lane == 0) {  // producer: the query tile once, then per item the (up to) two stages' chunks
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar_q), 65536);
            ptx::bulk_g2s(s_q, qhi + uint64_t(tq) * 16384, 32768, ptx::smem_u32(&bar_q));
            ptx::bulk_g2s(s_q + 32768, qlo + uint64_t(tq) * 16384, 32768, ptx::smem_u32(&bar_q));
            uint32_t k = 0;  // ring steps
            for (uint32_t it = rep; it < n_items; it += cpq) {
                const uint32_t sp = it / maxch, c = it % maxch;
                for (uint32_t h = 0; h < 2; ++h) {
                    const uint32_t st = 2 * sp + h;
                    if (!has(st, c)) continue;
                    const uint32_t b = k & 1u, u = k >> 1;
                    ptx::mbar_wait(ptx::smem_u32(&e_empty[b]), (u & 1u) ^ 1u);
                    const uint64_t eo = kst[st].eff16_off + uint64_t(c) * 18432;
                    ptx::mbar_arrive_expect_tx(ptx::smem_u32(&e_full[b]), 65536);
                    ptx::bulk_g2s(s_e(b), eff16 + eo, 32768, ptx::smem_u32(&e_full[b]));
                    ptx::bulk_g2s(s_e(b) + 32768, eff16lo + eo, 32768, ptx::smem_u32(&e_full[b]));
                    ++k;
                }
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {  // MMA issuer
            constexpr uint32_t idesc = ptx::idesc_f16_f32(128, 128);
            ptx::mbar_wait(ptx::smem_u32(&bar_q), 0);
            uint32_t k = 0, ki = 0;
            for (uint32_t it = rep; it < n_items; it += cpq, ++ki) {
                const uint32_t sp = it / maxch, c = it % maxch;
                const uint32_t ab = ki & 1u, au = ki >> 1;
                ptx::mbar_wait(ptx::smem_u32(&acc_empty[ab]), (au & 1u) ^ 1u);
                ptx::tc_fence_after();
                for (uint32_t h = 0; h < 2; ++h) {
                    const uint32_t st = 2 * sp + h;
                    if (!has(st, c)) continue;
                    const uint32_t b = k & 1u, u = k >> 1;
                    ptx::mbar_wait(ptx::smem_u32(&e_full[b]), u & 1u);
                    ptx::tc_fence_after();
                    const uint32_t eh = s_e(b), el = eh + 32768, qh = s_q, ql = s_q + 32768;
                    const uint32_t A[3] = {eh, el, eh}, B[3] = {ql, qh, qh};  // small terms first
#pragma unroll
                    for (int part = 0; part < 3; ++part)
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint32_t koff = (kk >> 2) * 16384 + (kk & 3) * 32;
                            ptx::mma_f16_ss(tmem + 256u * ab + 128u * h, ptx::umma_desc_sw128(A[part] + koff),
                                            ptx::umma_desc_sw128(B[part] + koff), idesc, (part | kk) ? 1u : 0u);
                        }
                    ptx::mma_commit(ptx::smem_u32(&e_empty[b]));
                    ++k;
                }
                ptx::mma_commit(ptx::smem_u32(&acc_full[ab]));
            }
        }
    } else {
        // epilogue: thread = entry row j (TMEM lane); per pair the two stages' 4 heads = one 32 B store
        uint32_t ki = 0;
        for (uint32_t it = rep; it < n_items; it += cpq, ++ki) {
            const uint32_t sp = it / maxch, c = it % maxch;
            const uint32_t ab = ki & 1u, au = ki >> 1;
            const uint32_t j = c * 128u + warp * 32u + lane;
            const bool v0 = has(2 * sp, c) && j < kst[2 * sp].size;
            const bool v1 = has(2 * sp + 1, c) && j < kst[2 * sp + 1].size;
            ptx::mbar_wait(ptx::smem_u32(&acc_full[ab]), au & 1u);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem + ((warp * 32u) << 16) + 256u * ab;
#pragma unroll 1
            for (uint32_t q8 = 0; q8 < 4; ++q8) {  // 8 pairs (32 columns) per step
                float x0[32], x1[32];
                ptx::tmem_ld32(tbase + 32u * q8, x0);
                ptx::tmem_ld32(tbase + 128u + 32u * q8, x1);
                ptx::tc_wait_ld();
                if (q8 == 3) {
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(ptx::smem_u32(&acc_empty[ab]));
                }
                if (!(v0 || v1)) continue;
#pragma unroll
                for (int pp = 0; pp < 8; ++pp) {
                    const uint32_t pair = tq * 32 + q8 * 8 + pp;
                    if (pair < n_pairs) {
                        const float4 sc = reinterpret_cast<const float4*>(sc_s)[q8 * 8 + pp];
                        float o[8];
                        o[0] = v0 ? x0[4 * pp] * sc.x : 0.f;
                        o[1] = v0 ? x0[4 * pp + 1] * sc.y : 0.f;
                        o[2] = v0 ? x0[4 * pp + 2] * sc.z : 0.f;
                        o[3] = v0 ? x0[4 * pp + 3] * sc.w : 0.f;
                        o[4] = v1 ? x1[4 * pp] * sc.x : 0.f;
                        o[5] = v1 ? x1[4 * pp + 1] * sc.y : 0.f;
                        o[6] = v1 ? x1[4 * pp + 2] * sc.z : 0.f;
                        o[7] = v1 ? x1[4 * pp + 3] * sc.w : 0.f;
                        ptx::stg256(lut + lut_off(pair, ng, R, 2 * sp, j), o);
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
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


// block-wide max / sum of 4 values per thread (one barrier pair for the 4 heads)
__device__ __forceinline__ float4 block_max4(float4 v, float4* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x = fmaxf(v.x, __shfl_xor_sync(0xffffffffu, v.x, o));
        v.y = fmaxf(v.y, __shfl_xor_sync(0xffffffffu, v.y, o));
        v.z = fmaxf(v.z, __shfl_xor_sync(0xffffffffu, v.z, o));
        v.w = fmaxf(v.w, __shfl_xor_sync(0xffffffffu, v.w, o));
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float4 r = red[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
        const float4 x = red[w];
        r = make_float4(fmaxf(r.x, x.x), fmaxf(r.y, x.y), fmaxf(r.z, x.z), fmaxf(r.w, x.w));
    }
    return r;
}
__device__ __forceinline__ float4 block_sum4(float4 v, float4* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
        v.z += __shfl_xor_sync(0xffffffffu, v.z, o);
        v.w += __shfl_xor_sync(0xffffffffu, v.w, o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float4 r = red[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
        const float4 x = red[w];
        r = make_float4(r.x + x.x, r.y + x.y, r.z + x.z, r.w + x.w);
    }
    return r;
}

__device__ __forceinline__ void lds128(uint32_t addr, float2& a, float2& b) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y) : "r"(addr));
}
__device__ __forceinline__ float2 add2v(float2 a, float2 b) {  // volatile: keeps its place among the LDS
    uint64_t r, x = *reinterpret_cast<uint64_t*>(&a), y = *reinterpret_cast<uint64_t*>(&b);
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ void red_shared_add(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Field K (0..7) of an 80-bit attention record (w0 = bits 0-31, w1 = 32-63, w2 = 64-79),
// shifted so its 10 bits sit at bits 7-16 (the code's row offset, 128 B per code); the bits
// below are the previous field's and are masked off by the caller.  One SHF each.
template <int K>
__device__ __forceinline__ uint32_t field_at7(uint32_t w0, uint32_t w1, uint32_t w2) {
    if constexpr (K == 0) return w0 << 7;
    else if constexpr (K <= 3) return __funnelshift_r(w0, w1, 10 * K - 7);
    else return __funnelshift_r(w1, w2, 10 * K - 39);
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// L2 cache policies: streamed-once code records evict first, the per-pair LUTs (re-read once per
// chunk by every CTA on the pair) evict last
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint2 ldg_stream_u2(const uint2* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_stream_u16(const uint16_t* p, uint64_t pol) {
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2_hint(const void* p, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol) : "memory");
}

// raw init/local rows: one CTA per pair, direct fp32 attention (no codebooks).  Runs on a side
// stream beside the LUT build; its (o, m, l) is one more partial of the pair's LSE merge.
struct RawArgs {
    const float* q;
    const float* init_k;
    const float* init_v;
    uint64_t n_init;
    const float* local_k;
    const float* local_v;
    uint64_t n_local;
    uint64_t init_stride, local_stride;  // rows between pairs
    float scale;
    uint32_t slot0;  // partial slot of pair 0
    float* part_o;
    float* part_m;
    float* part_l;
};

__global__ void __launch_bounds__(kThreads) attend_raw_rows_kernel(RawArgs a) {
    extern __shared__ __align__(16) float rsm[];
#ifndef VQKV_RAW_BATCH
#define VQKV_RAW_BATCH 16
#endif
    constexpr int kRowBatch = VQKV_RAW_BATCH;
    const uint32_t pair = blockIdx.x, slot = a.slot0 + pair;
    const uint32_t n_raw = uint32_t(a.n_init + a.n_local);
    if (n_raw == 0) {
        if (threadIdx.x < kG) {
            a.part_m[uint64_t(slot) * kG + threadIdx.x] = -INFINITY;
            a.part_l[uint64_t(slot) * kG + threadIdx.x] = 0.f;
        }
        return;
    }
    float* red = rsm;                  // 64
    float* qs = rsm + 64;              // G*D
    float* po = qs + kG * kD;          // [4 row groups][G][D] partial outputs
    float* ls = po + 4 * kG * kD;      // logits / weights [n_raw][G]
    for (uint32_t i = threadIdx.x; i < kG * kD; i += blockDim.x) qs[i] = a.q[uint64_t(pair) * kG * kD + i];
    __syncthreads();
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
            a.part_m[uint64_t(slot) * kG + g] = m;
            a.part_l[uint64_t(slot) * kG + g] = l;
        }
    }
    __syncthreads();
    // o[g][d] = sum_r p[r][g] v_r[d]: warp = row stream (rows warp, warp + 16, ...), lane = 4 columns:
    // one coalesced 512 B row per warp-load, kRowBatch rows in flight per warp, each value feeding the
    // 4 heads; the 16 streams' partials are summed in a fixed order (4 rounds into 4 smem slices)
    {
        const float4* iv = reinterpret_cast<const float4*>(a.init_v + uint64_t(pair) * a.init_stride * kD) + lane;
        const float4* lv = reinterpret_cast<const float4*>(a.local_v + uint64_t(pair) * a.local_stride * kD) + lane;
        const float4* p4 = reinterpret_cast<const float4*>(ls);
        float4 acc[kG];
#pragma unroll
        for (int g = 0; g < kG; ++g) acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t r0 = warp; r0 < n_raw; r0 += nw * kRowBatch) {
            float4 x[kRowBatch];
#pragma unroll
            for (int u = 0; u < kRowBatch; ++u) {
                const uint32_t r = r0 + u * nw;
                x[u] = (r >= n_raw) ? make_float4(0.f, 0.f, 0.f, 0.f)
                                    : (r < a.n_init) ? __ldg(iv + uint64_t(r) * (kD / 4))
                                                     : __ldg(lv + uint64_t(r - a.n_init) * (kD / 4));
            }
#pragma unroll
            for (int u = 0; u < kRowBatch; ++u) {
                const uint32_t r = r0 + u * nw;
                if (r < n_raw) {
                    const float4 p = p4[r];
                    const float pw[kG] = {p.x, p.y, p.z, p.w};
#pragma unroll
                    for (int g = 0; g < kG; ++g) {
                        acc[g].x = fmaf(pw[g], x[u].x, acc[g].x);
                        acc[g].y = fmaf(pw[g], x[u].y, acc[g].y);
                        acc[g].z = fmaf(pw[g], x[u].z, acc[g].z);
                        acc[g].w = fmaf(pw[g], x[u].w, acc[g].w);
                    }
                }
            }
        }
        // streams 4k .. 4k + 3 in round k add into slice (warp & 3)
        float4* po4 = reinterpret_cast<float4*>(po);
        for (uint32_t k = 0; k < nw / 4u; ++k) {
            if (warp / 4u == k) {
#pragma unroll
                for (int g = 0; g < kG; ++g) {
                    float4& o = po4[((warp & 3u) * kG + g) * (kD / 4) + lane];
                    if (k == 0) {
                        o = acc[g];
                    } else {
                        o.x += acc[g].x;
                        o.y += acc[g].y;
                        o.z += acc[g].z;
                        o.w += acc[g].w;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t gd = threadIdx.x; gd < kG * kD; gd += blockDim.x) {
        float o = 0.f;
        for (uint32_t rg = 0; rg < 4u; ++rg) o += po[rg * kG * kD + gd];
        a.part_o[uint64_t(slot) * kG * kD + gd] = o;
    }
}

// Compressed tokens.  The pairs' tokens are cut into 512-token units and those into chunks of 16
// units per pair (pair-major; a pair's last chunk partial); CTA b of the persistent grid takes chunks
// [C b / n_cta, C (b + 1) / n_cta), i.e. a contiguous token range that may span a pair boundary.  Its work is processed in chunks of up to 16 units of one
// pair; a run of chunks of one pair is a segment, whose partial (o, m, l) goes to slot b + pair
// (unique: CTA ranges are monotone in the pair).
struct MainArgs {
    const float4* lut;       // grouped layout (lut_off)
    uint32_t ng, R;
    const uint8_t* krec;     // attention records, krec_stride bytes between pairs, cap tokens per group segment
    uint64_t krec_stride, cap;
    const uint8_t* vcodes;   // value CodeMatrix rows
    uint64_t vstride, vrow_bits;
    const uint8_t* vend;     // end of the last pair's value payload (reads stop here)
    const StageInfo* vst;
    uint32_t vn;
    uint32_t vnwin;          // 64-bit windows of the value row (stages grouped, <= 64 bits each)
    uint2 vwin[16];          // [vnwin]: (start bit, s0 | s1 << 8) -- kernel parameters, no per-call copy
    uint8_t vwin_of[kMaxVStages];  // [vn]: window of each stage
    uint32_t vtotal;         // sum S_v (<= kHistStride): histogram entries per head
    uint32_t vslab;          // value rows staged in shared memory per slab (row_bits <= kMaxSlabRowBits)
    const float* veff;
    uint64_t n_comp;
    uint32_t n_pairs;
    uint32_t units_per_pair; // ceil(n_comp / 512)
    uint32_t n_cta;          // persistent CTAs (<= total chunks, so none is empty)
    float* part_o;           // [slots][G][D]: unnormalised sum p v
    float* part_m;           // [slots][G]
    float* part_l;           // [slots][G]
    float4* park;            // [n_cta][ncol * 128]: accumulators handed across CTA boundaries (slot = boundary)
    float4* pmeta;           // [n_cta][2]: their running max and sum
    uint32_t* bsync;         // [2 n_cta], zeroed per call: arrivals per boundary, then ready flags
};

// VQKV_ATTN_PHASES (diagnostics builds only): thread 0 of every CTA accumulates clock64 per phase
// into vqkv_attn_phase_clk[cta][8]: keys (incl. LUT waits), LUT waits, softmax, values, fold, contraction, chunks
#ifdef VQKV_ATTN_PHASES
__device__ unsigned long long vqkv_attn_phase_clk[256][16];
#define PHASE_T(v) long long v = clock64()
#define PHASE_ADD(i, t0) do { ph_acc[i] += clock64() - (t0); } while (0)
#define PHASE_CNT(i) do { ph_acc[i] += 1; } while (0)
#define PHASE_DECL unsigned long long ph_acc[16] = {0};
#define PHASE_FLUSH do { if (threadIdx.x == 0) for (int i_ = 0; i_ < 16; ++i_) vqkv_attn_phase_clk[blockIdx.x][i_] += ph_acc[i_]; } while (0)
#else
#define PHASE_CNT(i) (void)0
#define PHASE_DECL
#define PHASE_FLUSH (void)0
#define PHASE_T(v) (void)0
#define PHASE_ADD(i, t0) (void)0
#endif

constexpr uint32_t kUnit = kThreads;           // tokens per unit (one per thread)
constexpr uint32_t kUnitsPerChunk = kTok;      // 16 units = one 8192-token chunk
constexpr uint32_t kHistStride = 8192;         // histogram words per head: [head][entry]
constexpr uint32_t kTmemCols = 512;            // [0, 256): fp32 accumulator [head][entry] (4 x 64 columns x 128 lanes);
                                               // [256, 512): the chunk's fixed-point weights (16 tokens x 4 heads per thread)

// the CTA owning unit x: largest b with floor(U b / n) <= x
__host__ __device__ __forceinline__ uint32_t cta_of_unit(uint64_t x, uint64_t U, uint32_t n) {
    uint64_t b = (x * n) / U;
    while (b + 1 < n && (U * (b + 1)) / n <= x) ++b;
    while (b > 0 && (U * b) / n > x) --b;
    return uint32_t(b);
}

// The value tables of the chunk loop (smem control block) and the pair's value rows.
struct ValueHist {
    const uint8_t* vc;     // the pair's value payload
    const uint8_t* vend;   // end of the last pair's payload (reads stop here)
    uint64_t row_bits;
    uint32_t nwin;
    const uint8_t* ctl;    // smem control block: vrow / vsz / vfld / wstart / wrange tables
    uint32_t hist;         // smem address of the histograms [head][entry]
};

// One (token, head) entry of the value phase: the token's value row is read in 64-bit windows (the
// loads of the first 4 windows issued up front) and each stage's bin of that head gets one shared
// atomic.  Out of line: keeps the chunk loop's registers for the logits.
__device__ __noinline__ void hist_entry(const ValueHist& vh, uint32_t t, uint32_t g, uint32_t Pv) {
    const uint32_t* vrow = reinterpret_cast<const uint32_t*>(vh.ctl + 512);
    const uint32_t* vfld = vrow + 128;
    const uint32_t* wstart = vfld + 64;
    const uint32_t* wrange = wstart + 16;
    const uint64_t* vc64 = reinterpret_cast<const uint64_t*>(reinterpret_cast<uintptr_t>(vh.vc) & ~uintptr_t(7));
    const uint32_t vbase_bits = uint32_t((reinterpret_cast<uintptr_t>(vh.vc) & 7u) * 8u);
    const uint64_t vwords = (reinterpret_cast<uintptr_t>(vh.vend) - reinterpret_cast<uintptr_t>(vc64)) >> 3;
    const uint32_t hb = vh.hist + g * (kHistStride * 4u);
    const uint64_t rbit = uint64_t(vbase_bits) + uint64_t(t) * vh.row_bits;
    constexpr int kW = 4;  // windows loaded up front (16 x 9-bit value rows need 3)
    uint64_t lo[kW], hi[kW];
#pragma unroll
    for (int w = 0; w < kW; ++w) {
        lo[w] = hi[w] = 0;
        if (uint32_t(w) < vh.nwin) {
            const uint64_t wi = (rbit + wstart[w]) >> 6;
            if (wi + 1 < vwords) {
                lo[w] = __ldg(vc64 + wi);
                hi[w] = __ldg(vc64 + wi + 1);
            }
        }
    }
    for (uint32_t w = 0; w < vh.nwin; ++w) {
        const uint64_t pos = rbit + wstart[w];
        uint64_t x;
        if ((pos >> 6) + 1 < vwords) {
            uint64_t l, h;
            if (w < uint32_t(kW)) {
                l = lo[0], h = hi[0];
#pragma unroll
                for (int k = 1; k < kW; ++k)
                    if (w == uint32_t(k)) l = lo[k], h = hi[k];
            } else {
                l = __ldg(vc64 + (pos >> 6));
                h = __ldg(vc64 + (pos >> 6) + 1);
            }
            const uint32_t sh = uint32_t(pos & 63u);
            x = sh ? ((l >> sh) | (h << (64u - sh))) : l;
        } else {  // the last words of the buffer
            x = read_bits64(vh.vc, uint64_t(t) * vh.row_bits + wstart[w], vh.vend);
        }
        const uint32_t r = wrange[w];
        for (uint32_t st = r & 0xFFu; st < (r >> 8); ++st) {
            const uint32_t f = vfld[st];
            const uint32_t z = uint32_t(x >> (f & 0xFFu)) & ((1u << (f >> 8)) - 1u);
            red_shared_add(hb + (vrow[st] + z) * 4u, Pv);
        }
    }
}

// hist_entry with the token's value row staged in shared memory: rbit = the row's first bit relative to
// the (16 B-aligned) slab buffer at smem address vbuf.
__device__ __noinline__ void hist_entry_smem(uint32_t vbuf, uint32_t rbit, uint32_t nwin, const uint8_t* ctl,
                                             uint32_t hb, uint32_t Pv) {
    const uint32_t* vrow = reinterpret_cast<const uint32_t*>(ctl + 512);
    const uint32_t* vfld = vrow + 128;
    const uint32_t* wstart = vfld + 64;
    const uint32_t* wrange = wstart + 16;
    for (uint32_t w = 0; w < nwin; ++w) {
        const uint32_t pos = rbit + wstart[w];
        uint64_t l, h;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(l) : "r"(vbuf + ((pos >> 6) << 3)));
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(h) : "r"(vbuf + ((pos >> 6) << 3) + 8u));
        const uint32_t sh = pos & 63u;
        const uint64_t x = sh ? ((l >> sh) | (h << (64u - sh))) : l;
        const uint32_t r = wrange[w];
        for (uint32_t st = r & 0xFFu; st < (r >> 8); ++st) {
            const uint32_t f = vfld[st];
            const uint32_t z = uint32_t(x >> (f & 0xFFu)) & ((1u << (f >> 8)) - 1u);
            red_shared_add(hb + (vrow[st] + z) * 4u, Pv);
        }
    }
}

// A slab of a chunk's value rows, [st0, st1) of the pair, as bulk-copied into a slab buffer: the copy
// covers the 16 B-aligned bytes around the rows (never past the payload's last 16 B-aligned byte);
// head = bits between the buffer start and row st0; staged = bits of the buffer holding row data.
struct Slab {
    const uint8_t* src;
    uint32_t bytes, head, staged;
};
__device__ __forceinline__ Slab slab_of(const uint8_t* vc, const uint8_t* vend, uint64_t row_bits, uint32_t st0,
                                        uint32_t st1) {
    Slab sl;
    const uint8_t* b0 = vc + (uint64_t(st0) * row_bits >> 3);  // st0 * row_bits is a multiple of 8 (st0 % 512 == 0)
    const uint8_t* b1 = vc + ((uint64_t(st1) * row_bits + 7) >> 3);
    const uintptr_t s0 = reinterpret_cast<uintptr_t>(b0) & ~uintptr_t(15);
    uintptr_t s1 = (reinterpret_cast<uintptr_t>(b1) + 15) & ~uintptr_t(15);
    const uintptr_t e16 = reinterpret_cast<uintptr_t>(vend) & ~uintptr_t(15);
    if (s1 > e16) s1 = e16 > s0 ? e16 : s0;
    sl.src = reinterpret_cast<const uint8_t*>(s0);
    sl.bytes = uint32_t(s1 - s0);
    sl.head = uint32_t(reinterpret_cast<uintptr_t>(b0) - s0) * 8u;
    sl.staged = sl.bytes * 8u;
    return sl;
}

// L2 prefetch of the records of one LUT group of a chunk (both planes), ahead of the LDGs.  Out of line:
// thread 0 runs it inside the key loop.
__device__ __noinline__ void prefetch_group(const uint8_t* krec, uint64_t krec_stride, uint64_t cap, uint32_t pair,
                                            uint32_t g, uint32_t c0, uint32_t t1, uint64_t pol) {
    const uint8_t* seg = krec + uint64_t(pair) * krec_stride + uint64_t(g) * cap * 10u;
    const uint64_t n = t1 - c0;
    const uint32_t lo = uint32_t(umin64((n * 8u + 15u) & ~uint64_t(15), (cap - c0) * 8u));
    const uint32_t hi = uint32_t(umin64((n * 2u + 15u) & ~uint64_t(15), (cap - c0) * 2u));
    if (lo) prefetch_l2_hint(seg + uint64_t(c0) * 8u, lo, pol);
    if (hi) prefetch_l2_hint(seg + cap * 8u + uint64_t(c0) * 2u, hi, pol);
}

// L2 prefetch of a chunk's value rows (read by the value phase after the key phase)
__device__ __noinline__ void prefetch_values(const uint8_t* vc, uint64_t row_bits, uint32_t c0, uint32_t t1,
                                             const uint8_t* vend, uint64_t pol) {
    const uint8_t* p0 = vc + (uint64_t(c0) * row_bits >> 3);
    const uint8_t* p1 = vc + ((uint64_t(t1) * row_bits + 7) >> 3);
    if (p1 > vend) p1 = vend;
    p0 = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(p0) & ~uintptr_t(15));
    while (p0 < p1) {
        const uint32_t n = uint32_t(umin64(uint64_t(p1 - p0 + 15) & ~uint64_t(15), 65536u));
        if (p0 + n > vend) break;  // the tail that would overrun the buffer is read on demand
        prefetch_l2_hint(p0, n, pol);
        p0 += n;
    }
}

// Fold a chunk's int32 histograms (smem, [head][entry]) into the segment's fp32 accumulator in TMEM:
// acc = acc * al + H * be (acc = H * be for the first chunk).  Warp = (head, TMEM lane quarter);
// thread = entries e = 128 c + 32 quarter + lane, c < ncol (TMEM column 64 head + c): conflict-free smem
// reads, one tcgen05.ld / st per 32 columns.  Out of line: keeps the chunk loop's registers for the logits.
__device__ __noinline__ void chunk_fold(const uint8_t* lutb, uint32_t tmem, uint32_t ncol, bool first, float alg,
                                        float beg) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t hg = warp >> 2, hlq = warp & 3u;
    const uint32_t* Hw = reinterpret_cast<const uint32_t*>(lutb) + hg * kHistStride + hlq * 32u + lane;
    for (uint32_t cb = 0; cb < ncol; cb += 32u) {
        const uint32_t taddr = tmem + ((hlq * 32u) << 16) + hg * 64u + cb;
        float v[32];
        if (!first) {
            ptx::tmem_ld32(taddr, v);
            ptx::tc_wait_ld();
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            const uint32_t col = cb + uint32_t(c);
            const float hv = col < ncol ? float(Hw[col * 128u]) * beg : 0.f;
            v[c] = first ? hv : fmaf(v[c], alg, hv);
        }
        ptx::tmem_st32(taddr, v);
    }
    ptx::tc_wait_st();
}

// Segment end: o[g][d] = sum_e acc[g][e] * e_v[e][d] (e = the value stack's stage-concatenated entry),
// the TMEM accumulator staged into the smem buffer; writes the segment's partial (o, m, l).
// Pairs split between CTAs are contracted once.  At each CTA boundary the pair continues across, both
// CTAs' segments arrive (one atomic per boundary): the first parks its accumulator (float4 [entry], with
// its running max and sum) and moves on; the second merges it before going on.  A segment meets at most
// two boundaries (its CTA's right one first, then the left one); it parks, or ends with the merged
// accumulator contracted.  A second arriver only waits for the first one's park stores, so no CTA
// waits on a CTA that has not arrived.
struct Handoff {
    float4* park;      // [n_cta][n_ent]
    float4* pmeta;     // [n_cta][2]
    uint32_t* bsync;   // [2 n_cta]: arrivals, ready flags
    uint32_t n_cta;
    uint32_t kright, kleft;  // boundary indices, ~0u when the segment does not meet that boundary
    uint32_t* bcast;   // shared-memory word
};
__device__ __noinline__ void segment_contract(const float* __restrict__ veff, uint32_t vtotal, float* part_o,
                                              float* part_m, float* part_l, uint8_t* lutb, uint32_t tmem,
                                              uint32_t ncol, uint32_t slot, float4 Mn, float4 Lrun, Handoff h) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t hg = warp >> 2, hlq = warp & 3u;
    // the accumulator, staged from TMEM into the smem buffer as float4 [entry] x (4 heads)
    float* accs = reinterpret_cast<float*>(lutb);
    for (uint32_t cb = 0; cb < ncol; cb += 32u) {
        float v[32];
        ptx::tmem_ld32(tmem + ((hlq * 32u) << 16) + hg * 64u + cb, v);
        ptx::tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (cb + uint32_t(c) < ncol) accs[((cb + uint32_t(c)) * 128u + hlq * 32u + lane) * kG + hg] = v[c];
    }
    ptx::tc_fence_before();
    __syncthreads();
    const uint32_t n_ent = ncol * 128u;
    float4* a4 = reinterpret_cast<float4*>(accs);
    auto empty_partial = [&]() {
        if (tid == 0) {
            reinterpret_cast<float4*>(part_m)[slot] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            reinterpret_cast<float4*>(part_l)[slot] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    // arrive at boundary k: true for the first arriver; the second waits for the first one's park
    auto arrive = [&](uint32_t k) {
        if (tid == 0) {
            const uint32_t first = atomicAdd(h.bsync + k, 1u) == 0u;
            if (!first)
                while (ld_acquire_gpu(h.bsync + h.n_cta + k) == 0u) __nanosleep(256);
            *h.bcast = first;
        }
        __syncthreads();
        const bool first = *h.bcast != 0u;
        __syncthreads();
        return first;
    };
    auto park = [&](uint32_t k) {  // the accumulator (or an empty one: max -inf, data not written)
        if (Mn.x > -INFINITY)
            for (uint32_t e = tid; e < n_ent; e += kThreads) __stcg(h.park + uint64_t(k) * n_ent + e, a4[e]);
        if (tid == 0) {
            __stcg(h.pmeta + 2u * k, Mn);
            __stcg(h.pmeta + 2u * k + 1u, Lrun);
        }
        __threadfence();  // every thread's park stores before the ready flag
        __syncthreads();
        if (tid == 0) st_release_gpu(h.bsync + h.n_cta + k, 1u);
    };
    auto merge = [&](uint32_t k) {  // acc = acc e^(Mn - M) + parked e^(Mp - M), M = max(Mn, Mp)
        const float4 Mp = __ldcg(h.pmeta + 2u * k), Lp = __ldcg(h.pmeta + 2u * k + 1u);
        if (!(Mp.x > -INFINITY)) return;  // an empty park
        const float4 M = make_float4(fmaxf(Mn.x, Mp.x), fmaxf(Mn.y, Mp.y), fmaxf(Mn.z, Mp.z), fmaxf(Mn.w, Mp.w));
        const float4 al = make_float4(__expf(Mn.x - M.x), __expf(Mn.y - M.y), __expf(Mn.z - M.z), __expf(Mn.w - M.w));
        const float4 be = make_float4(__expf(Mp.x - M.x), __expf(Mp.y - M.y), __expf(Mp.z - M.z), __expf(Mp.w - M.w));
        const float4* src = h.park + uint64_t(k) * n_ent;
        for (uint32_t e = tid; e < n_ent; e += kThreads) {
            const float4 x = a4[e], y = __ldcg(src + e);
            a4[e] = make_float4(fmaf(y.x, be.x, x.x * al.x), fmaf(y.y, be.y, x.y * al.y), fmaf(y.z, be.z, x.z * al.z),
                                fmaf(y.w, be.w, x.w * al.w));
        }
        Lrun = make_float4(fmaf(Lp.x, be.x, Lrun.x * al.x), fmaf(Lp.y, be.y, Lrun.y * al.y),
                           fmaf(Lp.z, be.z, Lrun.z * al.z), fmaf(Lp.w, be.w, Lrun.w * al.w));
        Mn = M;
        __syncthreads();
    };
    if (h.kright != ~0u) {
        if (arrive(h.kright)) {
            park(h.kright);
            Mn = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);  // given away: e^(-inf - M) = 0 below
            Lrun = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            merge(h.kright);
        }
    }
    if (h.kleft != ~0u) {
        if (arrive(h.kleft)) {
            park(h.kleft);
            empty_partial();
            __syncthreads();
            return;
        }
        merge(h.kleft);
    }
    if (!(Mn.x > -INFINITY)) {  // everything handed over
        empty_partial();
        __syncthreads();
        return;
    }
    // warp = a slice of the entries, lane = 4 output columns: per entry one coalesced 512 B row read
    // (L2-resident codebook) and one broadcast LDS.128 of the 4 heads' weights feed 16 FMAs
    const float4* acc4 = reinterpret_cast<const float4*>(accs);
    const uint32_t per = (vtotal + 15u) / 16u, j0 = warp * per, j1 = min(vtotal, j0 + per);
    float o[kG][4];
#pragma unroll
    for (int g = 0; g < kG; ++g) o[g][0] = o[g][1] = o[g][2] = o[g][3] = 0.f;
    const float4* e4 = reinterpret_cast<const float4*>(veff) + lane;
    uint32_t j = j0;
#ifndef VQKV_CONTRACT_MLP
#define VQKV_CONTRACT_MLP 16
#endif
    constexpr uint32_t kM = VQKV_CONTRACT_MLP;  // codebook rows in flight per warp
    for (; j + kM <= j1; j += kM) {
        float4 x[kM];
#pragma unroll
        for (int i = 0; i < int(kM); ++i) x[i] = __ldg(e4 + uint64_t(j + i) * (kD / 4));
#pragma unroll
        for (int i = 0; i < int(kM); ++i) {
            const float4 w = acc4[j + i];
            const float wg[kG] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int g = 0; g < kG; ++g) {
                o[g][0] = fmaf(wg[g], x[i].x, o[g][0]);
                o[g][1] = fmaf(wg[g], x[i].y, o[g][1]);
                o[g][2] = fmaf(wg[g], x[i].z, o[g][2]);
                o[g][3] = fmaf(wg[g], x[i].w, o[g][3]);
            }
        }
    }
    for (; j < j1; ++j) {
        const float4 x = __ldg(e4 + uint64_t(j) * (kD / 4));
        const float4 w = acc4[j];
        const float wg[kG] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int g = 0; g < kG; ++g) {
            o[g][0] = fmaf(wg[g], x.x, o[g][0]);
            o[g][1] = fmaf(wg[g], x.y, o[g][1]);
            o[g][2] = fmaf(wg[g], x.z, o[g][2]);
            o[g][3] = fmaf(wg[g], x.w, o[g][3]);
        }
    }
    __syncthreads();  // accumulator consumed
    float4* po = reinterpret_cast<float4*>(lutb);  // [warp][head][lane] x float4 (4 columns)
#pragma unroll
    for (int g = 0; g < kG; ++g) po[(warp * kG + g) * 32u + lane] = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
    __syncthreads();
    {
        const uint32_t g = tid >> 7, d = tid & (kD - 1u);
        const float* pf = reinterpret_cast<const float*>(po);
        float r = 0.f;
        for (uint32_t w = 0; w < kThreads / 32u; ++w) r += pf[(w * kG + g) * kD + d];
        part_o[(uint64_t(slot) * kG + g) * kD + d] = r;
    }
    if (tid == 0) {
        reinterpret_cast<float4*>(part_m)[slot] = Mn;
        reinterpret_cast<float4*>(part_l)[slot] = Lrun;
    }
}

__global__ void __launch_bounds__(kThreads, 1) attend_atr_kernel(MainArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint8_t* const lutb = smem_raw;  // [0, 128 KB): one LUT group; the chunk's value histograms; the contraction's accumulator
    uint8_t* const ctl = smem_raw + kLutBytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(ctl);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ctl + 8);
    float4* red = reinterpret_cast<float4*>(ctl + 64);           // 16 x float4
    // value stage tables: first histogram entry (the stage's first effective row), size, field position
    // within its 64-bit window | bits << 8; window start bits and stage ranges
    uint32_t* vrow = reinterpret_cast<uint32_t*>(ctl + 512);      // [64]
    uint32_t* vsz = vrow + 64;                                    // [64]
    uint32_t* vfld = vsz + 64;                                    // [64]
    uint32_t* wstart = vfld + 64;                                 // [16]
    uint32_t* wrange = wstart + 16;                               // [16]: s0 | s1 << 8
    uint2* queue = reinterpret_cast<uint2*>(smem_raw + kLutBytes + kSmemCtl) + warp * kQueueCap;
    uint64_t* vbar = reinterpret_cast<uint64_t*>(ctl + 48);      // [2]: slab buffers full
    const uint32_t vbuf0 = ptx::smem_u32(smem_raw + kLutBytes + kSmemCtl + kQueueBytes);
    if (tid == 0) {
        ptx::mbar_init(ptx::smem_u32(bar), 1);
        ptx::mbar_init(ptx::smem_u32(&vbar[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&vbar[1]), 1);
        ptx::fence_mbar_init();
    }
    if (tid < a.vn) {
        const StageInfo si = a.vst[tid];
        vrow[tid] = uint32_t(si.eff_off / kD);
        vsz[tid] = si.size;
        vfld[tid] = (si.bit_off - a.vwin[a.vwin_of[tid]].x) | (si.bits << 8);
    }
    if (tid < a.vnwin) {
        wstart[tid] = a.vwin[tid].x;
        wrange[tid] = a.vwin[tid].y;
    }
    if (warp == 0) {
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), kTmemCols);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    PHASE_DECL
    PHASE_T(t_kernel);
    const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
    const uint32_t lut_s = ptx::smem_u32(lutb);
    const uint32_t barp = ptx::smem_u32(bar);
    const uint32_t grp_bytes = a.R * kRowBytes;
    const uint32_t upp = a.units_per_pair;
    const uint32_t U = a.n_pairs * upp;  // units (< 2^32: checked at launch)
    // CTA ranges are whole chunks (the pair-major chunk list: ceil(upp / 16) chunks per pair, the last
    // one partial): a range cut inside a chunk would cost its CTA an extra chunk (all the LUT groups
    // and per-chunk fixed work again for a few tokens)
    const uint32_t cpp = (upp + kUnitsPerChunk - 1) / kUnitsPerChunk;
    const uint32_t C = a.n_pairs * cpp;
    auto unit_of_chunk = [&](uint32_t k) {
        const uint32_t p = k / cpp;
        return min(p * upp + (k - p * cpp) * kUnitsPerChunk, U);
    };
    const uint32_t u_begin = unit_of_chunk(uint32_t(uint64_t(C) * blockIdx.x / a.n_cta));
    const uint32_t u_end = unit_of_chunk(uint32_t(uint64_t(C) * (blockIdx.x + 1) / a.n_cta));
    // CTA b's chunks are [cta_chunk0(b), cta_chunk0(b + 1))
    auto cta_chunk0 = [&](uint32_t b) { return uint32_t(uint64_t(C) * b / a.n_cta); };
    auto chunk_pair = [&](uint32_t k) { return k / cpp; };

    // chunk of unit u: its pair, token range [c0, t1) within the pair and the unit after it
    struct Chunk {
        uint32_t pair, c0, t1, next;
    };
    auto chunk_at = [&](uint32_t u) {
        Chunk c;
        c.pair = u / upp;
        const uint32_t pu = c.pair * upp;
        c.next = min(min(u_end, pu + upp), u + kUnitsPerChunk);
        c.c0 = (u - pu) * kUnit;
        c.t1 = uint32_t(umin64(a.n_comp, uint64_t(c.next - pu) * kUnit));
        return c;
    };
    auto issue = [&](uint32_t pair, uint32_t g) {  // one thread: the group's rows, one contiguous block
        ptx::mbar_arrive_expect_tx(barp, grp_bytes);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(a.lut + (uint64_t(pair) * a.ng + g) * a.R * kGS);
        for (uint32_t off = 0; off < grp_bytes; off += 32768u)
            bulk_g2s_hint(lut_s + off, src + off, min(32768u, grp_bytes - off), barp, pol_last);
    };
    // slab sl of a chunk's value rows into slab buffer sl & 1 (thread 0)
    auto issue_slab = [&](uint32_t pair, uint32_t c0, uint32_t t1, uint32_t sl) {
        const uint32_t st0 = c0 + sl * kSlabTok;
        if (st0 >= t1) return;
        const Slab x = slab_of(a.vcodes + uint64_t(pair) * a.vstride, a.vend, a.vrow_bits, st0, min(t1, st0 + kSlabTok));
        const uint32_t vb = ptx::smem_u32(&vbar[sl & 1u]);
        ptx::mbar_arrive_expect_tx(vb, x.bytes);
        for (uint32_t off = 0; off < x.bytes; off += 32768u)
            bulk_g2s_hint(vbuf0 + (sl & 1u) * kSlabBytes + off, x.src + off, min(32768u, x.bytes - off), vb, pol_first);
    };
    uint32_t vph = 0;  // slab buffer parities
    const uint32_t l7 = (lane & 7u) << 4;  // this lane's slot rotation (token & 7 == lane & 7: units are 512-aligned)
    const uint32_t hg = warp >> 2, hlq = warp & 3u;  // fold / contraction: head, TMEM lane quarter
    const uint32_t ncol = (a.vtotal + 127u) >> 7;     // accumulator columns per head (<= 64)

    // segment state (block-uniform) lives in shared memory: registers go to the logits
    float4* segM = reinterpret_cast<float4*>(ctl + 16);  // running max, then running sum at ctl + 32
    float4* segL = reinterpret_cast<float4*>(ctl + 32);
    if (tid == 0) {
        *segM = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        *segL = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    bool first = true;
    uint32_t phase = 0;
    if (tid == 0) {
        const Chunk c = chunk_at(u_begin);
        prefetch_group(a.krec, a.krec_stride, a.cap, c.pair, 0, c.c0, c.t1, pol_first);
        issue(c.pair, 0);
    }
    for (uint32_t u = u_begin; u < u_end;) {
        const Chunk ch = chunk_at(u);
        const uint32_t pair = ch.pair;
        const uint32_t c0 = ch.c0, t1 = ch.t1;
        const uint32_t nt = t1 - c0;
        const bool has_next = ch.next < u_end;
        const uint8_t* krec = a.krec + uint64_t(pair) * a.krec_stride;
        PHASE_T(t_keys);
        float2 lg[kTok][2];
#pragma unroll
        for (int k = 0; k < kTok; ++k) lg[k][0] = lg[k][1] = make_float2(0.f, 0.f);
        // ---- keys: per LUT group, 8 conflict-free lookups per token; record loads run one batch of
        // 4 tokens ahead of the lookups
        constexpr int kB = VQKV_ATTN_KB;  // tokens per record batch (loaded one batch ahead of the lookups)
        uint2 w[kB];
        uint32_t h[kB];
        const uint32_t tok0 = c0 + tid, tlast = t1 - 1u;  // record indices fit 32 bits
        auto load_batch = [&](uint32_t g, int kb, uint2 (&wo)[kB], uint32_t (&ho)[kB]) {
            const uint8_t* seg = krec + uint64_t(g) * a.cap * 10u;
            const uint2* rlo = reinterpret_cast<const uint2*>(seg);
            const uint16_t* rhi = reinterpret_cast<const uint16_t*>(seg + a.cap * 8u);
            // re-derived per batch (an opaque copy of tok0): hoisted, the 16 clamped indices would be
            // spilled and reloaded in the key loop
            uint32_t t0v;
            asm volatile("mov.u32 %0, %1;" : "=r"(t0v) : "r"(tok0));
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                // tokens past the range read the last valid record (their logits are masked)
                const uint32_t t = min(t0v + uint32_t(kb + k) * kThreads, tlast);
                wo[k] = ldg_stream_u2(rlo + t, pol_first);
                ho[k] = ldg_stream_u16(rhi + t, pol_first);
            }
        };
        load_batch(0, 0, w, h);
        for (uint32_t g = 0; g < a.ng; ++g) {
            if (tid == 0) {
                if (g + 1 < a.ng) {
                    prefetch_group(a.krec, a.krec_stride, a.cap, pair, g + 1, c0, t1, pol_first);
                } else if (has_next) {
                    const Chunk nx = chunk_at(ch.next);
                    prefetch_group(a.krec, a.krec_stride, a.cap, nx.pair, 0, nx.c0, nx.t1, pol_first);
                }
            }
            if (tid == 64) {
                // the next LUT group (or the next chunk's first) into L2 while this group is read
                const uint32_t npair = (g + 1 < a.ng) ? pair : (has_next ? ch.next / upp : pair);
                const uint32_t ng1 = (g + 1 < a.ng) ? g + 1 : 0u;
                if (g + 1 < a.ng || has_next) {
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(a.lut + (uint64_t(npair) * a.ng + ng1) * a.R * kGS);
                    for (uint32_t off = 0; off < grp_bytes; off += 32768u)
                        prefetch_l2_hint(src + off, min(32768u, grp_bytes - off), pol_last);
                }
            }
            if (g + 1 == a.ng) {  // the value rows: the first two slabs into shared memory (or L2) ahead of the value phase
                if (a.vslab) {
                    if (tid == 0) {
                        issue_slab(pair, c0, t1, 0);
                        issue_slab(pair, c0, t1, 1);
                    }
                } else if (tid == 32) {
                    prefetch_values(a.vcodes + uint64_t(pair) * a.vstride, a.vrow_bits, c0, t1, a.vend, pol_last);
                }
            }
            PHASE_T(tw);
            ptx::mbar_wait(barp, phase);
            PHASE_ADD(1, tw);
            phase ^= 1u;
#pragma unroll
            for (int kb = 0; kb < kTok; kb += kB) {
                uint2 wn[kB];
                uint32_t hn[kB];
                if (kb + kB < kTok) load_batch(g, kb + kB, wn, hn);
                else if (g + 1 < a.ng) load_batch(g + 1, 0, wn, hn);
#pragma unroll
                for (int k = 0; k < kB; ++k) {
                    const uint32_t w0 = w[k].x, w1 = w[k].y, w2 = h[k];
                    float2* L = lg[kb + k];
                    // four lookups in flight per thread (volatile order): the logits keep their
                    // registers, and 16 warps x 4 LDS.128 keep the LDS pipe full
#define VQKV_LOOK4(K0, K1, K2, K3)                                                          \
    {                                                                                       \
        const uint32_t x0 = field_at7<K0>(w0, w1, w2), x1 = field_at7<K1>(w0, w1, w2);      \
        const uint32_t x2 = field_at7<K2>(w0, w1, w2), x3 = field_at7<K3>(w0, w1, w2);      \
        float2 a0, b0, a1, b1, a2, b2, a3, b3;                                              \
        lds128(lut_s + ((x0 & 0x1FF80u) | (l7 ^ uint32_t((K0) << 4))), a0, b0);            \
        lds128(lut_s + ((x1 & 0x1FF80u) | (l7 ^ uint32_t((K1) << 4))), a1, b1);            \
        lds128(lut_s + ((x2 & 0x1FF80u) | (l7 ^ uint32_t((K2) << 4))), a2, b2);            \
        lds128(lut_s + ((x3 & 0x1FF80u) | (l7 ^ uint32_t((K3) << 4))), a3, b3);            \
        L[0] = add2v(L[0], a0);                                                             \
        L[1] = add2v(L[1], b0);                                                             \
        L[0] = add2v(L[0], a1);                                                             \
        L[1] = add2v(L[1], b1);                                                             \
        L[0] = add2v(L[0], a2);                                                             \
        L[1] = add2v(L[1], b2);                                                             \
        L[0] = add2v(L[0], a3);                                                             \
        L[1] = add2v(L[1], b3);                                                             \
    }
                    VQKV_LOOK4(0, 1, 2, 3) VQKV_LOOK4(4, 5, 6, 7)
#undef VQKV_LOOK4
                }
                if (kb + kB < kTok || g + 1 < a.ng) {
#pragma unroll
                    for (int k = 0; k < kB; ++k) {
                        w[k] = wn[k];
                        h[k] = hn[k];
                    }
                }
            }
            __syncthreads();  // every lane is done with this group's rows
            if (tid == 0 && g + 1 < a.ng) issue(pair, g + 1);
        }

        PHASE_ADD(0, t_keys);
        PHASE_T(t_soft);
        // ---- chunk softmax statistics (exact fp32 weights)
        float4 mloc = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
        for (int k = 0; k < kTok; ++k)
            if (uint32_t(k) * kThreads + tid < nt) {
                mloc.x = fmaxf(mloc.x, lg[k][0].x);
                mloc.y = fmaxf(mloc.y, lg[k][0].y);
                mloc.z = fmaxf(mloc.z, lg[k][1].x);
                mloc.w = fmaxf(mloc.w, lg[k][1].y);
            }
        const float4 mc = block_max4(mloc, red);
        float4 lloc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < kTok; ++k) {
            const bool ok = uint32_t(k) * kThreads + tid < nt;
            const float p0 = ok ? __expf(lg[k][0].x - mc.x) : 0.f, p1 = ok ? __expf(lg[k][0].y - mc.y) : 0.f;
            const float p2 = ok ? __expf(lg[k][1].x - mc.z) : 0.f, p3 = ok ? __expf(lg[k][1].y - mc.w) : 0.f;
            lg[k][0] = make_float2(p0, p1);
            lg[k][1] = make_float2(p2, p3);
            lloc.x += p0;
            lloc.y += p1;
            lloc.z += p2;
            lloc.w += p3;
        }
        const float4 lc = block_sum4(lloc, red);
        // fixed point relative to the chunk's normaliser: P = rint(p / u_c), u_c = l_c 2^-28.  The weights go
        // to this thread's TMEM columns (256 + 64 (warp / 4) + 4 k + g): the value phase reads them back 4
        // tokens at a time, so the logit registers are free for its row loads
        const float4 qs = make_float4(kQuantum / lc.x, kQuantum / lc.y, kQuantum / lc.z, kQuantum / lc.w);
        const uint32_t tP = tmem + ((hlq * 32u) << 16) + 256u + hg * 64u;
#pragma unroll
        for (int k0 = 0; k0 < kTok; k0 += 8) {
            float pw[32];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                pw[4 * k + 0] = __uint_as_float(__float2uint_rn(lg[k0 + k][0].x * qs.x));
                pw[4 * k + 1] = __uint_as_float(__float2uint_rn(lg[k0 + k][0].y * qs.y));
                pw[4 * k + 2] = __uint_as_float(__float2uint_rn(lg[k0 + k][1].x * qs.z));
                pw[4 * k + 3] = __uint_as_float(__float2uint_rn(lg[k0 + k][1].y * qs.w));
            }
            ptx::tmem_st32(tP + uint32_t(k0) * 4u, pw);
        }
        ptx::tc_wait_st();
        PHASE_ADD(2, t_soft);
        PHASE_T(t_val);
        // ---- values: int32 histograms [head][entry] over the LUT buffer.  The (token, head) pairs with a
        // nonzero weight are compacted into a per-warp queue and processed 32 at a time, lane = entry:
        // the token's value row is read in 64-bit windows (all loads first) and each stage's bin of
        // that head gets one shared atomic.
        for (uint32_t i = tid; i < kLutBytes / 16u; i += kThreads) reinterpret_cast<uint4*>(lutb)[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        PHASE_ADD(8, t_val);
        {
            ValueHist vh;
            vh.vc = a.vcodes + uint64_t(pair) * a.vstride;
            vh.vend = a.vend;
            vh.row_bits = a.vrow_bits;
            vh.nwin = a.vnwin;
            vh.ctl = ctl;
            vh.hist = lut_s;
            const uint8_t* vcp = a.vcodes + uint64_t(pair) * a.vstride;
            // lane = (entry, stage) processing: this lane's stage and its field / histogram row
            const uint32_t lanes_e = a.vn <= 16u ? 16u : (a.vn <= 32u ? 32u : 0u);
            const uint32_t s_st = lanes_e ? lane % lanes_e : 0u;
            const bool s_on = lanes_e != 0u && s_st < a.vn;
            const StageInfo s_si = a.vst[s_on ? s_st : 0u];
            const uint32_t s_bit = s_si.bit_off, s_bits = s_si.bits, s_row = vrow[s_on ? s_st : 0u];
            const uint32_t s_mask = s_bits >= 32u ? 0xFFFFFFFFu : ((1u << s_bits) - 1u);
            for (uint32_t sl = 0; sl < uint32_t(kTok) / 4u; ++sl) {
                const uint32_t st0 = c0 + sl * kSlabTok;
                if (st0 >= t1) break;
                const Slab x = slab_of(vcp, a.vend, a.vrow_bits, st0, min(t1, st0 + kSlabTok));
                const uint32_t vbuf = vbuf0 + (sl & 1u) * kSlabBytes;
                // every row of the slab in the staged bytes (all but the payload buffer's last rows)
                const bool all_staged = a.vslab && x.head + (min(t1, st0 + kSlabTok) - st0) * uint32_t(a.vrow_bits) <= x.staged;
                PHASE_T(t_sw);
                if (a.vslab) {
                    ptx::mbar_wait(ptx::smem_u32(&vbar[sl & 1u]), (vph >> (sl & 1u)) & 1u);
                    vph ^= 1u << (sl & 1u);
                }
                PHASE_ADD(9, t_sw);
                PHASE_T(t_cp);
                // a batch of queued entries, lane = (entry, stage): lanes_e lanes per entry (16 when the
                // value stack has <= 16 stages), each extracting its stage's code from the staged row and
                // doing that bin's one atomic -- short dependency chains instead of a 16-stage loop per lane
                auto process_batch = [&](uint32_t b0, uint32_t n) {
                    if (!all_staged || lanes_e == 0u) {  // generic path: lane = entry
                        if (lane < n) {
                            const uint2 e = queue[b0 + lane];
                            const uint32_t lt = e.x & 0xFFFFu, g = e.x >> 16;
                            const uint32_t rbit = x.head + (c0 + lt - st0) * uint32_t(a.vrow_bits);
                            if (a.vslab && rbit + uint32_t(a.vrow_bits) <= x.staged)
                                hist_entry_smem(vbuf, rbit, a.vnwin, ctl, lut_s + g * (kHistStride * 4u), e.y);
                            else
                                hist_entry(vh, c0 + lt, g, e.y);
                        }
                        return;
                    }
                    if (lanes_e == 16u) {
                        // two entries per step (lanes 0-15 / 16-31), four steps in flight, no branches
                        const uint32_t sub = lane >> 4;
#ifndef VQKV_VAL_STEPS
#define VQKV_VAL_STEPS 4
#endif
                        constexpr int kU = VQKV_VAL_STEPS;  // steps (entry pairs) in flight
                        for (uint32_t i0 = 0; i0 < n; i0 += 2u * kU) {
                            uint32_t addr[kU], pv[kU];
                            uint64_t lw[kU], hw[kU];
                            uint32_t sh[kU];
#pragma unroll
                            for (int u = 0; u < kU; ++u) {
                                const uint32_t i = i0 + 2u * uint32_t(u) + sub;
                                const uint2 e = queue[b0 + min(i, n - 1u)];
                                const uint32_t lt = e.x & 0xFFFFu, g = e.x >> 16;
                                const uint32_t pos = x.head + (c0 + lt - st0) * uint32_t(a.vrow_bits) + s_bit;
                                const uint32_t wa = vbuf + ((pos >> 6) << 3);
                                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(lw[u]) : "r"(wa));
                                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(hw[u]) : "r"(wa + 8u));
                                sh[u] = pos & 63u;
                                addr[u] = lut_s + (g * kHistStride + s_row) * 4u;
                                pv[u] = (i < n && s_on) ? e.y : 0u;  // padding steps add nothing
                            }
#pragma unroll
                            for (int u = 0; u < kU; ++u) {
                                const uint32_t z = uint32_t(sh[u] ? ((lw[u] >> sh[u]) | (hw[u] << (64u - sh[u]))) : lw[u]) & s_mask;
                                red_shared_add(addr[u] + z * 4u, pv[u]);
                            }
                        }
                        return;
                    }
                    const uint32_t per = 32u / lanes_e, sub = lane / lanes_e;
#pragma unroll 4
                    for (uint32_t i = sub; i < n; i += per) {
                        const uint2 e = queue[b0 + i];
                        const uint32_t lt = e.x & 0xFFFFu, g = e.x >> 16;
                        const uint32_t pos = x.head + (c0 + lt - st0) * uint32_t(a.vrow_bits) + s_bit;
                        if (!s_on) continue;
                        const uint32_t wa = vbuf + ((pos >> 6) << 3);
                        uint64_t l, h;
                        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(l) : "r"(wa));
                        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(h) : "r"(wa + 8u));
                        const uint32_t shf = pos & 63u;
                        const uint32_t z = uint32_t(shf ? ((l >> shf) | (h << (64u - shf))) : l) & s_mask;
                        red_shared_add(lut_s + (g * kHistStride + s_row + z) * 4u, e.y);
                    }
                };
                uint32_t qlen = 0;
                uint32_t P4[16];
                ptx::tmem_ld16(tP + sl * 16u, P4);
                ptx::tc_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t lt = (sl * 4u + uint32_t(k)) * kThreads + tid;  // token within the chunk
#pragma unroll
                    for (int g = 0; g < kG; ++g) {
                        const bool act = lt < nt && P4[4 * k + g] != 0u;
                        const uint32_t mask = __ballot_sync(0xffffffffu, act);
                        if (act)
                            queue[qlen + __popc(mask & ((1u << lane) - 1u))] = make_uint2(lt | (uint32_t(g) << 16), P4[4 * k + g]);
                        qlen += __popc(mask);
                    }
                    if (qlen >= 32u) {
                        __syncwarp();
                        const uint32_t full = qlen & ~31u;
                        for (uint32_t b = 0; b < full; b += 32u) process_batch(b, 32u);
                        __syncwarp();
                        if (lane < qlen - full) queue[lane] = queue[full + lane];  // keep the remainder
                        __syncwarp();
                        qlen -= full;
                    }
                }
                __syncwarp();
                process_batch(0, qlen);  // the slab's remainder (its buffer is recycled next)
                PHASE_ADD(10, t_cp);
                PHASE_T(t_sb);
                __syncthreads();
                PHASE_ADD(11, t_sb);
                if (a.vslab && tid == 0 && sl + 2u < uint32_t(kTok) / 4u) issue_slab(pair, c0, t1, sl + 2u);
            }
        }
        __syncthreads();
        PHASE_ADD(3, t_val);
        PHASE_T(t_fold);
        // ---- fold the chunk into the segment's fp32 accumulator in TMEM, rescaled to the running max.
        // Warp = (head hg, TMEM lane quarter hlq); thread = entries e = 128 c + 32 hlq + lane, c < ncol
        // (TMEM column 64 hg + c): conflict-free smem reads, one tcgen05.ld/st per 32 columns.
        const float4 M = *segM;
        const float4 Mn = make_float4(fmaxf(M.x, mc.x), fmaxf(M.y, mc.y), fmaxf(M.z, mc.z), fmaxf(M.w, mc.w));
        const float4 al = first ? make_float4(0.f, 0.f, 0.f, 0.f)
                                : make_float4(__expf(M.x - Mn.x), __expf(M.y - Mn.y), __expf(M.z - Mn.z), __expf(M.w - Mn.w));
        const float4 ec = make_float4(__expf(mc.x - Mn.x), __expf(mc.y - Mn.y), __expf(mc.z - Mn.z), __expf(mc.w - Mn.w));
        chunk_fold(lutb, tmem, ncol, first, hg == 0 ? al.x : hg == 1 ? al.y : hg == 2 ? al.z : al.w,
                   (hg == 0 ? lc.x : hg == 1 ? lc.y : hg == 2 ? lc.z : lc.w) / kQuantum *
                       (hg == 0 ? ec.x : hg == 1 ? ec.y : hg == 2 ? ec.z : ec.w));
        const float4 Lo = *segL;
        const float4 Lrun = make_float4(fmaf(Lo.x, al.x, lc.x * ec.x), fmaf(Lo.y, al.y, lc.y * ec.y),
                                        fmaf(Lo.z, al.z, lc.z * ec.z), fmaf(Lo.w, al.w, lc.w * ec.w));
        first = false;
        ptx::tc_fence_before();
        __syncthreads();  // histograms consumed, segM / segL read by every thread
        ptx::tc_fence_after();
        if (tid == 0) {
            *segM = Mn;
            *segL = Lrun;
        }
        const uint32_t next_pair = has_next ? ch.next / upp : pair;
        PHASE_ADD(4, t_fold);
        PHASE_T(t_con);

        if (!has_next || next_pair != pair) {
            // ---- segment end (out of line: keeps the chunk loop's registers for the logits); a pair that
            // continues into the next CTA or from the previous one is handed over (segment_contract)
            const uint32_t b = blockIdx.x;
            Handoff ho{a.park, a.pmeta, a.bsync, a.n_cta, ~0u, ~0u, reinterpret_cast<uint32_t*>(ctl + 320)};
            if (VQKV_ATTN_HANDOFF && a.park) {
                if (!has_next && b + 1u < a.n_cta && chunk_pair(cta_chunk0(b + 1u)) == pair) ho.kright = b;
                if (b > 0u && chunk_pair(cta_chunk0(b)) == pair && chunk_pair(cta_chunk0(b) - 1u) == pair) ho.kleft = b - 1u;
            }
            segment_contract(a.veff, a.vtotal, a.part_o, a.part_m, a.part_l, lutb, tmem, ncol, blockIdx.x + pair, Mn,
                             Lrun, ho);
            if (tid == 0) {
                *segM = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
                *segL = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            first = true;
        }
        __syncthreads();  // the buffer takes the next chunk's first LUT group; segment state updated
        PHASE_ADD(5, t_con);
        PHASE_CNT(6);
        if (tid == 0 && has_next) issue(next_pair, 0);
        u = ch.next;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, kTmemCols);
    PHASE_ADD(7, t_kernel);
    PHASE_FLUSH;
}

// out[pair][g] = sum_c exp(m_c - M) o_c / sum_c exp(m_c - M) l_c over the pair's segments and its
// raw partial; lse = M + log L (natural log of the sum of exp(scale * logits)).
__global__ void atr_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_m,
                                   const float* __restrict__ part_l, uint32_t n_cta, uint32_t upp, uint32_t n_pairs,
                                   uint32_t raw_slot0, float* __restrict__ out, float* __restrict__ lse) {
    const uint32_t pair = blockIdx.x, d = threadIdx.x, g = blockIdx.y;  // one CTA per (pair, head)
    uint32_t s_lo = 1, s_hi = 0;  // segment slots [s_lo, s_hi] (empty when there are no compressed tokens)
    if (n_cta > 0) {  // the CTAs holding the pair's first and last chunks (ranges are whole chunks)
        const uint64_t cpp = (upp + kUnitsPerChunk - 1) / kUnitsPerChunk, C = uint64_t(n_pairs) * cpp;
        s_lo = cta_of_unit(uint64_t(pair) * cpp, C, n_cta) + pair;
        s_hi = cta_of_unit(uint64_t(pair + 1) * cpp - 1, C, n_cta) + pair;
    }
    const uint32_t raw = raw_slot0 + pair;
    {
        float M = part_m[uint64_t(raw) * kG + g];
        for (uint32_t sl = s_lo; sl <= s_hi; ++sl) M = fmaxf(M, part_m[uint64_t(sl) * kG + g]);
        float L = 0.f, o = 0.f;
        auto add = [&](uint32_t sl) {
            const float m = part_m[uint64_t(sl) * kG + g];
            if (m > -INFINITY) {
                const float w = __expf(m - M);
                L = fmaf(w, part_l[uint64_t(sl) * kG + g], L);
                o = fmaf(w, part_o[(uint64_t(sl) * kG + g) * kD + d], o);
            }
        };
        for (uint32_t sl = s_lo; sl <= s_hi; ++sl) add(sl);
        add(raw);
        out[(uint64_t(pair) * kG + g) * kD + d] = o / L;
        if (d == 0 && lse) lse[uint64_t(pair) * kG + g] = M + logf(L);
    }
}

// ---- attention records -----------------------------------------------------------------
// CodeMatrix rows -> records: thread = (token, group, pair); field k of token t's record is
// the code of stage 8g + ((t & 7) ^ k) (0 for stages past the stack).
__global__ void atr_pack_kernel(const uint8_t* __restrict__ payload, uint64_t payload_stride, uint64_t row_bits,
                                const uint8_t* payload_end, const StageInfo* __restrict__ kst, uint32_t kn,
                                uint64_t src_row, uint64_t count, uint8_t* __restrict__ rec, uint64_t cap,
                                uint64_t rec_stride, uint64_t dst_row) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint32_t g = blockIdx.y, pair = blockIdx.z;
    if (i >= count) return;
    const uint64_t t = dst_row + i;  // the record's token index fixes its rotation
    const uint8_t* src = payload + pair * payload_stride;
    const uint64_t rb = (src_row + i) * row_bits;
    uint64_t lo = 0;
    uint32_t hi = 0;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t s = g * 8u + ((uint32_t(t) & 7u) ^ k);
        uint32_t z = 0;
        if (s < kn) {
            const StageInfo si = kst[s];
            z = uint32_t(read_bits64(src, rb + si.bit_off, payload_end)) & ((1u << si.bits) - 1u);
        }
        const uint32_t b = 10u * k;
        if (b + 10u <= 64u) {
            lo |= uint64_t(z) << b;
        } else if (b >= 64u) {
            hi |= z << (b - 64u);
        } else {  // field 6 straddles bit 64
            lo |= uint64_t(z) << b;
            hi |= z >> (64u - b);
        }
    }
    uint8_t* seg = rec + pair * rec_stride + uint64_t(g) * cap * 10u;
    reinterpret_cast<uint64_t*>(seg)[t] = lo;
    reinterpret_cast<uint16_t*>(seg + cap * 8u)[t] = uint16_t(hi);
}

// records -> CodeMatrix rows [0, count) of a dense per-pair payload: thread = output byte; each
// of its 8 bits is looked up as (token, stage, bit) and read from the token's record.
__global__ void atr_unpack_kernel(const uint8_t* __restrict__ rec, uint64_t cap, uint64_t rec_stride,
                                  const StageInfo* __restrict__ kst, uint32_t kn, uint64_t row_bits, uint64_t count,
                                  uint8_t* __restrict__ payload, uint64_t payload_stride) {
    extern __shared__ uint16_t bit_stage[];  // [row_bits]: stage of each row bit
    for (uint32_t b = threadIdx.x; b < row_bits; b += blockDim.x) {
        uint32_t s = 0;
        while (s + 1 < kn && b >= kst[s + 1].bit_off) ++s;
        bit_stage[b] = uint16_t(s);
    }
    __syncthreads();
    const uint64_t nbytes = (count * row_bits + 7) / 8;
    const uint64_t byte = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    const uint32_t pair = blockIdx.y;
    if (byte >= nbytes) return;
    const uint8_t* r = rec + pair * rec_stride;
    uint32_t out = 0;
    for (uint32_t i = 0; i < 8; ++i) {
        const uint64_t bit = byte * 8 + i;
        if (bit >= count * row_bits) break;
        const uint64_t t = bit / row_bits;
        const uint32_t rb = uint32_t(bit - t * row_bits), s = bit_stage[rb];
        const uint32_t g = s >> 3, k = (uint32_t(t) & 7u) ^ (s & 7u), fb = rb - kst[s].bit_off;
        const uint8_t* seg = r + uint64_t(g) * cap * 10u;
        const uint64_t lo = reinterpret_cast<const uint64_t*>(seg)[t];
        const uint32_t hi = reinterpret_cast<const uint16_t*>(seg + cap * 8u)[t];
        const uint32_t pos = 10u * k + fb;  // bit of the 80-bit record
        const uint32_t v = pos < 64u ? uint32_t(lo >> pos) & 1u : (hi >> (pos - 64u)) & 1u;
        out |= v << i;
    }
    payload[pair * payload_stride + byte] = uint8_t(out);
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

static uint32_t key_groups(const vqkv_stack_s& ks) { return (ks.n + kGS - 1) / kGS; }
static uint32_t max_size(const vqkv_stack_s& st) {
    uint32_t m = 0;
    for (const auto& s : st.stages) m = std::max(m, s.size);
    return m;
}

bool gm_supported(const vqkv_stack_s& ks) {
    if (ks.dim != kD) return false;
    for (const auto& st : ks.stages)
        if (st.size > 1024 || st.bits > 10) return false;
    return true;
}

// 64-bit windows of a value row: consecutive stages whose fields fit in 64 bits from the
// window's first field (one unaligned 64-bit read per window in the value phase)
static std::vector<uint2> value_windows(const vqkv_stack_s& vs, std::vector<uint8_t>* of = nullptr) {
    std::vector<uint2> w;
    uint32_t s0 = 0;
    while (s0 < vs.n) {
        const uint32_t b0 = vs.stages[s0].bit_off;
        uint32_t s1 = s0;
        while (s1 < vs.n && vs.stages[s1].bit_off + vs.stages[s1].bits - b0 <= 64) ++s1;
        if (of)
            for (uint32_t s = s0; s < s1; ++s) of->push_back(uint8_t(w.size()));
        w.push_back(make_uint2(b0, s0 | (s1 << 8)));
        s0 = s1;
    }
    return w;
}

bool attend_lut_supported(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a) {
    if (!gm_supported(ks) || vs.dim != kD || a.group != kG) return false;
    if (a.n_init + a.n_local > kChunk) return false;  // the raw CTA keeps one weight per raw row in smem
    if (vs.n > kMaxVStages || vs.total_rows * 4 * 4 > kLutBytes) return false;  // histograms fit the LUT buffer
    for (const auto& s : vs.stages)
        if (s.bits > 32) return false;
    if (value_windows(vs).size() > 16) return false;
    return true;
}

uint64_t gm_pair_bytes(const vqkv_stack_s& ks, uint64_t cap) { return uint64_t(key_groups(ks)) * cap * 10u; }

void launch_keycodes_to_gm(const vqkv_stack_s& ks, const uint8_t* payload, uint64_t payload_stride, uint32_t n_pairs,
                           uint64_t src_row, uint64_t count, uint8_t* gm, uint64_t cap, uint64_t gm_stride,
                           uint64_t dst_row, cudaStream_t s) {
    const uint64_t pb = payload_bytes(ks.row_bits, src_row + count);
    const uint8_t* end = payload + uint64_t(n_pairs - 1) * payload_stride + pb;
    dim3 grid(unsigned((count + 255) / 256), key_groups(ks), n_pairs);
    atr_pack_kernel<<<grid, 256, 0, s>>>(payload, payload_stride, ks.row_bits, end, ks.d_stages, ks.n, src_row, count, gm,
                                         cap, gm_stride, dst_row);
    launch_check("atr_pack_kernel");
}

void launch_keycodes_from_gm(const vqkv_stack_s& ks, const uint8_t* gm, uint64_t cap, uint64_t gm_stride,
                             uint32_t n_pairs, uint64_t count, uint8_t* payload, uint64_t payload_stride,
                             cudaStream_t s) {
    const uint64_t nbytes = payload_bytes(ks.row_bits, count);
    if (nbytes == 0) return;
    dim3 grid(unsigned((nbytes + 255) / 256), n_pairs);
    atr_unpack_kernel<<<grid, 256, sizeof(uint16_t) * ks.row_bits, s>>>(gm, cap, gm_stride, ks.d_stages, ks.n,
                                                                          ks.row_bits, count, payload, payload_stride);
    launch_check("atr_unpack_kernel");
}

// the streams of a decode-attention call beside the caller's (one pair per stack, created on first
// use): the main kernel at the highest priority, the raw-row kernel at the lowest, so that the main
// kernel's CTAs take every SM first and the raw-row CTAs run in its tail as its CTAs retire
static void attend_streams(const vqkv_stack_s& ks, cudaStream_t& lo, cudaStream_t& hi) {
    auto& st = const_cast<vqkv_stack_s&>(ks);
    std::lock_guard<std::mutex> lk(st.mu);
    if (!st.cs_attn) {
        int least = 0, greatest = 0;
        VQKV_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        cudaStream_t l = nullptr, h = nullptr;
        VQKV_CUDA(cudaStreamCreateWithPriority(&l, cudaStreamNonBlocking, least));
        const cudaError_t e = cudaStreamCreateWithPriority(&h, cudaStreamNonBlocking, greatest);
        if (e != cudaSuccess) cudaStreamDestroy(l);
        VQKV_CUDA(e);
        st.cs_attn = l;  // both or neither
        st.cs_attn_hi = h;
    }
    lo = st.cs_attn;
    hi = st.cs_attn_hi;
}

void launch_attend_lut(const vqkv_stack_s& ks, const vqkv_stack_s& vs, const vqkv_attend_args& a, cudaStream_t s) {
    const uint32_t ng = key_groups(ks), R = max_size(ks);
    const double scale = a.scale > 0.0 ? a.scale : 1.0 / std::sqrt(double(kD));
    const uint64_t n_comp = a.n_comp;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ks.device);
    // persistent main grid: one CTA per SM, balanced over 512-token units (never more CTAs than units)
    const uint32_t upp = uint32_t((n_comp + kUnit - 1) / kUnit);
    const uint64_t units = uint64_t(a.n_pairs) * upp;
    const uint64_t chunks_total = uint64_t(a.n_pairs) * ((upp + kUnitsPerChunk - 1) / kUnitsPerChunk);
    const uint32_t n_cta = uint32_t(std::min<uint64_t>(uint64_t(sms), chunks_total));  // every CTA has a chunk
    // partial slots: segments b + pair (< n_cta + n_pairs), then one raw slot per pair
    const uint32_t raw_slot0 = n_cta + a.n_pairs;
    const uint32_t n_slots = raw_slot0 + a.n_pairs;
    std::vector<uint8_t> win_of;
    const std::vector<uint2> wins = value_windows(vs, &win_of);
    // key records: the caller's attention layout, or transcoded from CodeMatrix rows here
    const uint8_t* krec = a.kcodes_dev;
    uint64_t kstride = 0, cap = a.kcodes_cap;
    uint8_t* ktmp = nullptr;
    if (n_comp > 0) {
        if (a.kcodes_layout == VQKV_KEYCODES_GROUP_MAJOR) {
            kstride = a.kcodes_stride ? a.kcodes_stride : gm_pair_bytes(ks, cap);
        } else {
            cap = (n_comp + 15) / 16 * 16;
            kstride = gm_pair_bytes(ks, cap);
            VQKV_CUDA(cudaMallocAsync(&ktmp, kstride * a.n_pairs, s));
            const uint64_t kpb = payload_bytes(ks.row_bits, n_comp);
            launch_keycodes_to_gm(ks, a.kcodes_dev, a.kcodes_stride ? a.kcodes_stride : kpb, a.n_pairs, 0, n_comp, ktmp,
                                  cap, kstride, 0, s);
            krec = ktmp;
        }
    }
    float4* lut = nullptr;
    float *po = nullptr, *pm = nullptr, *pl = nullptr;
    VQKV_CUDA(cudaMallocAsync(&po, sizeof(float) * n_slots * kG * kD, s));
    VQKV_CUDA(cudaMallocAsync(&pm, sizeof(float) * n_slots * kG, s));
    VQKV_CUDA(cudaMallocAsync(&pl, sizeof(float) * n_slots * kG, s));
    // boundary hand-off scratch: one parked accumulator per CTA boundary, arrival counters and ready flags
    const uint64_t park_ent = uint64_t((vs.total_rows + 127) / 128) * 128u;
    float4 *park = nullptr, *pmeta = nullptr;
    uint32_t* bsync = nullptr;
    if (n_comp > 0) {
        VQKV_CUDA(cudaMallocAsync(&park, sizeof(float4) * park_ent * n_cta, s));
        VQKV_CUDA(cudaMallocAsync(&pmeta, sizeof(float4) * 2 * n_cta, s));
        VQKV_CUDA(cudaMallocAsync(&bsync, sizeof(uint32_t) * 2 * n_cta, s));
        VQKV_CUDA(cudaMemsetAsync(bsync, 0, sizeof(uint32_t) * 2 * n_cta, s));
    }

    if (n_comp > 0) {
        VQKV_CUDA(cudaMallocAsync(&lut, sizeof(float4) * a.n_pairs * ng * R * kGS, s));
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
            const char* lv = getenv("VQKV_LUT_TC1");  // dev A/B: 1 = per-chunk kernel, 2 = per-stage items
            uint32_t maxch4 = 0;
            for (const auto& st : ks.stages) maxch4 = std::max(maxch4, (st.size + 127) / 128);
            if (!(lv && (lv[0] == '1' || lv[0] == '2'))) {
                const uint32_t cpq = std::max<uint32_t>(1u, uint32_t(sms) / qt);
                VQKV_CUDA(cudaFuncSetAttribute(lut_tc4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               int(kLutTc2Smem)));
                lut_tc4_kernel<<<qt * cpq, 192, kLutTc2Smem, s>>>(ks.d_eff16, ks.d_eff16lo, ks.d_stages, ks.n, qh, ql,
                                                                  qs, a.n_pairs, cpq, maxch4, ng, R, lut);
                launch_check("lut_tc4_kernel");
            } else if (ks.n <= kLutTc2MaxStages && !(lv && lv[0] == '1')) {
                const uint32_t cpq = std::max<uint32_t>(1u, uint32_t(sms) / qt);
                VQKV_CUDA(cudaFuncSetAttribute(lut_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               int(kLutTc2Smem)));
                lut_tc2_kernel<<<qt * cpq, 192, kLutTc2Smem, s>>>(ks.d_eff16, ks.d_eff16lo, ks.d_stages, ks.n, qh, ql,
                                                                  qs, a.n_pairs, cpq, ng, R, lut);
                launch_check("lut_tc2_kernel");
            } else {
                VQKV_CUDA(cudaFuncSetAttribute(lut_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLutTcSmem)));
                uint32_t maxch = 0;
                for (const auto& st : ks.stages) maxch = std::max(maxch, (st.size + 127) / 128);
                lut_tc_kernel<<<dim3(maxch, ks.n), 160, kLutTcSmem, s>>>(ks.d_eff16, ks.d_eff16lo, ks.d_stages, qh, ql,
                                                                        qs, a.n_pairs, qt, ng, R, lut);
                launch_check("lut_tc_kernel");
            }
            VQKV_CUDA(cudaFreeAsync(qh, s));
            VQKV_CUDA(cudaFreeAsync(ql, s));
            VQKV_CUDA(cudaFreeAsync(qs, s));
        } else {
            LutArgs la{a.q_dev, ks.d_eff, ks.d_stages, ks.n, ks.total_rows, float(scale), lut, ng, R};
            dim3 grid(unsigned((ks.total_rows + kLutEntries - 1) / kLutEntries), (a.n_pairs + 7) / 8);
            const int lsmem = int(sizeof(float) * (8 * kG * kD + kLutEntries * kLutStride));
            VQKV_CUDA(cudaFuncSetAttribute(lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lsmem));
            lut_kernel<<<grid, 256, lsmem, s>>>(la, a.n_pairs);
            launch_check("lut_kernel");
        }
        if (ks.n % kGS) {
            lut_zero_missing_kernel<<<a.n_pairs, 32, 0, s>>>(lut, ng, R, ks.n);
            launch_check("lut_zero_missing_kernel");
        }
    }
    cudaStream_t side, hi;
    attend_streams(ks, side, hi);
    cudaEvent_t ev_fork, ev_join, ev_main;
    VQKV_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    VQKV_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    VQKV_CUDA(cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming));
    VQKV_CUDA(cudaEventRecord(ev_fork, s));
    VQKV_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    VQKV_CUDA(cudaStreamWaitEvent(hi, ev_fork, 0));
    // raw init/local rows on the low-priority stream once the LUT is built: they run in the main
    // kernel's tail (fork / join with events)
    {
        RawArgs ra{};
        ra.q = a.q_dev;
        ra.init_k = a.init_k_dev;
        ra.init_v = a.init_v_dev;
        ra.n_init = a.n_init;
        ra.local_k = a.local_k_dev;
        ra.local_v = a.local_v_dev;
        ra.n_local = a.n_local;
        ra.init_stride = a.init_stride ? a.init_stride : a.n_init;
        ra.local_stride = a.local_stride ? a.local_stride : a.n_local;
        ra.scale = float(scale);
        ra.slot0 = raw_slot0;
        ra.part_o = po;
        ra.part_m = pm;
        ra.part_l = pl;
        const uint32_t n_raw = uint32_t(a.n_init + a.n_local);
        const int rsmem = int(sizeof(float) * (64 + kG * kD + 4 * kG * kD + uint64_t(n_raw) * kG));
        VQKV_CUDA(cudaFuncSetAttribute(attend_raw_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rsmem));
        // the largest shared-memory carveout: an SM running raw-row CTAs can take a LUT-build CTA beside
        // them (the carveout of an SM only changes when it is idle)
        VQKV_CUDA(cudaFuncSetAttribute(attend_raw_rows_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attend_raw_rows_kernel<<<a.n_pairs, kThreads, rsmem, side>>>(ra);
        launch_check("attend_raw_rows_kernel");
    }
    VQKV_CUDA(cudaEventRecord(ev_join, side));

    if (n_comp > 0) {
        ProfScope ps("attend", hi);
        const uint64_t vpb = payload_bytes(vs.row_bits, n_comp);
        const uint64_t vstr = a.vcodes_stride ? a.vcodes_stride : vpb;
        MainArgs ma{};
        ma.lut = lut;
        ma.ng = ng;
        ma.R = R;
        ma.krec = krec;
        ma.krec_stride = kstride;
        ma.cap = cap;
        ma.vcodes = a.vcodes_dev;
        ma.vstride = vstr;
        ma.vrow_bits = vs.row_bits;
        // end of the last pair's value payload: reads stop here (earlier pairs may read into the next)
        ma.vend = a.vcodes_dev + uint64_t(a.n_pairs - 1) * vstr + vpb;
        ma.vst = vs.d_stages;
        ma.vn = vs.n;
        ma.vnwin = uint32_t(wins.size());
        for (size_t w = 0; w < wins.size() && w < 16; ++w) ma.vwin[w] = wins[w];
        for (size_t st = 0; st < win_of.size() && st < kMaxVStages; ++st) ma.vwin_of[st] = win_of[st];
        ma.vtotal = uint32_t(vs.total_rows);
        ma.vslab = vs.row_bits <= kMaxSlabRowBits ? 1u : 0u;
        ma.veff = vs.d_eff;
        ma.n_comp = n_comp;
        ma.n_pairs = a.n_pairs;
        ma.units_per_pair = upp;
        ma.n_cta = n_cta;
        ma.part_o = po;
        ma.part_m = pm;
        ma.part_l = pl;
        ma.park = park;
        ma.pmeta = pmeta;
        ma.bsync = bsync;
        VQKV_CUDA(cudaFuncSetAttribute(attend_atr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMainSmem)));
        attend_atr_kernel<<<n_cta, kThreads, kMainSmem, hi>>>(ma);
        launch_check("attend_atr_kernel");
    }
    VQKV_CUDA(cudaEventRecord(ev_main, hi));
    VQKV_CUDA(cudaStreamWaitEvent(s, ev_main, 0));
    VQKV_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    {
        ProfScope ps("attend_combine", s);
        atr_combine_kernel<<<dim3(a.n_pairs, kG), kD, 0, s>>>(po, pm, pl, n_comp > 0 ? n_cta : 0u, upp, a.n_pairs, raw_slot0,
                                                    a.out_dev, a.lse_dev);
        launch_check("atr_combine_kernel");
    }
    cudaEventDestroy(ev_fork);
    cudaEventDestroy(ev_join);
    cudaEventDestroy(ev_main);
    if (lut) VQKV_CUDA(cudaFreeAsync(lut, s));
    if (ktmp) VQKV_CUDA(cudaFreeAsync(ktmp, s));
    VQKV_CUDA(cudaFreeAsync(po, s));
    VQKV_CUDA(cudaFreeAsync(pm, s));
    VQKV_CUDA(cudaFreeAsync(pl, s));
    if (park) VQKV_CUDA(cudaFreeAsync(park, s));
    if (pmeta) VQKV_CUDA(cudaFreeAsync(pmeta, s));
    if (bsync) VQKV_CUDA(cudaFreeAsync(bsync, s));
}

}  // namespace vqkv_dev

#ifdef VQKV_ATTN_PHASES
// diagnostics builds only (not part of include/vqkv_c.h): read-and-clear the per-CTA phase clocks
extern "C" int vqkv_attn_phase_read(unsigned long long* out) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, vqkv_dev::vqkv_attn_phase_clk, sizeof(unsigned long long) * 256 * 16) != cudaSuccess) return 1;
    static unsigned long long zero[256 * 16];
    return cudaMemcpyToSymbol(vqkv_dev::vqkv_attn_phase_clk, zero, sizeof(zero)) != cudaSuccess;
}
#endif
