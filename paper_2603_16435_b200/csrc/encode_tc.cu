// encode_tc.cu -- K1: residual SimVQ encode on tcgen05 tensor cores (D == 128).
//
// Replaces quantize_batch -> quantize -> nearest_scored
// (proj/core/src/codebook.cpp:158-237) with bit-identical codes.
//
// Per 128-row tile and residual stage s the scores
//     s_j = ||e_j||^2 - 2 r.e_j        (codebook.cpp:168)
// are computed as one fp16 GEMM on the tensor cores (A = fp16(r * 2^sigma),
// B = fp16 effective entries, fp32 accumulation in TMEM), finished by one FFMA
// per score in the epilogue.  The epilogue never tracks per-score indices: it
// keeps the min over contiguous 32-entry "A groups" and over the 32 residue
// classes j mod 32 ("B groups").  With a rigorous per-row bound W on
// |approx - reference| score error, every entry that can be the reference's
// argmin lies in {32a + b : mA[a] <= m + W, mB[b] <= m + W}.  When that set
// is a single entry it IS the reference's argmin; otherwise the candidates are
// rescored exactly with the reference's fp32 GEMV order (no FMA) and the
// lowest index wins ties, as nearest_scored does.  The residual update
// r -= e_z uses the exact fp32 entries, so every later stage sees the same
// residual as the reference.  Rows with non-finite input go to the exact
// SIMT encoder (their tensor-core pass runs on zeros and is discarded).
//
// CTA layout (one CTA per SM, persistent over pairs of 128-row tiles that
// advance independently -- each tile has its own chunk ring, A tile and
// accumulator, so one tile's stage end overlaps the other tile's MMAs):
//   warps 0 / 2 (lane 0)  bulk-copy producer of tile 0 / 1 (TMA engine):
//               36 KB pre-swizzled fp16 codebook chunks (128 entries x
//               (K=128 + 16-wide ||e||^2 block)) into a 2-slot ring per tile
//   warps 1 / 3 (lane 0)  MMA issuer of tile 0 / 1: per chunk 8 x
//               tcgen05.mma M128 N128 K16 + one K16 MMA for the norm block
//   warp 2      also allocates TMEM
//   warps 4-7   epilogue of tile 0 (thread = row = TMEM lane)
//   warps 8-11  epilogue of tile 1
// TMEM (512 columns): [0,128) acc tile0, [128,256) acc tile1,
//                     [256,384) fp32 residual tile0, [384,512) residual tile1.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "tc_ptx.cuh"
#include "vqkv_internal.cuh"

namespace vqkv_dev {

void launch_encode_exact_rows(const vqkv_stack_s& st, const float* xs, const uint32_t* rows_dev,
                              const uint32_t* n_rows_dev, uint64_t max_rows, uint64_t search_block, uint16_t* codes,
                              float* norms, float* residuals, cudaStream_t s);
void launch_pack_listed_rows(const uint16_t* codes, const uint32_t* rows_dev, const uint32_t* n_rows_dev,
                             uint64_t max_rows, uint64_t rows, uint32_t n_stages, const vqkv_stack_s& st,
                             uint8_t* payload, cudaStream_t s);

namespace {

constexpr int kThreads = 384;
constexpr int kNB = 2;                    // codebook chunk ring depth per tile (single-CTA kernel)
#ifndef VQKV_NBPAIR
#define VQKV_NBPAIR 3
#endif
constexpr int kNBPair = VQKV_NBPAIR;               // ring depth per tile of the CTA-pair kernel (half chunks)
constexpr uint32_t kChunkBytes = 36864;   // 128 entries x (128 + 16) fp16
constexpr uint32_t kATileBytes = 36864;   // 128 rows x (128 + 16) fp16
constexpr uint32_t kExtOff = 32768;       // the 16-wide K block (||e||^2 / row scale)
constexpr uint32_t kHalfBytes = 18432;    // CTA-pair kernel: this CTA's 64 entries of a chunk
constexpr int kMaxChunks = 8;            // chunks per super-block (1024 entries)
constexpr int kMaxSuper = 4;             // super-blocks per stage: S <= 4096
constexpr uint32_t kSmemStages = 128;     // stage descriptors cached in smem
// One N=128 MMA group per 128-entry chunk.  (Splitting a chunk into two N=64
// halves to double-buffer the accumulator was measured slower: SS-mode MMAs
// re-read A from shared memory per instruction, and at N=64 that pushes the
// operand traffic to 192 B/clk, above the ~128 B/clk smem path.)
constexpr uint32_t kIdesc = ptx::idesc_f16_f32(128, 128);
constexpr uint32_t kIdescPair = ptx::idesc_f16_f32(256, 128);
// register split: 128 x kCtlRegs + 256 x kEpiRegs <= 64K (launch allocation 168)
constexpr uint32_t kCtlRegs = 56, kEpiRegs = 224;
// setmaxnreg.inc blocks until the registers exist: what the control warpgroup releases plus the
// register file's slack over the launch allocation (168 x 384) must cover the epilogue's increase
static_assert((168u - kCtlRegs) * 128u + (65536u - 168u * kThreads) >= (kEpiRegs - 168u) * 256u,
              "register hand-over would block");
constexpr uint32_t kSleepNs = 1000000;  // control-thread barrier suspend hint

struct __align__(8) SmemCtl {
    uint64_t b_full[2][kNBPair];   // per tile: its own codebook-chunk ring
    uint64_t b_empty[2][kNBPair];
    uint64_t acc_full[2];
    uint64_t acc_empty[2];
    uint64_t a_ready[2];
    uint32_t tmem_base;
    // the first kSmemStages stage descriptors (global loads would miss L1, which the
    // 217 KB of operand buffers leave small); pad_ = 1 when the stage's last search
    // block holds a single entry (Eigen's 1-row GEMV uses the dot order for it)
    StageInfo st[kSmemStages];
};
constexpr size_t kSmemBytes = 1024 /*align slack*/ + 2 * kATileBytes + 2 * kNB * kChunkBytes + sizeof(SmemCtl);
constexpr size_t kSmemBytesPair = 1024 + 2 * kATileBytes + 2 * kNBPair * kHalfBytes + sizeof(SmemCtl);
static_assert(kNBPair * kHalfBytes <= kNB * kChunkBytes, "pair ring must fit the single-CTA layout");

// tree maximum of 32 values with 3-input FMNMX
__device__ __forceinline__ float max32(const float (&v)[32]) {
    float a[11];
#pragma unroll
    for (int i = 0; i < 10; ++i) a[i] = ptx::fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    a[10] = fmaxf(v[30], v[31]);
    float b0 = ptx::fmax3(a[0], a[1], a[2]), b1 = ptx::fmax3(a[3], a[4], a[5]);
    float b2 = ptx::fmax3(a[6], a[7], a[8]), b3 = fmaxf(a[9], a[10]);
    return fmaxf(ptx::fmax3(b0, b1, b2), b3);
}

// Power-of-two row scale so that m * 2^sigma < 2^14 (ideally in [2^13, 2^14)),
// clamped to [-23, 16] so that the ext-column factor -2^(sigma-1) is an exact
// fp16 value.  Rows whose magnitude needs sigma < -23 go to the exact path.
__device__ __forceinline__ int sigma_of(float m) {
    if (!(m > 0.f) || !isfinite(m)) return 0;
    int e;
    frexpf(m, &e);  // m in [2^(e-1), 2^e)
    return min(16, max(-23, 14 - e));
}

// ext K block of the A tile (no swizzle, 8x16 B core matrices): row i's
// columns 0..7 = {-2^(sigma-1), -2^(sigma-1), 0, ...}; columns 8..15 stay 0.
__device__ __forceinline__ void store_a_ext(uint8_t* a_tile, uint32_t i, int sigma) {
    const __half h = __float2half_rn(-ldexpf(1.0f, sigma - 1));
    __half2 hh = __halves2half2(h, h);
    uint4 w;
    w.x = *reinterpret_cast<uint32_t*>(&hh);
    w.y = w.z = w.w = 0u;
    uint8_t* p = a_tile + kExtOff + (i >> 3) * 256 + (i & 7) * 16;
    *reinterpret_cast<uint4*>(p) = w;
    *reinterpret_cast<uint4*>(p + 128) = make_uint4(0u, 0u, 0u, 0u);
}

// order-preserving map float -> uint32 (for packed (score, index) keys)
__device__ __forceinline__ uint32_t f2ord(float x) {
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// fp16(v * sc) for columns [32*c4, 32*c4+32) of row i into the SW128 K-major A tile
__device__ __forceinline__ void store_a_chunk(uint8_t* a_tile, uint32_t i, int c4, const float (&v)[32], float sc) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int kk = 32 * c4 + 8 * g;
        const int kb = kk >> 6, gi = (kk & 63) >> 3;
        const float2 s2 = make_float2(sc, sc);
        const float2 x0 = ptx::mul2(make_float2(v[8 * g + 0], v[8 * g + 1]), s2);
        const float2 x1 = ptx::mul2(make_float2(v[8 * g + 2], v[8 * g + 3]), s2);
        const float2 x2 = ptx::mul2(make_float2(v[8 * g + 4], v[8 * g + 5]), s2);
        const float2 x3 = ptx::mul2(make_float2(v[8 * g + 6], v[8 * g + 7]), s2);
        __half2 h0 = __floats2half2_rn(x0.x, x0.y);
        __half2 h1 = __floats2half2_rn(x1.x, x1.y);
        __half2 h2 = __floats2half2_rn(x2.x, x2.y);
        __half2 h3 = __floats2half2_rn(x3.x, x3.y);
        uint4 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        w.z = *reinterpret_cast<uint32_t*>(&h2);
        w.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(a_tile + kb * 16384 + i * 128 + ((gi ^ (i & 7)) << 4)) = w;
    }
}

// (pair, stage, chunk) job sequence of one tile slot of this CTA
struct JobIter {
    const StageInfo* st;
    uint32_t n_stages;
    uint32_t n_pairs, p, stride;  // work items (< 2^25: rows per call < 2^32)
    uint32_t s = 0, c = 0, nch = 0;
    bool done;
    __device__ JobIter(const StageInfo* stg, uint32_t ns, uint32_t np, uint32_t first, uint32_t step)
        : st(stg), n_stages(ns), n_pairs(np), p(first), stride(step) {
        done = p >= n_pairs;
        nch = done ? 0 : st[0].pad_size / 128;
    }
    __device__ void next() {
        if (++c < nch) return;
        c = 0;
        if (++s == n_stages) {
            s = 0;
            p += stride;
            done = p >= n_pairs;
        }
        if (!done) nch = st[s].pad_size / 128;
    }
};

struct Tile {
    uint64_t stream, row0, nvalid;  // rows [row0, row0+nvalid) of `stream`
};

__device__ __forceinline__ Tile tile_of(uint64_t t, uint64_t tiles_per_stream, uint64_t rows, uint64_t n_tiles) {
    Tile r{0, 0, 0};
    if (t >= n_tiles) return r;
    r.stream = t / tiles_per_stream;
    r.row0 = (t % tiles_per_stream) * 128;
    r.nvalid = (rows - r.row0 < 128) ? (rows - r.row0) : 128;
    return r;
}

// kPair = false: one CTA per SM, M=128 tiles.  kPair = true: clusters of two CTAs (one SM pair);
// each tile slot is a 256-row pair tile (128 rows per CTA) computed by cta_group::2 MMAs that the
// leader CTA issues: A rows come from each CTA's own shared memory, each CTA stages only its 64
// entries of every codebook chunk (half the chunk stream and half the B operand reads per SM), and
// each CTA's epilogue reads its own rows' accumulators from its own TMEM.
template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
encode_tc_kernel(const StageInfo* __restrict__ stages, uint32_t n_stages, const __half* __restrict__ eff16,
                 const float* __restrict__ sqn_pad, const float* __restrict__ eff, const float* __restrict__ xs,
                 uint32_t n_streams, uint64_t rows, uint64_t search_block, uint16_t* __restrict__ codes,
                 float* __restrict__ norms, float* __restrict__ residuals, uint32_t* __restrict__ exact_list,
                 uint32_t* __restrict__ exact_count, unsigned long long* __restrict__ counters, uint32_t dbg,
                 uint8_t* __restrict__ payload, uint64_t pay_stride, uint32_t row_bytes) {
    constexpr int NB = kPair ? kNBPair : kNB;
    constexpr uint32_t kSlot = kPair ? kHalfBytes : kChunkBytes;  // ring slot bytes
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a_tiles = smem;                                  // 2 x 36 KB
    uint8_t* b_ring = smem + 2 * kATileBytes;                 // 2 tiles x NB x slot
    SmemCtl* ctl = reinterpret_cast<SmemCtl*>(b_ring + 2 * NB * kSlot);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // (these are re-derived from special registers and parameters where used: the epilogue keeps
    // its registers for the score tiles)
    // cluster rank (clusters are consecutive CTA pairs along x): 0 = leader, issues the MMAs
#define VQKV_RANK (kPair ? (blockIdx.x & 1u) : 0u)
    const uint64_t tiles_per_stream = (rows + 127) / 128;
    const uint64_t n_tiles = tiles_per_stream * n_streams;
    // work items: pairs of tiles (one per tile slot), or quads (a pair tile per slot) per cluster
#define VQKV_N_ITEMS uint32_t(kPair ? (((rows + 127) / 128) * n_streams + 3) / 4 : (((rows + 127) / 128) * n_streams + 1) / 2)
#define VQKV_ITEM0 (kPair ? blockIdx.x >> 1 : blockIdx.x)
#define VQKV_ITEM_STEP (kPair ? gridDim.x >> 1 : gridDim.x)

    if (threadIdx.x == 0) {
        for (int t = 0; t < 2; ++t)
            for (int i = 0; i < NB; ++i) {
                // the leader's full barrier also collects the peer's "my half landed" arrival
                ptx::mbar_init(ptx::smem_u32(&ctl->b_full[t][i]), (kPair && VQKV_RANK == 0) ? 2 : 1);
                ptx::mbar_init(ptx::smem_u32(&ctl->b_empty[t][i]), 1);
            }
        for (int t = 0; t < 2; ++t) {
            ptx::mbar_init(ptx::smem_u32(&ctl->acc_full[t]), 1);
            // pair kernel: one arrival per epilogue warp of both CTAs
            ptx::mbar_init(ptx::smem_u32(&ctl->acc_empty[t]), kPair ? 8 : 128);
            ptx::mbar_init(ptx::smem_u32(&ctl->a_ready[t]), kPair ? 8 : 128);
        }
        ptx::fence_mbar_init();
    }
    for (uint32_t i = threadIdx.x; i < n_stages && i < kSmemStages; i += blockDim.x) {
        StageInfo si = stages[i];
        si.pad_ = (search_block == 1 || uint64_t(si.size) % search_block == 1) ? 1.f : 0.f;
        ctl->st[i] = si;
    }
    if (warp == 2) {
        if constexpr (kPair) {
            ptx::tmem_alloc2(ptx::smem_u32(&ctl->tmem_base), 512);
            ptx::tmem_relinquish2();
        } else {
            ptx::tmem_alloc(ptx::smem_u32(&ctl->tmem_base), 512);
            ptx::tmem_relinquish();
        }
    }
    ptx::tc_fence_before();
    if constexpr (kPair)
        ptx::cluster_sync();  // both CTAs' barriers and TMEM exist before any cross-CTA traffic
    else
        __syncthreads();
    ptx::tc_fence_after();
    // a 512-column allocation owns all of TMEM, so its address is lane 0, column 0 (a constant keeps
    // it out of the epilogue's registers)
    const uint32_t tmem = 0u;
    if (threadIdx.x == 0 && ctl->tmem_base != 0u) __trap();
    const StageInfo* stg = (n_stages <= kSmemStages) ? ctl->st : stages;  // producer / MMA stage walk
    // control warpgroup (producer / MMA threads) hands registers to the epilogue
    if (warp < 4)
        ptx::reg_dealloc<kCtlRegs>();
    else
        ptx::reg_alloc<kEpiRegs>();

    if (warp < 4) {
        // One producer thread (warps 0 / 2) and one MMA-issuer thread (warps 1 / 3)
        // per tile slot.  The two tiles advance independently (own chunk ring,
        // own accumulator), so one tile's stage-end work overlaps the other
        // tile's MMAs; every wait is a blocking mbarrier try_wait.
        const uint32_t t = warp >> 1;
        if (lane == 0 && (warp & 1) == 0) {
            // ------------------------------------------------------------ producer
            JobIter it(stg, n_stages, VQKV_N_ITEMS, VQKV_ITEM0, VQKV_ITEM_STEP);
            uint32_t slot = 0, ph = 0, n_loaded = 0;
            while (!it.done) {
                ptx::mbar_wait_sleep(ptx::smem_u32(&ctl->b_empty[t][slot]), ph ^ 1, kSleepNs);
                const uint32_t bar = ptx::smem_u32(&ctl->b_full[t][slot]);
                if ((dbg & 4u) || ((dbg & 8u) && n_loaded >= uint32_t(NB))) {
                    // timing experiments only (wrong codes): bit 2 no codebook traffic at all,
                    // bit 3 keep re-using the first ring fill (realistic ambiguity, no chunk stream)
                    ptx::mbar_arrive(bar);
                } else {
                    ptx::mbar_arrive_expect_tx(bar, kSlot);
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(eff16 + stg[it.s].eff16_off) +
                                         uint64_t(it.c) * kChunkBytes;
                    const uint32_t dst = ptx::smem_u32(b_ring + (t * NB + slot) * kSlot);
                    if constexpr (kPair) {
                        // this CTA's entries [64 rank, 64 rank + 64) of the chunk: both 64-wide K blocks
                        // (SW128 rows of 128 B) and the ext block's 8 core-matrix row groups
                        ptx::bulk_g2s(dst, src + VQKV_RANK * 8192u, 8192u, bar);
                        ptx::bulk_g2s(dst + 8192u, src + 16384u + VQKV_RANK * 8192u, 8192u, bar);
                        ptx::bulk_g2s(dst + 16384u, src + kExtOff + VQKV_RANK * 2048u, 2048u, bar);
                    } else {
                        ptx::bulk_g2s(dst, src, kChunkBytes, bar);
                    }
                    ++n_loaded;
                }
                if (++slot == NB) {
                    slot = 0;
                    ph ^= 1;
                }
                it.next();
            }
        } else if (lane == 0 && kPair && VQKV_RANK != 0) {
            // ------------------------------------------------------------ peer: half-chunk forwarder
            // the leader's MMAs read this CTA's half of each chunk: tell its full barrier when it landed
            JobIter it(stg, n_stages, VQKV_N_ITEMS, VQKV_ITEM0, VQKV_ITEM_STEP);
            uint32_t slot = 0, ph = 0;
            while (!it.done) {
                const uint32_t bar = ptx::smem_u32(&ctl->b_full[t][slot]);
                ptx::mbar_wait_sleep(bar, ph, kSleepNs);
                ptx::mbar_arrive_cluster(ptx::mapa(bar, 0u));
                if (++slot == NB) {
                    slot = 0;
                    ph ^= 1;
                }
                it.next();
            }
        } else if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            JobIter it(stg, n_stages, VQKV_N_ITEMS, VQKV_ITEM0, VQKV_ITEM_STEP);
            uint32_t slot = 0, ph = 0, a_ph = 0, e_ph = 1;
            const uint32_t a_base = ptx::smem_u32(a_tiles) + t * kATileBytes;
            const uint32_t b_base = ptx::smem_u32(b_ring);
            // K-block stride of the B operand in shared memory: 64 or 128 entry rows of 128 B
            constexpr uint32_t kBkb = kPair ? 8192u : 16384u;
            constexpr uint32_t kBext = kPair ? 16384u : kExtOff;
#ifdef VQKV_PHASE_CLOCKS
            unsigned long long mk[4] = {0, 0, 0, 0};
            long long m0 = clock64(), m1;
#define VQKV_MCLK(k) { m1 = clock64(); mk[k] += (unsigned long long)(m1 - m0); m0 = m1; }
#else
#define VQKV_MCLK(k) {}
#endif
            while (!it.done) {
                // (pair kernel: the peer's arrivals use default .cta semantics, as in CUTLASS's 2-SM
                // pipelines; the data they hand over is ordered by tcgen05 / proxy fences)
                ptx::mbar_wait_sleep(ptx::smem_u32(&ctl->b_full[t][slot]), ph, kSleepNs);
                VQKV_MCLK(2)
                if (it.c == 0) {
                    ptx::mbar_wait_sleep(ptx::smem_u32(&ctl->a_ready[t]), a_ph, kSleepNs);
                    a_ph ^= 1;
                }
                VQKV_MCLK(3)
                ptx::mbar_wait_sleep(ptx::smem_u32(&ctl->acc_empty[t]), e_ph, kSleepNs);
                VQKV_MCLK(0)
                const uint32_t bb = b_base + (t * NB + slot) * kSlot;
                e_ph ^= 1;
                ptx::tc_fence_after();
                const uint32_t d = tmem + 128u * t;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t koff = (k & 3) * 32;
                    const uint64_t ad = ptx::umma_desc_sw128(a_base + (k >> 2) * 16384 + koff);
                    const uint64_t bd = ptx::umma_desc_sw128(bb + (k >> 2) * kBkb + koff);
                    if constexpr (kPair)
                        ptx::mma2_f16_ss(d, ad, bd, kIdescPair, k > 0 ? 1u : 0u);
                    else
                        ptx::mma_f16_ss(d, ad, bd, kIdesc, k > 0 ? 1u : 0u);
                }
                // + (-2^(sigma-1)) * (||e||^2 hi + lo): the score's norm term
                if (!(dbg & 1u)) {
                    const uint64_t ad = ptx::umma_desc_noswz(a_base + kExtOff, 128, 256);
                    const uint64_t bd = ptx::umma_desc_noswz(bb + kBext, 128, 256);
                    if constexpr (kPair)
                        ptx::mma2_f16_ss(d, ad, bd, kIdescPair, 1u);
                    else
                        ptx::mma_f16_ss(d, ad, bd, kIdesc, 1u);
                }
                if constexpr (kPair) {
                    ptx::mma2_commit_mc(ptx::smem_u32(&ctl->acc_full[t]), uint16_t(3));
                    ptx::mma2_commit_mc(ptx::smem_u32(&ctl->b_empty[t][slot]), uint16_t(3));
                } else {
                    ptx::mma_commit(ptx::smem_u32(&ctl->acc_full[t]));
                    ptx::mma_commit(ptx::smem_u32(&ctl->b_empty[t][slot]));
                }
                VQKV_MCLK(1)
                if (++slot == NB) {
                    slot = 0;
                    ph ^= 1;
                }
                it.next();
            }
#ifdef VQKV_PHASE_CLOCKS
            if ((dbg & 2u) && counters)
                for (int k = 0; k < 4; ++k) atomicAdd(&counters[21 + k], mk[k]);
#endif
#undef VQKV_MCLK
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const uint32_t t = (warp - 4) >> 2;          // tile slot
        const uint32_t q = warp & 3;                 // TMEM lane quadrant
        const uint32_t i = q * 32 + lane;            // row within tile
        const uint32_t lane_off = (q * 32u) << 16;
        const uint32_t t_acc = tmem + lane_off + 128u * t;
        const uint32_t t_res = tmem + lane_off + 256u + 128u * t;
        const uint32_t bar_full = ptx::smem_u32(&ctl->acc_full[t]);
        const uint32_t bar_empty = ptx::smem_u32(&ctl->acc_empty[t]);
        const uint32_t bar_aready = ptx::smem_u32(&ctl->a_ready[t]);
        uint8_t* a_tile = a_tiles + t * kATileBytes;
        uint32_t f_ph = 0;
        unsigned long long n_amb = 0, n_rs = 0, n_rowstages = 0;
        // per-phase clock totals (lane 0 of each epilogue warp, dbg bit 1): compiled in
        // only for diagnostics builds (VQKV_PHASE_CLOCKS), they cost ~28 registers
#ifdef VQKV_PHASE_CLOCKS
        const bool clk_on = (dbg & 2u) && counters && lane == 0;
        unsigned long long ck[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        long long ck_t = clock64();
#define VQKV_PHASE(k)                               \
    if (clk_on) {                                   \
        const long long now_ = clock64();           \
        ck[k] += (unsigned long long)(now_ - ck_t); \
        ck_t = now_;                                \
    }
        // clock read ordered after `dep` is available (waits for the load feeding it)
#define VQKV_PHASE_DEP(k, dep)                                                       \
    if (clk_on) {                                                                    \
        long long now_;                                                              \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(now_) : "f"(dep) : "memory");   \
        ck[k] += (unsigned long long)(now_ - ck_t);                                  \
        ck_t = now_;                                                                 \
    }
#else
#define VQKV_PHASE(k) {}  // a complete (empty) statement: call sites follow `if (...)`
#define VQKV_PHASE_DEP(k, dep) {}
#endif

        // release of the accumulator / the next A tile to the MMA issuer: every thread (single CTA),
        // or one lane per warp after the warp's own tcgen05 / shared-memory work (CTA pair: the
        // peer CTA's warps arrive on the leader's barriers)
        auto release = [&](uint32_t bar, bool smem_written) {
            if constexpr (kPair) {
                if (smem_written) __syncwarp();  // the other lanes' proxy fences precede lane 0's arrive
                // the leader's barrier (mapa of its own address is itself)
                ptx::mbar_arrive_cluster_if(ptx::mapa(bar, 0u), lane == 0);
            } else {
                ptx::mbar_arrive(bar);
            }
        };
        for (uint32_t p = VQKV_ITEM0; p < VQKV_N_ITEMS; p += VQKV_ITEM_STEP) {
            const Tile tl = tile_of(kPair ? 4ull * p + 2 * t + VQKV_RANK : 2ull * p + t, tiles_per_stream, rows, n_tiles);
            const bool valid = i < tl.nvalid;
            const uint64_t grow = tl.stream * rows + tl.row0 + i;  // global row index
            bool exact_row = false;
            if (valid) n_rowstages += n_stages;

            // ---- x -> TMEM residual (pass 1), stats
            float R2 = 0.f, mx = 0.f;
            {
                const float4* x4 = reinterpret_cast<const float4*>(xs + grow * 128);
#pragma unroll 1
                for (int c4 = 0; c4 < 4; ++c4) {
                    float v[32];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        float4 a = valid ? __ldg(x4 + c4 * 8 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[4 * k] = a.x;
                        v[4 * k + 1] = a.y;
                        v[4 * k + 2] = a.z;
                        v[4 * k + 3] = a.w;
                    }
#pragma unroll
                    for (int k = 0; k < 32; ++k) exact_row |= !isfinite(v[k]);
                    ptx::tmem_st32(t_res + 32u * c4, v);
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        R2 = fmaf(v[k], v[k], R2);
                        mx = fmaxf(mx, fabsf(v[k]));
                    }
                }
                // magnitudes beyond the fp16 row-scale range also take the exact path
                exact_row |= !(mx < 68719476736.0f);  // 2^36
            }
            if (exact_row) {
                // hand the row to the exact path; run the tensor-core pass on zeros
                const uint32_t slot = atomicAdd(exact_count, 1u);
                exact_list[slot] = uint32_t(grow);
                if (counters) atomicAdd(&counters[2], 1ull);
                R2 = 0.f;
                mx = 0.f;
            }
            if (__any_sync(0xffffffffu, exact_row)) {
                // tcgen05.ld/st are warp-collective: the whole warp rewrites its rows
                ptx::tc_wait_st();
#pragma unroll 1
                for (int c4 = 0; c4 < 4; ++c4) {
                    float v[32];
                    ptx::tmem_ld32(t_res + 32u * c4, v);
                    ptx::tc_wait_ld();
#pragma unroll
                    for (int k = 0; k < 32; ++k) v[k] = exact_row ? 0.f : v[k];
                    ptx::tmem_st32(t_res + 32u * c4, v);
                }
            }
            ptx::tc_wait_st();
            int sigma = sigma_of(mx);
            {   // ---- pass 2: A tile for stage 0
                const float sc = ldexpf(1.0f, sigma);
#pragma unroll 1
                for (int c4 = 0; c4 < 4; ++c4) {
                    float v[32];
                    ptx::tmem_ld32(t_res + 32u * c4, v);
                    ptx::tc_wait_ld();
                    store_a_chunk(a_tile, i, c4, v, sc);
                }
                store_a_ext(a_tile, i, sigma);
                ptx::fence_async_smem();
                ptx::tc_fence_before();
                release(bar_aready, true);
            }
            VQKV_PHASE(0)

            // CodeMatrix row written directly (payload != nullptr: row_bits % 16 == 0): the row's
            // LSB-first bit stream (codebook.cpp:96-120) is assembled stage by stage and stored 16 bits
            // at a time; otherwise u16 codes go to the scratch for the pack kernel
            uint32_t pk_acc = 0, pk_n = 0;
            uint16_t* pk_dst = payload ? reinterpret_cast<uint16_t*>(payload + tl.stream * pay_stride +
                                                                      (tl.row0 + i) * uint64_t(row_bytes))
                                       : nullptr;
            for (uint32_t s = 0; s < n_stages; ++s) {
                const StageInfo& si = (s < kSmemStages) ? ctl->st[s] : stages[s];
                const bool any_one_s = (s < kSmemStages) ? (si.pad_ != 0.f)
                                                         : (search_block == 1 || uint64_t(si.size) % search_block == 1);
                if (dbg & 32u) {
                    // timing experiment only (wrong codes): the epilogue just drains the
                    // accumulators and re-releases the A tile -- the bare MMA pipeline
                    const uint32_t nchx = si.pad_size / 128;
                    for (uint32_t c = 0; c < nchx; ++c) {
                        ptx::mbar_wait(bar_full, f_ph);
                        f_ph ^= 1;
                        ptx::tc_fence_after();
                        ptx::tc_fence_before();
                        release(bar_empty, false);
                    }
                    if (s + 1 < n_stages) release(bar_aready, true);
                    continue;
                }
                // ---- error window ("exactness of the tensor-core encoder")
                const float R = sqrtf(R2 * 1.0001f);
                const float E = si.max_norm;
                const float Bnd = 2.1e-3f * R * E + 1.6e-5f * si.max_sqnorm + 6.8e-7f * (ldexpf(E, -sigma) + R) +
                                  ldexpf(2.3e-13f, -sigma) + 6e-8f + 1e-30f;
                // The MMA yields Y_j = 2^sigma r.e_j - 2^(sigma-1)||e_j||^2 = -2^(sigma-1) score_j,
                // so argmin score == argmax Y and the window scales by 2^(sigma-1).
                const float W = ldexpf(2.02f * Bnd, sigma - 1);

                // ---- max over A groups (32 contiguous entries) and B groups (j mod 32),
                // per super-block of <= kMaxChunks chunks (1024 entries).  A block's
                // candidate masks use the running maximum, which only grows, so the
                // masks of earlier blocks stay supersets of the final candidate set.
                const uint32_t nch = si.pad_size / 128;
                const uint32_t nsb = (nch + kMaxChunks - 1) / kMaxChunks;
                const float* sqn_s = sqn_pad + si.pad_off;
                float m1 = -INFINITY;
                uint32_t CAs[kMaxSuper], CBs[kMaxSuper];
                float mbs[kMaxSuper];  // per-block maxima
#pragma unroll
                for (int k = 0; k < kMaxSuper; ++k) {
                    CAs[k] = CBs[k] = 0u;
                    mbs[k] = -INFINITY;
                }
#pragma unroll
                for (int sb = 0; sb < kMaxSuper; ++sb) {
                    if (sb >= int(nsb)) break;
                    float mA[4 * kMaxChunks], mB[32];
#pragma unroll
                    for (int k = 0; k < 4 * kMaxChunks; ++k) mA[k] = -INFINITY;
#pragma unroll
                    for (int k = 0; k < 32; ++k) mB[k] = -INFINITY;
#pragma unroll
                    for (int c = 0; c < kMaxChunks; ++c) {
                        if (sb * kMaxChunks + c < int(nch)) {
                            VQKV_PHASE(2)
                            ptx::mbar_wait(bar_full, f_ph);
                            VQKV_PHASE(1)
                            f_ph ^= 1;
                            ptx::tc_fence_after();
                            // all 128 columns in flight at once, one wait, then the
                            // accumulator goes back to the MMA issuer before the max trees
                            float v0[32], v1[32], v2[32], v3[32];
                            ptx::tmem_ld32(t_acc, v0);
                            ptx::tmem_ld32(t_acc + 32u, v1);
                            ptx::tmem_ld32(t_acc + 64u, v2);
                            ptx::tmem_ld32(t_acc + 96u, v3);
                            ptx::tc_wait_ld();
                            ptx::tc_fence_before();
                            release(bar_empty, false);
                            VQKV_PHASE_DEP(12, v3[31])
                            mA[4 * c] = max32(v0);
                            mA[4 * c + 1] = max32(v1);
                            mA[4 * c + 2] = max32(v2);
                            mA[4 * c + 3] = max32(v3);
#pragma unroll
                            for (int b = 0; b < 32; ++b)
                                mB[b] = ptx::fmax3(mB[b], ptx::fmax3(v0[b], v1[b], v2[b]), v3[b]);
                        }
                    }
                    VQKV_PHASE(2)
                    // ---- candidates {1024 sb + 32a + b : mA[a] >= m - W, mB[b] >= m - W}
                    float mb = -INFINITY;
#pragma unroll
                    for (int k = 0; k < 4 * kMaxChunks; ++k) mb = fmaxf(mb, mA[k]);
                    mbs[sb] = mb;
                    m1 = fmaxf(m1, mb);
                    const float thr = m1 - W;
                    uint32_t CA = 0, CB = 0;
#pragma unroll
                    for (int k = 0; k < 4 * kMaxChunks; ++k) CA |= (mA[k] >= thr ? 1u : 0u) << k;
#pragma unroll
                    for (int b = 0; b < 32; ++b) CB |= (mB[b] >= thr ? 1u : 0u) << b;
                    CAs[sb] = CA;
                    CBs[sb] = CB;
                }
                uint32_t total = 0, zu = 0;
#pragma unroll
                for (int sb = 0; sb < kMaxSuper; ++sb) {
                    // a block whose maximum is below the final threshold holds no candidate
                    if (!(mbs[sb] >= m1 - W)) CAs[sb] = CBs[sb] = 0u;
                    const uint32_t cb = uint32_t(__popc(CAs[sb])) * uint32_t(__popc(CBs[sb]));
                    if (cb == 1u) zu = 1024u * sb + 32u * (__ffs(CAs[sb]) - 1) + (__ffs(CBs[sb]) - 1);
                    total += cb;
                }
                const bool unique = (total == 1u);
                uint32_t z = unique ? zu : 0u;
                const bool amb = !unique && valid && !exact_row;
                VQKV_PHASE(3)
                if (__any_sync(0xffffffffu, amb)) {
                    // ---- warp-cooperative exact rescoring in the reference's fp32 order
                    // (codebook.cpp:166-172).  The (row, candidate) items of all lanes
                    // are packed 32 per pass; r of the owning row is broadcast by shuffle.
                    // One round per super-block; the best (score, index) key carries over.
                    unsigned long long best = ~0ull;
                    uint32_t cnt_all = 0;
#pragma unroll 1
                    for (int sb = 0; sb < int(nsb); ++sb) {
                    uint32_t CA = CAs[0], CB = CBs[0];
#pragma unroll
                    for (int k = 1; k < kMaxSuper; ++k)
                        if (sb == k) {
                            CA = CAs[k];
                            CB = CBs[k];
                        }
                    const uint32_t na = __popc(CA), nb = __popc(CB);
                    const uint32_t cnt = amb ? na * nb : 0u;
                    cnt_all += cnt;
                    if (!__any_sync(0xffffffffu, cnt != 0u)) continue;
                    uint32_t incl = cnt;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                        if (lane >= uint32_t(off)) incl += y;
                    }
                    const uint32_t P = incl - cnt;
                    const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
                    const bool any_one = any_one_s;
                    for (uint32_t base = 0; base < T; base += 32) {
                        const uint32_t it = base + lane;
                        uint32_t o = 0;
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1) {
                            const uint32_t Pc = __shfl_sync(0xffffffffu, P, o + step);
                            if (Pc <= it) o += step;
                        }
                        const uint32_t li = it - __shfl_sync(0xffffffffu, P, o);
                        const uint32_t CAo = __shfl_sync(0xffffffffu, CA, o);
                        const uint32_t CBo = __shfl_sync(0xffffffffu, CB, o);
                        uint32_t j = 0xffffffffu;
                        if (it < T) {
                            // item li of the owner -> (a, b) = (li / nb)-th set bit of CA, (li % nb)-th of CB
                            const uint32_t nbo = __popc(CBo);
                            const uint32_t qa = uint32_t((float(li) + 0.5f) * __frcp_rn(float(nbo)));  // exact: li < 2^16
                            const uint32_t rb = li - qa * nbo;
                            uint32_t ma = CAo, mbb = CBo;
                            for (uint32_t k = 0; k < qa; ++k) ma &= ma - 1u;
                            for (uint32_t k = 0; k < rb; ++k) mbb &= mbb - 1u;
                            j = 1024u * uint32_t(sb) + 32u * uint32_t(__ffs(ma) - 1) + uint32_t(__ffs(mbb) - 1);
                            if (j >= si.size) j = 0xffffffffu;
                        }
                        VQKV_PHASE(5)
                        const bool has = (j != 0xffffffffu);
                        const float4* e4 = reinterpret_cast<const float4*>(eff + si.eff_off + uint64_t(has ? j : 0) * 128);
                        // the whole entry row and its norm in one L2 round trip
                        const float sqj = has ? __ldg(sqn_s + j) : 0.f;
                        float ev[128];
#pragma unroll
                        for (int kk = 0; kk < 16; ++kk) ptx::ldg256_na(reinterpret_cast<const float*>(e4) + 8 * kk, ev + 8 * kk);
                        float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
                        float r0[4] = {0.f, 0.f, 0.f, 0.f}, r1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) {
                            float v[32];
                            ptx::tmem_ld32(t_res + 32u * c4, v);
                            ptx::tc_wait_ld();
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk) {
                                // scalar FMUL + packed FADD2: each lane is the same IEEE op in the same
                                // order.  (ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even with
                                // --fmad=false, so the products must not be f32x2; tests/test_sass.py.)
                                float q[4];
#pragma unroll
                                for (int l = 0; l < 4; ++l)
                                    q[l] = __fmul_rn(ev[32 * c4 + 4 * kk + l], __shfl_sync(0xffffffffu, v[4 * kk + l], o));
                                const float2 p01 = make_float2(q[0], q[1]), p23 = make_float2(q[2], q[3]);
                                {
                                    float2 g01 = ptx::add2(make_float2(g0, g1), p01), g23 = ptx::add2(make_float2(g2, g3), p23);
                                    g0 = g01.x;
                                    g1 = g01.y;
                                    g2 = g23.x;
                                    g3 = g23.y;
                                }
                                if (any_one) {
                                    float* rr = (kk & 1) ? r1 : r0;
                                    const float2 a01 = ptx::add2(make_float2(rr[0], rr[1]), p01);
                                    const float2 a23 = ptx::add2(make_float2(rr[2], rr[3]), p23);
                                    rr[0] = a01.x;
                                    rr[1] = a01.y;
                                    rr[2] = a23.x;
                                    rr[3] = a23.y;
                                }
                            }
                        }
                        VQKV_PHASE(6)
                        unsigned long long key = ~0ull;
                        if (has) {
                            const bool one = any_one && (search_block == 1 || j + 1 == si.size);
                            float dot;
                            if (one) {
#pragma unroll
                                for (int l = 0; l < 4; ++l) r0[l] = __fadd_rn(r0[l], r1[l]);
                                dot = __fadd_rn(__fadd_rn(r0[0], r0[2]), __fadd_rn(r0[1], r0[3]));
                            } else {
                                dot = __fadd_rn(__fadd_rn(g0, g2), __fadd_rn(g1, g3));
                            }
                            const float sc = __fadd_rn(__fsub_rn(sqj, __fmul_rn(2.0f, dot)), 0.0f);
                            if (sc < INFINITY) key = (uint64_t(f2ord(sc)) << 32) | j;  // NaN / +inf never win
                        }
                        // segmented min over consecutive lanes of the same owner
#pragma unroll
                        for (int off = 1; off < 32; off <<= 1) {
                            const unsigned long long ok = __shfl_down_sync(0xffffffffu, key, off);
                            const uint32_t oo = __shfl_down_sync(0xffffffffu, o, off);
                            if (lane + off < 32 && oo == o && ok < key) key = ok;
                        }
                        const int head = int(P) - int(base);
                        const unsigned long long got = __shfl_sync(0xffffffffu, key, head < 0 ? 0 : (head > 31 ? 31 : head));
                        if (cnt != 0u && P + cnt > base && P < base + 32 && got < best) best = got;  // own items only
                        VQKV_PHASE(7)
                    }
                    }  // super-blocks
                    if (amb) {
                        z = (best == ~0ull) ? 0u : uint32_t(best & 0xffffffffu);
                        n_rs += cnt_all;
                        ++n_amb;
                        const float* ez = eff + si.eff_off + uint64_t(z) * 128;
#pragma unroll
                        for (int l = 0; l < 4; ++l) ptx::prefetch_l1(ez + 32 * l);
                    }
                }
                if (pk_dst) {
                    pk_acc |= z << pk_n;  // pk_n < 16 before, bits <= 16: pk_n stays below 32
                    pk_n += si.bits;
                    if (pk_n >= 16) {
                        if (valid && !exact_row) *pk_dst = uint16_t(pk_acc);
                        ++pk_dst;
                        pk_acc >>= 16;
                        pk_n -= 16;
                    }
                } else if (valid && !exact_row) {
                    codes[grow * n_stages + s] = uint16_t(z);
                }
                VQKV_PHASE(8)

                // ---- residual update r -= e_z (exact fp32) fused with the next stage's A tile
                const bool last = (s + 1 == n_stages);
                const int sigma_n = sigma_of(mx + si.max_abs);  // max|r - e| <= max|r| + max|e|
                const float sc_n = ldexpf(1.0f, sigma_n);
                if (!last) store_a_ext(a_tile, i, sigma_n);
                const float4* ez4 = reinterpret_cast<const float4*>(eff + si.eff_off + uint64_t(z) * 128);
                float2 R2p = make_float2(0.f, 0.f);
                float mxn = 0.f;
                float n0[4] = {0.f, 0.f, 0.f, 0.f}, n1[4] = {0.f, 0.f, 0.f, 0.f};
                float en[128];  // e_z in one L2 round trip
                if (dbg & 16u) {  // timing experiment only: no e_z gather (wrong residuals)
#pragma unroll
                    for (int k = 0; k < 128; ++k) en[k] = 0.f;
                } else {
#pragma unroll
                    for (int kk = 0; kk < 16; ++kk)
                        ptx::ldg256_na(reinterpret_cast<const float*>(ez4) + 8 * kk, en + 8 * kk);
                }
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    float v[32];
                    ptx::tmem_ld32(t_res + 32u * c4, v);
                    ptx::tc_wait_ld();
                    if (c4 == 0) VQKV_PHASE_DEP(9, v[0])
#pragma unroll
                    for (int k = 0; k < 32; k += 2) {  // FADD2 of -e: identical to v - e lane by lane
                        const float2 d = ptx::add2(make_float2(v[k], v[k + 1]),
                                                   make_float2(-en[32 * c4 + k], -en[32 * c4 + k + 1]));
                        v[k] = d.x;
                        v[k + 1] = d.y;
                    }
                    if (c4 == 0) VQKV_PHASE_DEP(10, v[31])
                    ptx::tmem_st32(t_res + 32u * c4, v);
                    if (!last) {
#pragma unroll
                        for (int k = 0; k < 32; k += 2) {  // two partial sums: R2 only feeds the (slacked) window bound
                            R2p = ptx::fma2(make_float2(v[k], v[k + 1]), make_float2(v[k], v[k + 1]), R2p);
                            mxn = ptx::fmax3(mxn, fabsf(v[k]), fabsf(v[k + 1]));
                        }
                        store_a_chunk(a_tile, i, c4, v, sc_n);
                    } else {
                        // final ||r|| in the reference's redux order (Eigen squaredNorm)
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            float* rr = (kk & 1) ? n1 : n0;
#pragma unroll
                            for (int l = 0; l < 4; l += 2) {  // FMUL + FADD2 (not FMUL2: see the rescoring loop)
                                const float2 x = make_float2(__fmul_rn(v[4 * kk + l], v[4 * kk + l]),
                                                             __fmul_rn(v[4 * kk + l + 1], v[4 * kk + l + 1]));
                                const float2 a = ptx::add2(make_float2(rr[l], rr[l + 1]), x);
                                rr[l] = a.x;
                                rr[l + 1] = a.y;
                            }
                        }
                        if (residuals && valid && !exact_row) {
                            float4* o4 = reinterpret_cast<float4*>(residuals + grow * 128 + 32 * c4);
#pragma unroll
                            for (int kk = 0; kk < 8; ++kk)
                                o4[kk] = make_float4(v[4 * kk], v[4 * kk + 1], v[4 * kk + 2], v[4 * kk + 3]);
                        }
                    }
                }
                VQKV_PHASE(11)
                ptx::tc_wait_st();
                if (!last) {
                    ptx::fence_async_smem();
                    ptx::tc_fence_before();
                    release(bar_aready, true);
                } else if (valid && !exact_row) {
#pragma unroll
                    for (int l = 0; l < 4; ++l) n0[l] = __fadd_rn(n0[l], n1[l]);
                    norms[grow] = __fsqrt_rn(__fadd_rn(__fadd_rn(n0[0], n0[2]), __fadd_rn(n0[1], n0[3])));
                }
                R2 = __fadd_rn(R2p.x, R2p.y);
                mx = mxn;
                sigma = sigma_n;
                VQKV_PHASE(4)
            }
        }
#undef VQKV_PHASE
#undef VQKV_PHASE_DEP
#ifdef VQKV_PHASE_CLOCKS
        if (clk_on)
            for (int k = 0; k < 13; ++k) atomicAdd(&counters[8 + k], ck[k]);
#endif
        if (counters) {
            atomicAdd(&counters[0], n_rowstages);
            if (n_amb) atomicAdd(&counters[1], n_amb);
            if (n_rs) atomicAdd(&counters[3], n_rs);
        }
    }
    __syncwarp();
    ptx::tc_fence_before();
#undef VQKV_RANK
#undef VQKV_N_ITEMS
#undef VQKV_ITEM0
#undef VQKV_ITEM_STEP
    if constexpr (kPair) {
        ptx::cluster_sync();  // the leader's last MMAs wrote the peer's TMEM
        if (warp == 2) ptx::tmem_dealloc2(tmem, 512);
    } else {
        __syncthreads();
        if (warp == 2) ptx::tmem_dealloc(tmem, 512);
    }
}

}  // namespace

// CTA-pair (cta_group::2) encoder: VQKV_ENC_PAIR=0 selects the single-CTA kernel
bool encode_pair_mode() {
    const char* e = getenv("VQKV_ENC_PAIR");
    return !(e && e[0] == '0');
}

uint32_t dbg_flags() {
    const char* e = getenv("VQKV_DBG");
    return e ? uint32_t(strtoul(e, nullptr, 0)) : 0u;
}

bool encode_tc_supported(const vqkv_stack_s& st) {
    if (st.dim != 128 || st.d_eff16 == nullptr) return false;
    for (const auto& s : st.stages) {
        if (s.pad_size > 128u * kMaxChunks * kMaxSuper) return false;
        // ||e||^2 must fit the fp16 ext column, entries the fp16 operand range
        if (!(s.max_sqnorm < 60000.f) || !(s.max_abs < 1073741824.f)) return false;
    }
    return true;
}

void launch_encode_tc(const vqkv_stack_s& st, const float* xs, uint32_t n_streams, uint64_t rows,
                      uint64_t search_block, uint8_t* payload, float* norms, float* residuals, cudaStream_t s) {
    const uint64_t total = uint64_t(n_streams) * rows;
    if (total == 0) return;
    if (total >= (1ull << 32)) fail(VQKV_UNSUPPORTED, "more than 2^32 rows per call");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st.device);
    uint16_t* codes = nullptr;
    uint32_t* list = nullptr;  // [0] = count, [1..] = rows
    VQKV_CUDA(cudaMallocAsync(&codes, sizeof(uint16_t) * total * st.n, s));
    VQKV_CUDA(cudaMallocAsync(&list, sizeof(uint32_t) * (total + 1), s));
    VQKV_CUDA(cudaMemsetAsync(list, 0, sizeof(uint32_t), s));
    // direct CodeMatrix stores from the epilogue when rows are whole 16-bit words
    bool direct = payload && st.row_bits > 0 && st.row_bits % 16 == 0 && (reinterpret_cast<uintptr_t>(payload) & 1) == 0;
    for (const auto& si : st.stages) direct = direct && si.bits <= 16;
    const uint64_t pb = payload_bytes(st.row_bits, rows);
    const uint64_t tiles = ((rows + 127) / 128) * n_streams;
    uint8_t* pay = direct ? payload : nullptr;
    const uint32_t rb = uint32_t(st.row_bits / 8);
    {
    ProfScope ps("encode_tc", s);
    bool launched = false;
    if (encode_pair_mode()) {
        // clusters of two CTAs on an SM pair, 4 tiles in flight per cluster
        const uint64_t quads = (tiles + 3) / 4;
        const unsigned clusters = unsigned(std::min<uint64_t>(quads, uint64_t(sms / 2)));
        VQKV_CUDA(cudaFuncSetAttribute(encode_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSmemBytesPair)));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * clusters);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmemBytesPair;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t le = cudaLaunchKernelEx(&cfg, encode_tc_kernel<true>, (const StageInfo*)st.d_stages, st.n,
                                                  (const __half*)st.d_eff16, (const float*)st.d_sqn_pad,
                                                  (const float*)st.d_eff, xs, n_streams, rows, search_block, codes,
                                                  norms, residuals, list + 1, list, st.d_counters, dbg_flags(), pay, pb,
                                                  rb);
        if (le == cudaSuccess) {
            launched = true;
        } else {
            // a context that cannot place SM-pair clusters (e.g. a partitioned GPU): the single-CTA
            // tensor-core kernel computes the same codes
            (void)cudaGetLastError();
        }
    }
    if (!launched) {
        const uint64_t pairs = (tiles + 1) / 2;
        const unsigned grid = unsigned(std::min<uint64_t>(pairs, uint64_t(sms)));
        // per launch: the attribute is per device, and the call is cheap (no static flag to race on)
        VQKV_CUDA(cudaFuncSetAttribute(encode_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSmemBytes)));
        encode_tc_kernel<false><<<grid, kThreads, kSmemBytes, s>>>(st.d_stages, st.n, st.d_eff16, st.d_sqn_pad, st.d_eff,
                                                                   xs, n_streams, rows, search_block, codes, norms,
                                                                   residuals, list + 1, list, st.d_counters, dbg_flags(),
                                                                   pay, pb, rb);
    }
    launch_check("encode_tc_kernel");
    }
    // rows with non-finite input: exact reference semantics
    launch_encode_exact_rows(st, xs, list + 1, list, total, search_block, codes, norms, residuals, s);
    if (direct)
        launch_pack_listed_rows(codes, list + 1, list, total, rows, st.n, st, payload, s);  // the exact rows only
    else
        launch_pack_codes(codes, n_streams, rows, st.n, st, payload, s);
    VQKV_CUDA(cudaFreeAsync(list, s));
    VQKV_CUDA(cudaFreeAsync(codes, s));
}

}  // namespace vqkv_dev
