// decode.cu -- K2: residual decode (replaces reconstruct_block / reconstruct,
// proj/core/src/codebook.cpp:208-250).
//
// out[r] = ((0 + e_0[z_0]) + e_1[z_1]) + ... in stage order, fp32 adds only:
// the same operation sequence as the reference, hence bit-exact for any
// partition of the rows.
//
// One warp per row.  Lanes extract up to 32 stage codes at a time straight
// from the CodeMatrix bit stream (only the bytes each field touches), then the
// warp walks the stages, broadcasting each code by shuffle and adding the
// selected codebook row (D = 128: one float4 per lane, 512 B coalesced gather
// per stage from the L2-resident codebook).  Output rows are written once with
// streaming stores.
#include <cstdlib>

#include "vqkv_internal.cuh"

namespace vqkv_dev {

namespace {

constexpr int kWarpsPerBlock = 8;

template <bool kD128>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
reconstruct_kernel(const StageInfo* __restrict__ stages, uint32_t n_stages, uint32_t D, uint64_t row_bits,
                   const float* __restrict__ eff, const uint8_t* __restrict__ payload, uint64_t stream_bytes,
                   uint32_t n_streams, uint64_t begin, uint64_t nrows, float* __restrict__ out,
                   int* __restrict__ err) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * kWarpsPerBlock) + (threadIdx.x >> 5);
    const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerBlock;
    const uint64_t total = uint64_t(n_streams) * nrows;
    for (uint64_t w = warp; w < total; w += nwarps) {
        const uint64_t stream = w / nrows;
        const uint64_t r = begin + (w % nrows);
        const uint8_t* pay = payload + stream * stream_bytes;
        const uint64_t rbit = r * row_bits;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float accg[4] = {0.f, 0.f, 0.f, 0.f};  // generic-D path: d = lane + 32*i (D <= 128 per pass)
        bool bad = false;
        for (uint32_t s0 = 0; s0 < n_stages; s0 += 32) {
            // lane l decodes stage s0 + l: its code and the element offset of the selected row
            uint32_t my = 0, my_off = 0;
            const uint32_t sl = s0 + lane;
            if (sl < n_stages) {
                const StageInfo si = stages[sl];
                my = read_bits(pay, rbit + si.bit_off, si.bits);
                if (my >= si.size) bad = true;
                my_off = uint32_t(si.eff_off + uint64_t(my < si.size ? my : 0u) * D);
            }
            const uint32_t cnt = (n_stages - s0 < 32) ? (n_stages - s0) : 32;
            if constexpr (kD128) {
                // kFly stage rows in flight per warp, added strictly in stage order
#ifndef VQKV_DEC_FLY
#define VQKV_DEC_FLY 8
#endif
                constexpr int kFly = VQKV_DEC_FLY;
                for (uint32_t t0 = 0; t0 < cnt; t0 += kFly) {
                    float4 v[kFly];
#pragma unroll
                    for (int u = 0; u < kFly; ++u) {
                        const uint32_t off = __shfl_sync(0xffffffffu, my_off, (t0 + u) & 31u);
                        v[u] = (t0 + u < cnt) ? __ldg(reinterpret_cast<const float4*>(eff + off) + lane)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < kFly; ++u)
                        if (t0 + u < cnt) {
                            acc.x = __fadd_rn(acc.x, v[u].x);
                            acc.y = __fadd_rn(acc.y, v[u].y);
                            acc.z = __fadd_rn(acc.z, v[u].z);
                            acc.w = __fadd_rn(acc.w, v[u].w);
                        }
                }
            } else {
                for (uint32_t t = 0; t < cnt; ++t) {
                    const uint32_t off = __shfl_sync(0xffffffffu, my_off, t);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t d = lane + 32u * i;
                        if (d < D) accg[i] = __fadd_rn(accg[i], __ldg(eff + off + d));
                    }
                }
            }
        }
        bad = __any_sync(0xffffffffu, bad);
        if (bad && lane == 0) atomicExch(err, VQKV_INVALID_CODE);
        float* o = out + w * D;
        if constexpr (kD128) {
            if (bad) acc = make_float4(NAN, NAN, NAN, NAN);
            __stcs(reinterpret_cast<float4*>(o) + lane, acc);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t d = lane + 32u * i;
                if (d < D) o[d] = bad ? NAN : accg[i];
            }
        }
    }
}

// D == 128 and at most 32 stages (the value stacks): the warp's next row's codes are read while the
// current row's stage rows are gathered, so the payload load (often from HBM) leaves the per-row chain.
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
reconstruct_few_kernel(const StageInfo* __restrict__ stages, uint32_t n_stages, uint64_t row_bits,
                       const float* __restrict__ eff, const uint8_t* __restrict__ payload, uint64_t stream_bytes,
                       uint32_t n_streams, uint64_t begin, uint64_t nrows, float* __restrict__ out,
                       int* __restrict__ err) {
    constexpr uint32_t D = 128;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * kWarpsPerBlock) + (threadIdx.x >> 5);
    const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerBlock;
    const uint64_t total = uint64_t(n_streams) * nrows;
    const bool on = lane < n_stages;
    StageInfo si{};
    if (on) si = stages[lane];
    // lane l: stage l's code of row w and the element offset of its codebook row
    auto codes_of = [&](uint64_t w, uint32_t& off, bool& bad) {
        off = 0;
        bad = false;
        if (w >= total || !on) return;
        const uint64_t stream = w / nrows, r = begin + (w % nrows);
        const uint32_t z = read_bits(payload + stream * stream_bytes, r * row_bits + si.bit_off, si.bits);
        bad = z >= si.size;
        off = uint32_t(si.eff_off + uint64_t(bad ? 0u : z) * D);
    };
    uint32_t off_n;
    bool bad_n;
    codes_of(warp, off_n, bad_n);
    for (uint64_t w = warp; w < total; w += nwarps) {
        const uint32_t my_off = off_n;
        const bool bad = __any_sync(0xffffffffu, bad_n);
        codes_of(w + nwarps, off_n, bad_n);  // the next row's codes, in flight during the gathers
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t t0 = 0; t0 < n_stages; t0 += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t off = __shfl_sync(0xffffffffu, my_off, (t0 + u) & 31u);
                v[u] = (t0 + u < n_stages) ? __ldg(reinterpret_cast<const float4*>(eff + off) + lane)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (t0 + u < n_stages) {
                    acc.x = __fadd_rn(acc.x, v[u].x);
                    acc.y = __fadd_rn(acc.y, v[u].y);
                    acc.z = __fadd_rn(acc.z, v[u].z);
                    acc.w = __fadd_rn(acc.w, v[u].w);
                }
        }
        if (bad && lane == 0) atomicExch(err, VQKV_INVALID_CODE);
        if (bad) acc = make_float4(NAN, NAN, NAN, NAN);
        __stcs(reinterpret_cast<float4*>(out + w * D) + lane, acc);
    }
}

// Generic fallback for D > 128: one thread per output element.
__global__ void reconstruct_wide_kernel(const StageInfo* __restrict__ stages, uint32_t n_stages, uint32_t D,
                                        uint64_t row_bits, const float* __restrict__ eff,
                                        const uint8_t* __restrict__ payload, uint64_t stream_bytes,
                                        uint32_t n_streams, uint64_t begin, uint64_t nrows, float* __restrict__ out,
                                        int* __restrict__ err) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(n_streams) * nrows * D) return;
    const uint64_t w = idx / D;
    const uint32_t d = uint32_t(idx % D);
    const uint64_t stream = w / nrows;
    const uint64_t r = begin + (w % nrows);
    const uint8_t* pay = payload + stream * stream_bytes;
    float acc = 0.f;
    bool bad = false;
    for (uint32_t s = 0; s < n_stages; ++s) {
        const StageInfo si = stages[s];
        uint32_t z = read_bits(pay, r * row_bits + si.bit_off, si.bits);
        if (z >= si.size) {
            bad = true;
            z = 0;
        }
        acc = __fadd_rn(acc, __ldg(eff + si.eff_off + uint64_t(z) * D + d));
    }
    if (bad) atomicExch(err, VQKV_INVALID_CODE);
    out[idx] = bad ? NAN : acc;
}

}  // namespace

void launch_reconstruct(const vqkv_stack_s& st, const uint8_t* payload, uint32_t n_streams, uint64_t rows,
                        uint64_t begin, uint64_t end, float* out, cudaStream_t s, uint64_t stream_stride) {
    const uint64_t nrows = end - begin;
    const uint64_t total = uint64_t(n_streams) * nrows;
    if (total == 0) return;
    const uint64_t sb = stream_stride ? stream_stride : payload_bytes(st.row_bits, rows);
    ProfScope ps("reconstruct", s);
    // warp-per-row kernel: 32-bit element offsets into the stage-concatenated codebook
    if (st.dim <= 128 && st.total_rows * st.dim < (1ull << 32)) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st.device);
        uint64_t blocks = (total + kWarpsPerBlock - 1) / kWarpsPerBlock;
        blocks = std::min<uint64_t>(blocks, uint64_t(sms) * 16);
        const char* fe = getenv("VQKV_DEC_FEW");  // dev A/B: 0 = the general kernel for <= 32 stages too
        if (st.dim == 128 && st.n <= 32 && !(fe && fe[0] == '0'))
            reconstruct_few_kernel<<<unsigned(blocks), kWarpsPerBlock * 32, 0, s>>>(
                st.d_stages, st.n, st.row_bits, st.d_eff, payload, sb, n_streams, begin, nrows, out, st.d_error);
        else if (st.dim == 128)
            reconstruct_kernel<true><<<unsigned(blocks), kWarpsPerBlock * 32, 0, s>>>(
                st.d_stages, st.n, st.dim, st.row_bits, st.d_eff, payload, sb, n_streams, begin, nrows, out,
                st.d_error);
        else
            reconstruct_kernel<false><<<unsigned(blocks), kWarpsPerBlock * 32, 0, s>>>(
                st.d_stages, st.n, st.dim, st.row_bits, st.d_eff, payload, sb, n_streams, begin, nrows, out,
                st.d_error);
        launch_check("reconstruct_kernel");
    } else {
        const uint64_t n = total * st.dim;
        reconstruct_wide_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(
            st.d_stages, st.n, st.dim, st.row_bits, st.d_eff, payload, sb, n_streams, begin, nrows, out, st.d_error);
        launch_check("reconstruct_wide_kernel");
    }
}

}  // namespace vqkv_dev
