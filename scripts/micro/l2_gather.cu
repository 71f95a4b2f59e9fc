// Microbenchmark: L2 -> SM bandwidth for (a) random 512 B row gathers with 256-bit
// L1-bypassing loads (thread per row, like the encoder's e_z gather) and (b) bulk
// async copies of contiguous 36 KB chunks into smem (like the codebook chunk stream).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather l2_gather.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_2603_16435_b200/csrc/tc_ptx.cuh"
using namespace vqkv_dev;

__global__ void gather(const float* __restrict__ tab, uint32_t rows, int iters, float* out) {
    uint32_t h = blockIdx.x * 1315423911u + threadIdx.x * 2654435761u;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        h = h * 1664525u + 1013904223u;
        const float* p = tab + uint64_t(h % rows) * 128;
        float v[128];
#pragma unroll
        for (int k = 0; k < 16; ++k) ptx::ldg256_na(p + 8 * k, v + 8 * k);
#pragma unroll
        for (int k = 0; k < 128; ++k) acc += v[k];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void bulk(const uint8_t* __restrict__ src, uint64_t chunks, int iters, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&bar[1]), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const uint32_t b = it & 1;
            if (it >= 2) ptx::mbar_wait(ptx::smem_u32(&bar[b]), ((it - 2) >> 1) & 1);
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar[b]), 36864);
            const uint64_t c = (uint64_t(blockIdx.x) * 7919 + it) % chunks;
            ptx::bulk_g2s(ptx::smem_u32(sm + b * 36864), src + c * 36864, 36864, ptx::smem_u32(&bar[b]));
        }
        for (int it = iters - 2; it < iters; ++it) ptx::mbar_wait(ptx::smem_u32(&bar[it & 1]), (it >> 1) & 1);
        out[blockIdx.x] = float(sm[threadIdx.x]);
    }
}

int main() {
    const uint32_t rows = 32768;  // 16 MB fp32 table, L2 resident
    float *tab, *out;
    cudaMalloc(&tab, size_t(rows) * 512);
    cudaMemset(tab, 0, size_t(rows) * 512);
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int warps : {4, 8, 16}) {
        const int iters = 200;
        gather<<<148, warps * 32>>>(tab, rows, 10, out);
        cudaEventRecord(a);
        gather<<<148, warps * 32>>>(tab, rows, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double bytes = 148.0 * warps * 32 * iters * 512;
        printf("gather 512B rows, %2d warps/SM: %.1f TB/s, %.1f B/clk/SM @1.9GHz\n", warps, bytes / ms / 1e9,
               bytes / ms / 1e-3 / 148 / 1.9e9);
    }
    uint8_t* src; cudaMalloc(&src, 36864ull * 512); cudaMemset(src, 1, 36864ull * 512);  // 18 MB of chunks
    cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 36864);
    for (int ctas : {148, 296}) {
        const int iters = 400;
        bulk<<<ctas, 32, 2 * 36864>>>(src, 512, 10, out);
        cudaEventRecord(a);
        bulk<<<ctas, 32, 2 * 36864>>>(src, 512, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double bytes = double(ctas) * iters * 36864;
        printf("bulk 36 KB chunks, %d CTAs (2 in flight each): %.1f TB/s, %.1f B/clk/SM\n", ctas, bytes / ms / 1e9,
               bytes / ms / 1e-3 / 148 / 1.9e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
