// Microbenchmark: shared-memory histogram update throughput on B200.
// modes: 0 = int32 atomicAdd (4 per item), 1 = float atomicAdd (CAS loop, 4 per item),
//        2 = float4 LDS+STS RMW (racy, bandwidth only), 3 = float LDS lookup float4 (LUT gather)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(int mode, int iters, uint32_t* out) {
  extern __shared__ uint32_t h[];  // 8192 bins x 4
  for (int i = threadIdx.x; i < 8192 * 4; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t b = (x >> 13) & 8191u;
    if (mode == 0) {
      atomicAdd(&h[4 * b + 0], x & 255u); atomicAdd(&h[4 * b + 1], 1u);
      atomicAdd(&h[4 * b + 2], 2u); atomicAdd(&h[4 * b + 3], 3u);
    } else if (mode == 1) {
      float* f = reinterpret_cast<float*>(h);
      atomicAdd(&f[4 * b + 0], 1.f); atomicAdd(&f[4 * b + 1], 1.f);
      atomicAdd(&f[4 * b + 2], 1.f); atomicAdd(&f[4 * b + 3], 1.f);
    } else if (mode == 2) {
      float4* f = reinterpret_cast<float4*>(h);
      float4 v = f[b]; v.x += 1.f; v.y += 1.f; v.z += 1.f; v.w += 1.f; f[b] = v;
    } else {
      float4 v = reinterpret_cast<float4*>(h)[b];
      acc += v.x + v.y + v.z + v.w;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[5] + (uint32_t)acc;
}
int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"int32 atomicAdd x4", "float atomicAdd x4 (CAS)", "float4 LDS+STS RMW", "float4 LDS gather"};
  for (int mode = 0; mode < 4; ++mode) for (int thr : {256, 512, 1024}) {
    int iters = 2000;
    k<<<sms, thr, 8192 * 16>>>(mode, 10, out);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, thr, 8192 * 16>>>(mode, iters, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double items = double(sms) * thr * iters;
    printf("%-26s thr=%4d: %.3f ms, %.1f G items/s, %.2f items/clk/SM (at 1.9GHz)\n", names[mode], thr, ms,
           items / ms / 1e6, items / (ms * 1e-3) / sms / 1.9e9);
  }
  return 0;
}
