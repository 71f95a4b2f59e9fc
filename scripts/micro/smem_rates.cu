// Microbenchmark: shared-memory instruction rates that bound the decode-attention kernel (K3).
// Reports warp-instructions per clock per SM for:
//   0 ATOMS.ADD u32, random bins (lane = token, [stage][head][code] histogram, S = 512)
//   1 ATOMS.ADD u32, conflict-free (lane = (slot, head): bank = 4*slot + head)
//   2 LDS.128 conflict-free rotated gather (8 lanes of a quarter-warp hit 8 distinct 16 B groups)
//   3 LDS.64 conflict-free rotated gather (16 lanes of a half-warp hit 16 distinct 8 B groups)
//   4 LDS.32 random
//   5 ATOMS.ADD u64, random bins (two heads' fixed-point weights packed in one 64-bit word)
//   6 LDS.128 rotated gather feeding two FADD2 each (the K3 key loop's shape)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_rates smem_rates.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <int mode>
__global__ void k(int iters, uint32_t* out, long long* clk) {
  extern __shared__ uint32_t h[];  // 128 KB
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) h[i] = i;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x * 97u + 12345u;
  uint32_t acc = 0;
  float2 fl[8];
  for (int i = 0; i < 8; ++i) fl[i] = make_float2(0.f, 0.f);
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(h);
  // addresses precomputed; the loop only flips a bit pattern per iteration (1 LOP per op)
  uint32_t ad[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    x = x * 1664525u + 1013904223u;
    const uint32_t c = (x >> 13) & 511u;
    // offsets (the per-iteration flip is applied before adding the window base: stays in bounds)
    if (mode == 0) ad[u] = 4u * ((u & 3u) * 512u + c);
    else if (mode == 1) ad[u] = 4u * (c * 32u + lane);
    else if (mode == 2 || mode == 6) ad[u] = ((c * 2u) << 7) + ((((lane & 7u) ^ u)) << 4);
    else if (mode == 3) ad[u] = ((c * 2u) << 7) + ((((lane & 15u) ^ u)) << 3);
    else if (mode == 4) ad[u] = 4u * ((x >> 3) & 32767u);
    else ad[u] = 8u * ((u & 3u) * 512u + c);
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t flip = (it & 63u) << 8;  // whole 256 B rows: keeps the bank pattern
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t a = base + (ad[u] ^ flip);
      if (mode <= 1) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(x) : "memory");
      } else if (mode == 5) {
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"((unsigned long long)x) : "memory");
      } else if (mode == 2) {
        uint32_t a0, a1, a2, a3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(a));
        acc += a0 ^ a1 ^ a2 ^ a3;
      } else if (mode == 6) {  // the K3 key loop's shape: LDS.128 of 4 heads' fp32 slots, two FADD2 per lookup
        float2 p0, p1;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(p0.x), "=f"(p0.y), "=f"(p1.x), "=f"(p1.y) : "r"(a));
        float2& L0 = fl[(u & 3) * 2], &L1 = fl[(u & 3) * 2 + 1];
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&L0))
            : "l"(*reinterpret_cast<unsigned long long*>(&L0)), "l"(*reinterpret_cast<unsigned long long*>(&p0)));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&L1))
            : "l"(*reinterpret_cast<unsigned long long*>(&L1)), "l"(*reinterpret_cast<unsigned long long*>(&p1)));
      } else if (mode == 3) {
        uint32_t a0, a1;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a0), "=r"(a1) : "r"(a));
        acc += a0 ^ a1;
      } else {
        uint32_t a0;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a0) : "r"(a));
        acc += a0;
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  for (int i = 0; i < 8; ++i) acc += __float_as_uint(fl[i].x) ^ __float_as_uint(fl[i].y);
  if (threadIdx.x == 0) { out[blockIdx.x] = h[5] + acc; clk[blockIdx.x] = t1 - t0; }
  else if (acc == 0xdeadbeef) out[0] = acc;
}
int main() {
  uint32_t* out; long long* clk;
  cudaMalloc(&out, 4096 * 4); cudaMalloc(&clk, 4096 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"ATOMS u32 random bins", "ATOMS u32 conflict-free", "LDS.128 rotated", "LDS.64 rotated",
                         "LDS.32 random", "ATOMS u64 random bins", "LDS.128 rotated + FADD2"};
  void (*fn[7])(int, uint32_t*, long long*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  for (int mode : {5, 0, 1, 2, 3, 4, 6}) {
    cudaFuncSetAttribute(fn[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int thr : {256, 512, 1024}) {
      const int iters = 4000;
      fn[mode]<<<sms, thr, 131072>>>(10, out, clk);
      fn[mode]<<<sms, thr, 131072>>>(iters, out, clk);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double winst = double(thr / 32) * iters * 8;
      printf("%-24s thr=%4d: %.3f warp-instr/clk/SM (%lld clk)\n", names[mode], thr, winst / c, c);
    }
  }
  return 0;
}
