// prints the shared-window address of dynamic shared memory (dev aid)
#include <cstdio>
extern "C" __global__ void k(unsigned* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned a;
    asm("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(sm));
    if (threadIdx.x == 0) out[0] = a;
}
int main() {
    unsigned* d; unsigned h;
    cudaMalloc(&d, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    k<<<1, 32, 140000>>>(d);
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("dynamic smem window address: 0x%x\n", h);
    return 0;
}
