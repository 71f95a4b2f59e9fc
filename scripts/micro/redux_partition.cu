// Does redux.sync with per-partition member masks (from match.any) reduce each partition separately?
#include <cstdio>
__global__ void k(unsigned* out) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned owner = lane / 5;                  // contiguous groups of 5 lanes
    const unsigned val = (lane * 2654435761u) >> 8;
    const unsigned grp = __match_any_sync(0xffffffffu, owner);
    out[lane] = __reduce_min_sync(grp, val);
    out[32 + lane] = grp;
}
int main() {
    unsigned* d; cudaMalloc(&d, 64 * 4); k<<<1, 32>>>(d);
    unsigned h[64]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int l = 0; l < 32; ++l) {
        unsigned m = 0xffffffffu;
        for (int j = 0; j < 32; ++j) if (j / 5 == l / 5) { unsigned v = (unsigned(j) * 2654435761u) >> 8; if (v < m) m = v; }
        if (h[l] != m) ++bad;
    }
    printf("partitioned redux: %s\n", bad ? "MISMATCH" : "ok");
    return bad != 0;
}
