// nccl_combine.cpp -- the one exchange step of a sequence-split decode attention (configs[4]):
// every rank attends its contiguous token shard and holds a partial (o, lse) for the same rows
// (query heads); one NCCL all-gather of those partials, then the identical LSE merge on every rank
// (vqkv_lse_combine).  Reference: attend's online softmax (proj/core/src/attention.cpp:45-66) is
// associative over token blocks, which is what the merge restates across ranks.
//
// NCCL is loaded on first use (dlopen of libnccl.so.2: the system NCCL, or the one already mapped into
// the process, e.g. by torch.distributed), so the library itself carries no NCCL link dependency.
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "vqkv_internal.cuh"

namespace {

// the NCCL ABI subset used here (nccl.h: ncclResult_t is an int enum, ncclComm_t an opaque pointer)
typedef int nccl_result_t;
typedef void* nccl_comm_t;
enum { kNcclFloat32 = 7 };  // ncclFloat32 / ncclFloat
struct NcclApi {
    nccl_result_t (*all_gather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*group_start)() = nullptr;
    nccl_result_t (*group_end)() = nullptr;
    nccl_result_t (*comm_init_all)(nccl_comm_t*, int, const int*) = nullptr;
    nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
    nccl_result_t (*comm_count)(nccl_comm_t, int*) = nullptr;
    const char* (*error_string)(nccl_result_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + n;
            return p;
        };
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
        api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
        api.comm_count = reinterpret_cast<decltype(api.comm_count)>(sym("ncclCommCount"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    });
    if (!api.error.empty()) vqkv_dev::fail(VQKV_CUDA_ERROR, api.error);
    return api;
}

void nccl_check(nccl_result_t r, const char* what) {
    if (r != 0) vqkv_dev::fail(VQKV_CUDA_ERROR, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

namespace vqkv_dev {

void nccl_comm_init_all(int ndev, const int* devs, void** comms) {
    nccl_check(nccl().comm_init_all(reinterpret_cast<nccl_comm_t*>(comms), ndev, devs), "ncclCommInitAll");
}

void nccl_comm_destroy(void* comm) { nccl_check(nccl().comm_destroy(comm), "ncclCommDestroy"); }

void lse_allgather_combine(void* comm, const float* part_o, const float* part_lse, uint64_t rows, uint32_t dv,
                           float* gather_o, float* gather_lse, float* out, float* out_lse, cudaStream_t s) {
    const NcclApi& api = nccl();
    int world = 0;
    nccl_check(api.comm_count(comm, &world), "ncclCommCount");
    float *go = gather_o, *gl = gather_lse;
    if (!go) VQKV_CUDA(cudaMallocAsync(&go, sizeof(float) * uint64_t(world) * rows * dv, s));
    if (!gl) VQKV_CUDA(cudaMallocAsync(&gl, sizeof(float) * uint64_t(world) * rows, s));
    nccl_check(api.group_start(), "ncclGroupStart");
    nccl_check(api.all_gather(part_o, go, rows * dv, kNcclFloat32, comm, s), "ncclAllGather(o)");
    nccl_check(api.all_gather(part_lse, gl, rows, kNcclFloat32, comm, s), "ncclAllGather(lse)");
    nccl_check(api.group_end(), "ncclGroupEnd");
    launch_lse_combine(go, gl, uint32_t(world), rows, dv, out, out_lse, s);  // rank-major: [world][rows][dv]
    if (!gather_o) VQKV_CUDA(cudaFreeAsync(go, s));
    if (!gather_lse) VQKV_CUDA(cudaFreeAsync(gl, s));
}

}  // namespace vqkv_dev
