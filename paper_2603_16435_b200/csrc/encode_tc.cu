// encode_tc.cu -- K1 placeholder (tensor-core encoder lands in a later commit).
#include "vqkv_internal.cuh"

namespace vqkv_dev {

bool encode_tc_supported(const vqkv_stack_s&) { return false; }

void launch_encode_tc(const vqkv_stack_s&, const float*, uint32_t, uint64_t, uint64_t, uint8_t*, float*,
                      float*, cudaStream_t) {
    fail(VQKV_UNSUPPORTED, "tensor-core encoder not built");
}

}  // namespace vqkv_dev
