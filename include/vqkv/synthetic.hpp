// vqkv/synthetic.hpp -- drop-in for proj/core/include/vqkv/synthetic.hpp (B200 build).
// generate() is the library's bit-identical restatement of synthetic.cpp:26-63 (vqkv_generate_synthetic:
// the same mt19937_64 / normal_distribution draws in the same order).
#pragma once

#include <cstdint>

#include "vqkv/dataset.hpp"

namespace vqkv {

enum class SyntheticKind : uint8_t {
    gaussian_mixture,
    rope_rotated_keys,  // mixture vectors rotated per position by the rotary scheme
};

struct SyntheticSpec {
    SyntheticKind kind = SyntheticKind::gaussian_mixture;
    int64_t dim = 64;
    int64_t count = 1000;
    uint32_t component_count = 8;
    uint64_t seed = 0;
    double rope_base = 10000.0;
    float component_std = 0.25f;  // within-component std; means ~ N(0, mean_scale^2 I)
    float mean_scale = 1.0f;

    void validate() const {
        if (dim < 1 || count < 1) throw InvalidInput("dim and count must be >= 1");
        if (component_count < 1) throw InvalidInput("component_count must be >= 1");
        if (kind == SyntheticKind::rope_rotated_keys && dim % 2 != 0)
            throw InvalidInput("rope_rotated_keys needs an even dimension");
        if (!(rope_base > 0.0)) throw InvalidInput("rope_base must be positive");
        if (component_std < 0.0f || mean_scale < 0.0f) throw InvalidInput("std and mean_scale must be nonnegative");
    }
};

inline VectorDataset generate(const SyntheticSpec& spec) {
    spec.validate();
    VectorDataset ds;
    ds.payload.resize(spec.count, spec.dim);
    detail::check(vqkv_generate_synthetic(int(spec.kind), uint32_t(spec.dim), uint64_t(spec.count),
                                          spec.component_count, spec.seed, spec.rope_base, spec.component_std,
                                          spec.mean_scale, ds.payload.data()));
    return ds;
}

}  // namespace vqkv
