// host_synthetic.cpp -- product-side restatement of the reference fixtures that
// define "the same synthetic inputs" (host C++, part of libvqkv_b200.so):
//   generate()        proj/core/src/synthetic.cpp:26-63
//   random_stack()    proj/tests/test_util.hpp:30-50
// Both use libstdc++'s std::mt19937_64 + std::normal_distribution<float>, so the
// values are bit-identical to the reference's for the same seeds.  Also the
// FNV-1a-64 used by stack_content_hash (codebook.cpp:326-336).
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "vqkv_c.h"

namespace {

void rope_rotate_row(float* row, int64_t d, int64_t position, double base) {
    for (int64_t i = 0; i < d / 2; ++i) {
        double freq = std::pow(base, -2.0 * double(i) / double(d));
        double angle = double(position) * freq;
        float c = float(std::cos(angle));
        float s = float(std::sin(angle));
        float a = row[2 * i], b = row[2 * i + 1];
        row[2 * i] = a * c - b * s;
        row[2 * i + 1] = a * s + b * c;
    }
}

}  // namespace

extern "C" {

int vqkv_generate_synthetic(int kind, uint32_t dim, uint64_t count, uint32_t comps, uint64_t seed, double base,
                            float cstd, float mscale, float* out) {
    if (dim < 1 || count < 1 || comps < 1) return VQKV_INVALID_INPUT;
    if (kind == 1 && dim % 2 != 0) return VQKV_INVALID_INPUT;
    if (!(base > 0.0) || cstd < 0.0f || mscale < 0.0f) return VQKV_INVALID_INPUT;
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    std::uniform_int_distribution<uint32_t> pick(0, comps - 1);
    std::vector<float> means(size_t(comps) * dim);
    for (auto& m : means) m = mscale * gauss(rng);
    for (uint64_t r = 0; r < count; ++r) {
        uint32_t c = pick(rng);
        float* row = out + r * dim;
        for (uint32_t j = 0; j < dim; ++j) row[j] = means[size_t(c) * dim + j] + cstd * gauss(rng);
        if (kind == 1) rope_rotate_row(row, dim, int64_t(r), base);
    }
    return VQKV_OK;
}

int vqkv_random_stack(uint64_t seed, uint32_t n_stages, uint32_t size, uint32_t dim, float* entries, float* projections) {
    if (n_stages < 1 || size < 1 || dim < 1) return VQKV_INVALID_INPUT;
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    const float proj_scale = 1.0f / std::sqrt(static_cast<float>(dim));
    for (uint32_t s = 0; s < n_stages; ++s) {
        float* e = entries + uint64_t(s) * size * dim;
        for (uint64_t i = 0; i < uint64_t(size) * dim; ++i) e[i] = gauss(rng);
        float* p = projections + uint64_t(s) * dim * dim;
        for (uint64_t i = 0; i < uint64_t(dim) * dim; ++i) p[i] = proj_scale * gauss(rng);
    }
    return VQKV_OK;
}

uint64_t vqkv_fnv1a64(const uint8_t* data, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= data[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

}  // extern "C"
