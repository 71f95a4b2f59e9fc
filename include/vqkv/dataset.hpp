// vqkv/dataset.hpp -- drop-in for proj/core/include/vqkv/dataset.hpp (B200 build).
//
// The "VECD" container of a flat corpus of D-dimensional fp32 vectors (dataset.cpp:11-69):
//   "VECD", u32 version = 1, u32 D, u64 count, count x D fp32 row-major.
// Host-side I/O only; the same errors as the reference (IoError, FormatError with the byte offset,
// InvalidInput for empty or non-finite data).
#pragma once

#include <cmath>
#include <cstdint>
#include <fstream>
#include <string>

#include "vqkv/codebook.hpp"

namespace vqkv {

struct VectorDataset {
    MatrixF payload;  // count x D

    int64_t dim() const { return payload.cols(); }
    int64_t count() const { return payload.rows(); }

    void validate() const {
        if (count() < 1 || dim() < 1) throw InvalidInput("dataset must have count >= 1 and D >= 1");
        for (int64_t i = 0; i < payload.size(); ++i)
            if (!std::isfinite(payload.data()[i])) throw InvalidInput("dataset contains non-finite values");
    }
};

inline void save_dataset(const VectorDataset& dataset, const std::string& path) {
    dataset.validate();
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path + " for writing");
    const uint32_t version = 1, d = uint32_t(dataset.dim());
    const uint64_t count = uint64_t(dataset.count());
    out.write("VECD", 4);
    out.write(reinterpret_cast<const char*>(&version), 4);
    out.write(reinterpret_cast<const char*>(&d), 4);
    out.write(reinterpret_cast<const char*>(&count), 8);
    out.write(reinterpret_cast<const char*>(dataset.payload.data()), std::streamsize(sizeof(float) * dataset.payload.size()));
    if (!out) throw IoError("write failed for " + path);
}

inline VectorDataset load_dataset(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    size_t off = 0;
    auto read = [&](void* p, size_t n, const char* what) {
        in.read(reinterpret_cast<char*>(p), std::streamsize(n));
        if (size_t(in.gcount()) != n) throw FormatError(std::string("truncated ") + what, off + size_t(in.gcount()));
        off += n;
    };
    char magic[4];
    read(magic, 4, "magic");
    if (std::string(magic, 4) != "VECD") throw FormatError("bad magic", 0);
    uint32_t version = 0, d = 0;
    uint64_t count = 0;
    read(&version, 4, "version");
    if (version != 1) throw FormatError("unsupported version " + std::to_string(version), off - 4);
    read(&d, 4, "dimension");
    read(&count, 8, "count");
    if (d < 1 || count < 1) throw FormatError("dimension and count must be >= 1", off - 12);
    VectorDataset ds;
    ds.payload.resize(int64_t(count), int64_t(d));
    const size_t data_off = off;
    read(ds.payload.data(), sizeof(float) * size_t(ds.payload.size()), "vector payload");
    for (int64_t i = 0; i < ds.payload.size(); ++i)
        if (!std::isfinite(ds.payload.data()[i])) throw FormatError("non-finite vector data", data_off);
    return ds;
}

}  // namespace vqkv
