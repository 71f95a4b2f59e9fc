// vqkv/bitpack.hpp -- drop-in for proj/core/include/vqkv/bitpack.hpp:14-45.
//
// Layout contract (shared with the device kernels and the CodeMatrix payload):
// LSB-first little-endian bit stream -- bit k of a field stored at absolute
// bit position p lands in byte p/8, bit p%8.  Fields up to 32 bits wide.
// Implemented byte-wise (whole bytes masked at once) rather than bit by bit.
#pragma once

#include <cstdint>
#include <vector>

namespace vqkv {

/// Stores the low `width` bits of `value` at bit offset `bit_pos`, growing the
/// buffer with zero bytes as needed; other bits of touched bytes are preserved.
inline void bit_write(std::vector<uint8_t>& buf, size_t bit_pos, uint32_t value, unsigned width) {
    if (width == 0) return;
    const size_t last = (bit_pos + width - 1) >> 3;
    if (buf.size() <= last) buf.resize(last + 1, 0);
    uint64_t field = (width >= 32 ? uint64_t(value) : (uint64_t(value) & ((uint64_t(1) << width) - 1)))
                     << (bit_pos & 7);
    uint64_t mask = (width >= 64 ? ~uint64_t(0) : ((uint64_t(1) << width) - 1)) << (bit_pos & 7);
    for (size_t i = bit_pos >> 3; i <= last; ++i, field >>= 8, mask >>= 8)
        buf[i] = uint8_t((buf[i] & ~uint8_t(mask)) | uint8_t(field));
}

/// Reads a `width`-bit field at bit offset `bit_pos`.
inline uint32_t bit_read(const std::vector<uint8_t>& buf, size_t bit_pos, unsigned width) {
    if (width == 0) return 0;
    const size_t first = bit_pos >> 3, last = (bit_pos + width - 1) >> 3;
    uint64_t acc = 0;
    for (size_t i = last + 1; i-- > first;) acc = (acc << 8) | buf[i];
    acc >>= (bit_pos & 7);
    return uint32_t(width >= 32 ? acc : (acc & ((uint64_t(1) << width) - 1)));
}

/// ceil(log2(size)); 0 for size <= 1.
inline unsigned index_bit_width(uint32_t size) {
    return size <= 1 ? 0u : unsigned(32 - __builtin_clz(size - 1));
}

}  // namespace vqkv
