#pragma once
// Drop-in for /root/reference/proj/include/neuzip/crc32.hpp (crc32.hpp:1-45):
// CRC-32 (IEEE 802.3, reflected 0xEDB88320) with the same Crc32 / crc32 API.
// The bytes are checksummed on the B200 (nzgpu_crc32_host); successive
// update() calls are joined on the host with GF(2) arithmetic:
//   raw(A || B) = raw(A) * x^(8|B|) mod P  xor  raw(B)
// where raw is the register value started from 0 without the final xor.

#include <cstdint>
#include <span>

#include "neuzip/errors.hpp"

namespace neuzip {

namespace detail {
// a * b mod P, reflected representation (x^0 = bit 31)
inline std::uint32_t gf2_mulmod(std::uint32_t a, std::uint32_t b) {
    std::uint32_t p = 0;
    for (std::uint32_t m = 1u << 31; m; m >>= 1) {
        if (a & m) p ^= b;
        b = (b & 1u) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}
// x^(8n) mod P
inline std::uint32_t gf2_x8n(std::uint64_t n) {
    std::uint32_t r = 1u << 31, sq = 1u << 23;
    for (; n; n >>= 1) {
        if (n & 1) r = gf2_mulmod(sq, r);
        sq = gf2_mulmod(sq, sq);
    }
    return r;
}
}  // namespace detail

/// Incremental CRC-32 accumulator (crc32.hpp:26-36).
class Crc32 {
public:
    void update(std::span<const std::uint8_t> data) {
        if (data.empty()) return;
        std::uint32_t c = 0;
        detail::check(nzgpu_crc32_host(data.data(), data.size(), &c), "crc32");
        // finalized crc of `data` -> raw, then join onto the running raw value
        const std::uint32_t init = detail::gf2_mulmod(detail::gf2_x8n(data.size()), 0xFFFFFFFFu);
        const std::uint32_t raw = c ^ 0xFFFFFFFFu ^ init;
        raw_ = detail::gf2_mulmod(detail::gf2_x8n(data.size()), raw_) ^ raw;
        len_ += data.size();
    }
    std::uint32_t value() const {
        return raw_ ^ detail::gf2_mulmod(detail::gf2_x8n(len_), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
    }

private:
    std::uint32_t raw_ = 0;
    std::uint64_t len_ = 0;
};

/// crc32.hpp:38-42
inline std::uint32_t crc32(std::span<const std::uint8_t> data) {
    Crc32 crc;
    crc.update(data);
    return crc.value();
}

}  // namespace neuzip
