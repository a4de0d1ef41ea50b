// decode_common.cuh -- helpers shared by the decode kernels.
#pragma once
#include "nzgpu_internal.cuh"

#ifndef NZ_CHAINS
#define NZ_CHAINS 2
#endif

namespace nzgpu {

constexpr int kDecodeThreads = 128;       // threads per decode CTA
constexpr int kChains = NZ_CHAINS;        // interleaved sub-ranges (ANS lanes) per thread
constexpr int kTileSubs = kDecodeThreads * kChains;
constexpr uint32_t kLutBytes = 4096 * 4;
constexpr uint32_t kSmemHeader = 128;

__host__ __device__ constexpr uint32_t exps_row_words(int log2k) { return (1u << log2k) / 4 + 1; }

// Dynamic shared memory of one decode CTA: header | LUT | exponent tile
// (one padded row per sub-range) | payload window (+ overrun slack).
__host__ __device__ constexpr uint32_t decode_smem_bytes(int log2k, uint32_t win_cap) {
    return kSmemHeader + kLutBytes + kTileSubs * exps_row_words(log2k) * 4 + win_cap + 2 * (1u << log2k) + 64;
}

__device__ __forceinline__ uint64_t chunk_offset(uint4 ci) { return (uint64_t)ci.x | ((uint64_t)ci.y << 32); }

// Sub-range j -> (chunk, index within chunk).  Sub-range indices are 32-bit
// (the host rejects tensors with >= 2^32 sub-ranges); S/K is usually a
// power of two (65536/128), which turns the division into shifts.
__device__ __forceinline__ void sub_to_chunk(const DecodeDesc& d, int log2k, uint32_t j, uint32_t& ch, uint32_t& jin) {
    if (d.log2_spc != 0xFFFFFFFFu) {
        ch = j >> d.log2_spc;
        jin = j & ((1u << d.log2_spc) - 1u);
    } else {
        const uint32_t spc = d.chunk_syms >> log2k;
        ch = j / spc;
        jin = j - ch * spc;
    }
}

// Absolute stream window [a, b) of renormalisation bytes a tile reads.
__device__ __forceinline__ void tile_window(const DecodeDesc& d, uint32_t sub0, uint32_t tile_subs, int log2k,
                                            uint32_t nsub, uint64_t& a, uint64_t& b) {
    uint32_t c0, j0in, c1, jlin;
    sub_to_chunk(d, log2k, sub0, c0, j0in);
    const uint4 ci0 = d.chunk_info[c0];
    const uint32_t lim0 = ci0.z >= 4 ? ci0.z - 4 : 0;
    const uint32_t e0 = j0in == 0 ? lim0 : min(d.ckpt[sub0].y, lim0);
    a = chunk_offset(ci0) + lim0 - e0;
    const uint32_t jl = sub0 + tile_subs - 1;
    sub_to_chunk(d, log2k, jl, c1, jlin);
    const uint4 ci1 = d.chunk_info[c1];
    const uint32_t lim1 = ci1.z >= 4 ? ci1.z - 4 : 0;
    const uint32_t jn = jl + 1;
    const bool chunk_end = ((uint64_t)(jlin + 1) << log2k) >= ci1.w;
    const uint32_t e1 = (jn < nsub && !chunk_end) ? min(d.ckpt[jn].y, lim1) : 0;
    b = chunk_offset(ci1) + lim1 - e1;
    if (b < a) b = a;
}

// Two bf16 from two exponent bytes and two sign/mantissa bytes packed as
// Y = e<<8 | s<<7 | m per 16-bit lane  ->  s<<15 | e<<7 | m
// (merge, bitfloat.hpp:64-71, on the tensorstore.hpp:119-123 fields).
__device__ __forceinline__ uint32_t assemble2(uint32_t y) {
    return ((y >> 1) & 0x7F807F80u) | (y & 0x007F007Fu) | ((y << 8) & 0x80008000u);
}

__device__ __forceinline__ uint4 merge8(uint32_t e4a, uint32_t s4a, uint32_t e4b, uint32_t s4b) {
    uint4 o;
    o.x = assemble2(__byte_perm(s4a, e4a, 0x5140));
    o.y = assemble2(__byte_perm(s4a, e4a, 0x7362));
    o.z = assemble2(__byte_perm(s4b, e4b, 0x5140));
    o.w = assemble2(__byte_perm(s4b, e4b, 0x7362));
    return o;
}

// decompress_lossy element (tensorstore.hpp:229-236) in exact FP32
// (correctly rounded multiply == the reference's double path, probe P5).
__device__ __forceinline__ uint16_t lossy_rebuild(uint32_t item, uint32_t e, int k, float c) {
    const uint32_t sgn = item >> k;
    const uint32_t m = item & ((1u << k) - 1u);
    const uint32_t normalized = (sgn << 15) | (e << 7) | (m << (7 - k));
    return bf16_from_float(__fmul_rn(__uint_as_float(normalized << 16), c));
}

__device__ __forceinline__ float scale_coef(uint32_t s) { return 1.0f + (float)s * (1.0f / 128.0f); }

// (k+1)-bit item i of a packed MSB-first stream (bitfloat.hpp:156-162).
__device__ __forceinline__ uint32_t packed_item(const uint8_t* packed, uint64_t i, int k) {
    const uint32_t width = (uint32_t)k + 1;
    const uint64_t bit = i * width;
    const uint32_t shift = 8 - width - (uint32_t)(bit & 7);
    return ((uint32_t)__ldg(packed + (bit >> 3)) >> shift) & ((1u << width) - 1u);
}

}  // namespace nzgpu
