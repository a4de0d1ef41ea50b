// decode_common.cuh -- helpers shared by the decode kernels.
#pragma once
#include "nzgpu_internal.cuh"

#ifndef NZ_CHAINS
#define NZ_CHAINS 1
#endif

namespace nzgpu {

#ifndef NZ_WINDOW
#define NZ_WINDOW 1  // renormalisation bytes from a per-lane register window
#endif

#ifndef NZ_MINBLOCKS
#define NZ_MINBLOCKS 1
#endif

#ifndef NZ_PF
#define NZ_PF 8  // 8-element groups of the mantissa plane prefetched into registers
#endif

#ifndef NZ_THREADS
#define NZ_THREADS 256
#endif

constexpr int kDecodeThreads = NZ_THREADS;  // threads per decode CTA
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

// Four bf16 from four exponent bytes E and four sign/mantissa bytes S
// (merge, bitfloat.hpp:64-71, on the tensorstore.hpp:119-123 fields):
// bf16 = s<<15 | e<<7 | m has high byte s<<7 | e>>1 and low byte
// (e&1)<<7 | m, so build all four high bytes and all four low bytes with
// one shift + one LOP3 each, then interleave them with two PRMTs.
__device__ __forceinline__ uint2 merge4(uint32_t e4, uint32_t s4) {
    const uint32_t hi = ((e4 >> 1) & 0x7F7F7F7Fu) | (s4 & 0x80808080u);
    const uint32_t lo = ((e4 << 7) & 0x80808080u) | (s4 & 0x7F7F7F7Fu);
    return make_uint2(__byte_perm(lo, hi, 0x5140), __byte_perm(lo, hi, 0x7362));
}

__device__ __forceinline__ uint4 merge8(uint32_t e4a, uint32_t s4a, uint32_t e4b, uint32_t s4b) {
    const uint2 a = merge4(e4a, s4a), b = merge4(e4b, s4b);
    return make_uint4(a.x, a.y, b.x, b.y);
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
