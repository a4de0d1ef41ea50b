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

// Absolute stream window [a, b) of the renormalisation bytes that sub-ranges
// [sub0, sub0 + subs) read, for sub0 a multiple of 32 (a unit start) and
// sub0 + subs a multiple of 32 or nsub: it starts at sub-range sub0's
// position and ends where the next unit starts (when that unit begins inside
// the last sub-range's chunk) or at that chunk's end.  O(1) in the index.
__device__ __forceinline__ void tile_window(const DecodeDesc& d, uint32_t sub0, uint32_t subs, int log2k,
                                            uint32_t nsub, uint64_t& a, uint64_t& b) {
    uint32_t c0, j0in, c1, jlin;
    sub_to_chunk(d, log2k, sub0, c0, j0in);
    const uint4 ci0 = d.chunk_info[c0];
    const uint32_t lim0 = ci0.z >= 4 ? ci0.z - 4 : 0;
    a = chunk_offset(ci0) + (j0in == 0 ? 0u : min(d.ck_base[sub0 >> 5], lim0));
    const uint32_t jl = sub0 + subs - 1, jn = jl + 1;
    sub_to_chunk(d, log2k, jl, c1, jlin);
    const uint4 ci1 = d.chunk_info[c1];
    const uint32_t lim1 = ci1.z >= 4 ? ci1.z - 4 : 0;
    const bool chunk_end = ((uint64_t)(jlin + 1) << log2k) >= ci1.w;
    b = chunk_offset(ci1) + ((jn < nsub && !chunk_end) ? min(d.ck_base[jn >> 5], lim1) : lim1);
    if (b < a) b = a;
}

// bitwise c ? a : b in one LOP3
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// Four bf16 from four exponent bytes E and four sign/mantissa bytes S
// (merge, bitfloat.hpp:64-71, on the tensorstore.hpp:119-123 fields):
// bf16 = s<<15 | e<<7 | m has high byte s<<7 | e>>1 and low byte
// (e&1)<<7 | m, so build all four high bytes and all four low bytes with
// one shift + one bit-select LOP3 each, then interleave them with two PRMTs.
__device__ __forceinline__ uint2 merge4(uint32_t e4, uint32_t s4) {
    const uint32_t hi = bitsel(e4 >> 1, s4, 0x7F7F7F7Fu);
    const uint32_t lo = bitsel(e4 << 7, s4, 0x80808080u);
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
    // Inf * c stays Inf; a NaN keeps its payload with the quiet bit set (what
    // the reference's double multiply does on the host, where the GPU would
    // return the canonical NaN).
    if (e == 255) return (uint16_t)(m ? normalized | 0x40u : normalized);
    return bf16_from_float(__fmul_rn(__uint_as_float(normalized << 16), c));
}

__device__ __forceinline__ float scale_coef(uint32_t s) { return 1.0f + (float)s * (1.0f / 128.0f); }

// Two bf16 lanes times two bf16 lanes, one correctly rounded (RNE) multiply.
__device__ __forceinline__ uint32_t bf16x2_mul(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// The lossy block coefficient 1 + s/128 (tensorstore.hpp:231) is exactly the
// bf16 with exponent 127 and mantissa s: 0x3F80 | s.
__device__ __forceinline__ uint32_t scale_coef_bf16(uint32_t s) { return 0x3F80u | s; }

// Eight lossy elements (decompress_lossy, tensorstore.hpp:229-236) on the
// bf16x2 pipe.  The reference multiplies the normalized bf16 (8 significant
// bits) by c (8 significant bits) in double and rounds once to bf16 through
// float; the product is exact in both, so a single RNE bf16 multiply gives
// the same bits for every finite and infinite operand.  NaN payloads differ
// (the hardware returns the canonical NaN) -- callers take the float path
// when the table can produce exponent 255 (kFlagHas255).
//
// raw holds the 8 packed (k+1)-bit items as loaded (first item in the MSBs
// of byte 0).  Each item (s<<k | m) becomes the byte s<<7 | m<<(7-k), the
// lossless sign/mantissa layout, so merge4 rebuilds the normalized values:
//   k=3: even/odd nibbles masked in place, interleaved by two PRMTs;
//   k=1: x * (1 + 2^10 + 2^20 + 2^30) moves 2-bit field j of byte x to bits
//        6-7 of byte j (the shifted copies do not overlap, so no carries);
//   k=0: x * (1 + 2^9 + 2^18 + 2^27) moves bit 7-j to bit 7 of byte j.
// lossy_unpack8 returns the 8 normalized values as 4 bf16x2 words.
template <int P>
__device__ __forceinline__ uint4 lossy_unpack8(uint32_t e0, uint32_t e1, uint32_t raw) {
    uint32_t sa, sb;
    if constexpr (P == 3) {
        const uint32_t ev = raw & 0xF0F0F0F0u, od = (raw << 4) & 0xF0F0F0F0u;
        sa = __byte_perm(ev, od, 0x5140);
        sb = __byte_perm(ev, od, 0x7362);
    } else if constexpr (P == 1) {
        sa = ((raw & 0xFFu) * 0x40100401u) & 0xC0C0C0C0u;
        sb = (((raw >> 8) & 0xFFu) * 0x40100401u) & 0xC0C0C0C0u;
    } else {
        static_assert(P == 0, "lossy precision");
        sa = ((raw & 0xFFu) * 0x08040201u) & 0x80808080u;
        sb = (((raw << 4) & 0xF0u) * 0x08040201u) & 0x80808080u;
    }
    const uint2 a = merge4(e0, sa), b = merge4(e1, sb);
    return make_uint4(a.x, a.y, b.x, b.y);
}

// All 8 elements scaled by one coefficient, given as a bf16x2 pair (cp = c | c << 16).
template <int P>
__device__ __forceinline__ uint4 lossy_merge8_cp(uint32_t e0, uint32_t e1, uint32_t raw, uint32_t cp) {
    const uint4 v = lossy_unpack8<P>(e0, e1, raw);
    return make_uint4(bf16x2_mul(v.x, cp), bf16x2_mul(v.y, cp), bf16x2_mul(v.z, cp), bf16x2_mul(v.w, cp));
}

// Elements [0, split) take coefficient c0, the rest c1 (bf16 bits).
template <int P>
__device__ __forceinline__ uint4 lossy_merge8(uint32_t e0, uint32_t e1, uint32_t raw, uint32_t c0, uint32_t c1,
                                              uint32_t split) {
    const uint4 v = lossy_unpack8<P>(e0, e1, raw);
    uint32_t cp[4];
    if (split >= 8) {
        cp[0] = cp[1] = cp[2] = cp[3] = c0 | (c0 << 16);
    } else {
#pragma unroll
        for (int p = 0; p < 4; ++p)
            cp[p] = ((uint32_t)(2 * p) < split ? c0 : c1) | (((uint32_t)(2 * p + 1) < split ? c0 : c1) << 16);
    }
    return make_uint4(bf16x2_mul(v.x, cp[0]), bf16x2_mul(v.y, cp[1]), bf16x2_mul(v.z, cp[2]),
                      bf16x2_mul(v.w, cp[3]));
}

// (k+1)-bit item i of a packed MSB-first stream (bitfloat.hpp:156-162).
__device__ __forceinline__ uint32_t packed_item(const uint8_t* packed, uint64_t i, int k) {
    const uint32_t width = (uint32_t)k + 1;
    const uint64_t bit = i * width;
    const uint32_t shift = 8 - width - (uint32_t)(bit & 7);
    return ((uint32_t)__ldg(packed + (bit >> 3)) >> shift) & ((1u << width) - 1u);
}

}  // namespace nzgpu
