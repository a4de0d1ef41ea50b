// decode.cu -- K5/K7 (tiled rANS decode fused with bf16 reassembly) and K8
// (sequential chunk decode: checkpoint-index build / irregular streams).
//
// K5/K7 replace ans_decode (ans.hpp:273-293) + decompress_lossless's merge
// loop (tensorstore.hpp:119-123) / decompress_lossy's rebuild loop
// (tensorstore.hpp:229-236) with ONE kernel per layer (a plan may group many
// tensors).  One CTA decodes a tile of 128 sub-ranges of K symbols:
//
//   1. thread 0 arms an mbarrier and issues two TMA bulk copies
//      (cp.async.bulk -> UBLKCP): the tensor's 16 KiB packed decode LUT and
//      the tile's contiguous window of payload bytes; it also issues an L2
//      bulk prefetch of the tile's sign/mantissa bytes;
//   2. every thread decodes its own sub-range (checkpoint index: state +
//      byte position every K symbols) from shared memory, packing four
//      exponents per 32-bit word into a padded (conflict-free) smem tile,
//      and verifies it lands exactly on the next checkpoint (the reference's
//      end-of-chunk desync check, ans.hpp:252, applied per sub-range);
//   3. the CTA merges exponents with the sign/mantissa plane in 16-element
//      groups: 128-bit coalesced loads, PRMT/LOP3 bit assembly, two 128-bit
//      coalesced stores per group.
//
// The byte format, the ratio and every output bit are the reference's; the
// side index only tells the decoder where sub-ranges start.
#include "nzgpu_internal.cuh"

namespace nzgpu {

constexpr int kDecodeThreads = 128;
constexpr uint32_t kLutBytes = 4096 * 4;
constexpr uint32_t kSmemHeader = 128;

__host__ __device__ constexpr uint32_t exps_row_words(int log2k) { return (1u << log2k) / 4 + 1; }

__host__ __device__ constexpr uint32_t decode_smem_bytes(int log2k, uint32_t win_cap) {
    return kSmemHeader + kLutBytes + kDecodeThreads * exps_row_words(log2k) * 4 + win_cap +
           2 * (1u << log2k) + 32;
}

__device__ __forceinline__ uint64_t chunk_offset(uint4 ci) { return (uint64_t)ci.x | ((uint64_t)ci.y << 32); }

// Absolute stream window [a, b) of renormalisation bytes a tile reads.
__device__ __forceinline__ void tile_window(const DecodeDesc& d, uint64_t sub0, uint32_t tile_subs,
                                            int log2k, uint64_t nsub, uint64_t& a, uint64_t& b) {
    const uint64_t spc = d.chunk_syms >> log2k;
    const uint64_t c0 = sub0 / spc;
    const uint4 ci0 = d.chunk_info[c0];
    const uint64_t lim0 = ci0.z >= 4 ? ci0.z - 4 : 0;
    const uint64_t e0 = (sub0 % spc == 0) ? lim0 : min((uint64_t)d.ckpt[sub0].y, lim0);
    a = chunk_offset(ci0) + lim0 - e0;
    const uint64_t jl = sub0 + tile_subs - 1;
    const uint64_t c1 = jl / spc;
    const uint4 ci1 = d.chunk_info[c1];
    const uint64_t lim1 = ci1.z >= 4 ? ci1.z - 4 : 0;
    const uint64_t jn = jl + 1;
    const uint64_t e1 = (jn < nsub && jn % spc != 0) ? min((uint64_t)d.ckpt[jn].y, lim1) : 0;
    b = chunk_offset(ci1) + lim1 - e1;
    if (b < a) b = a;
}

// Two bf16 from two exponent bytes and two sign/mantissa bytes packed as
// Y = e<<8 | s<<7 | m per 16-bit lane  ->  s<<15 | e<<7 | m.
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

__device__ __forceinline__ float scale_coef(uint8_t s) { return 1.0f + (float)s * (1.0f / 128.0f); }

// (k+1)-bit item i of a packed MSB-first stream (bitfloat.hpp:156-162).
__device__ __forceinline__ uint32_t packed_item(const uint8_t* packed, uint64_t i, int k) {
    const uint32_t width = (uint32_t)k + 1;
    const uint64_t bit = i * width;
    const uint32_t shift = 8 - width - (uint32_t)(bit & 7);
    return ((uint32_t)__ldg(packed + (bit >> 3)) >> shift) & ((1u << width) - 1u);
}

__device__ __forceinline__ void report(uint32_t* err, uint32_t bits) {
    if (bits) atomicOr(err, bits);
}

// One decode step (ans.hpp:240-251): LUT -> state transition -> renorm.
__device__ __forceinline__ uint32_t decode_step(uint32_t& x, const uint32_t* __restrict__ lut,
                                                const uint8_t*& pl) {
    const uint32_t v = lut[x & (kProbScale - 1)];
    x = (v >> 20) * (x >> kProbBits) + ((v >> 8) & 0xFFFu);
    if (x < kStateLow) {
        x = (x << 8) | *pl++;
        if (x < kStateLow) x = (x << 8) | *pl++;
    }
    return v;
}

template <int LOG2K, int P>
__global__ void __launch_bounds__(kDecodeThreads) decode_tiles_kernel(const DecodeDesc* __restrict__ descs,
                                                                      int ndesc,
                                                                      const uint64_t* __restrict__ tile_prefix,
                                                                      DecodeDesc one, uint32_t win_cap) {
    constexpr int T = kDecodeThreads;
    constexpr int K = 1 << LOG2K;
    constexpr int RW = exps_row_words(LOG2K);
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* win_base_s = reinterpret_cast<uint64_t*>(smem + 16);
    uint32_t* status_s = reinterpret_cast<uint32_t*>(smem + 24);
    uint32_t* lut_s = reinterpret_cast<uint32_t*>(smem + kSmemHeader);
    uint32_t* exps_s = reinterpret_cast<uint32_t*>(smem + kSmemHeader + kLutBytes);
    uint8_t* win_s = smem + kSmemHeader + kLutBytes + T * RW * 4;
    const int tid = threadIdx.x;

    // Locate the tensor of this tile (plans group many tensors per launch).
    uint64_t tile = blockIdx.x;
    const DecodeDesc* dp = &one;
    if (descs) {
        int lo = 0, hi = ndesc - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(tile_prefix + mid) <= tile) lo = mid; else hi = mid - 1;
        }
        dp = descs + lo;
        tile -= __ldg(tile_prefix + lo);
    }
    const DecodeDesc d = *dp;
    const uint64_t nsub = ceil_div(d.n, K);
    const uint64_t sub0 = tile * T;
    const uint32_t tile_subs = (uint32_t)min((uint64_t)T, nsub - sub0);
    const uint64_t sym0 = sub0 << LOG2K;
    const uint32_t tile_syms = (uint32_t)min((uint64_t)T * K, d.n - sym0);
    const bool single = d.flags & kFlagSingleSymbol;

    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        uint32_t st = 0;
        uint64_t wa = 0;
        if (!single) {
            uint64_t a, b;
            tile_window(d, sub0, tile_subs, LOG2K, nsub, a, b);
            wa = a & ~15ull;
            uint64_t bytes = ((b + 15) & ~15ull) - wa;
            if (bytes > win_cap) {  // corrupt index: never overrun shared memory
                st = kErrDesync;
                bytes = 0;
            }
            mbar_arrive_expect_tx(bar, kLutBytes + (uint32_t)bytes);
            bulk_g2s(lut_s, d.lut, kLutBytes, bar);
            if (bytes) bulk_g2s(win_s, d.stream + wa, (uint32_t)bytes, bar);
        }
        // Sign/mantissa bytes of the tile: warm L2 while the ANS lanes run.
        const uint64_t mb = ((uint64_t)tile_syms * (P + 1) / 8) & ~15ull;
        if (mb) prefetch_l2(d.mant + (sym0 * (P + 1) / 8), (uint32_t)mb);
        *win_base_s = wa;
        *status_s = st;
    }
    __syncthreads();

    uint32_t* row = exps_s + tid * RW;
    uint32_t errs = *status_s;
    if (tid < tile_subs) {
        const uint64_t spc = d.chunk_syms >> LOG2K;
        const uint64_t j = sub0 + tid;
        const uint64_t c = j / spc;
        const uint64_t jin = j - c * spc;
        const uint4 ci = d.chunk_info[c];
        const uint64_t off = chunk_offset(ci);
        const uint32_t len = ci.z, nsym = ci.w;
        const uint32_t sym_in = (uint32_t)(jin << LOG2K);
        const uint32_t cnt = nsym > sym_in ? min((uint32_t)K, nsym - sym_in) : 0u;
        if (jin == 0) {
            // The chunk's framing must agree with the index (ans.hpp:332-340).
            if (ld_u32le_bytes(d.stream + off - 8) != nsym || ld_u32le_bytes(d.stream + off - 4) != len)
                errs |= kErrLength;
        }
        if (len < 4) errs |= kErrTruncated;  // ans.hpp:231-233
        if (single) {
            // Constant path: a one-symbol table keeps the state at 2^23 and
            // consumes no bytes, so every chunk payload is exactly LE32(2^23).
            if (jin == 0 && len >= 4) {
                const uint32_t x0 = ld_u32le_bytes(d.stream + off + len - 4);
                if (x0 != kStateLow || len != 4) errs |= x0 < kStateLow ? kErrTruncated : kErrDesync;
            }
            const uint32_t w = d.single_symbol * 0x01010101u;
            for (uint32_t i = 0; i < (cnt + 3) / 4; ++i) row[i] = w;
        } else {
            const uint32_t limit = len >= 4 ? len - 4 : 0;
            const uint2 rec = d.ckpt[j];
            const bool last = sym_in + K >= nsym;
            const uint2 end = last ? make_uint2(kStateLow, 0u) : d.ckpt[j + 1];
            const uint32_t e_start = jin == 0 ? limit : rec.y;
            uint32_t x = jin == 0 ? ld_u32le_bytes(d.stream + off + limit) : rec.x;
            const uint64_t wa = *win_base_s;
            const int64_t p0 = (int64_t)(off + limit - e_start) - (int64_t)wa;
            const int64_t pe = (int64_t)(off + limit - min(end.y, limit)) - (int64_t)wa;
            if (e_start > limit || end.y > limit || p0 < 0 || p0 > (int64_t)win_cap) errs |= kErrDesync;
            mbar_wait(bar, 0);
            if (!errs) {
                const uint8_t* pl = win_s + p0;
                const uint32_t words = cnt >> 2;
#pragma unroll 2
                for (uint32_t w = 0; w < words; ++w) {
                    uint32_t v0 = decode_step(x, lut_s, pl);
                    uint32_t v1 = decode_step(x, lut_s, pl);
                    uint32_t v2 = decode_step(x, lut_s, pl);
                    uint32_t v3 = decode_step(x, lut_s, pl);
                    row[w] = __byte_perm(__byte_perm(v0, v1, 0x0040), __byte_perm(v2, v3, 0x0040), 0x5410);
                }
                uint32_t tailw = 0;
                for (uint32_t i = words * 4; i < cnt; ++i) {
                    const uint32_t v = decode_step(x, lut_s, pl);
                    tailw |= (v & 0xFFu) << (8 * (i & 3));
                }
                if (cnt & 3) row[words] = tailw;
                // End-of-sub-range check: the next checkpoint, or the
                // reference's end-of-chunk condition (x == 2^23, pos == len-4).
                const int64_t pos = pl - win_s;
                if (x != end.x || pos != pe) errs |= pos > pe ? kErrTruncated : kErrDesync;
            }
        }
    }
    if (!single && tid >= tile_subs) mbar_wait(bar, 0);  // never exit with a TMA in flight
    report(d.err, errs);
    __syncthreads();

    // ---- merge: exponents (smem) + sign/mantissa plane -> bf16 ---------------
    const uint32_t groups = tile_syms >> 4;
    uint4* out = reinterpret_cast<uint4*>(d.out + sym0);
    if constexpr (P == 7) {
        const uint4* sm4 = reinterpret_cast<const uint4*>(d.mant + sym0);
        for (uint32_t g = tid; g < groups; g += T) {
            const uint32_t e = g << 4;
            const uint32_t* er = exps_s + (e >> LOG2K) * RW + ((e & (K - 1)) >> 2);
            const uint4 s = __ldcs(sm4 + g);
            const uint32_t e0 = er[0], e1 = er[1], e2 = er[2], e3 = er[3];
            __stcs(out + 2 * g, merge8(e0, s.x, e1, s.y));
            __stcs(out + 2 * g + 1, merge8(e2, s.z, e3, s.w));
        }
        for (uint32_t i = groups * 16 + tid; i < tile_syms; i += T) {
            const uint32_t ex = (exps_s[(i >> LOG2K) * RW + ((i & (K - 1)) >> 2)] >> (8 * (i & 3))) & 0xFFu;
            const uint32_t sm = __ldg(d.mant + sym0 + i);
            d.out[sym0 + i] = (uint16_t)(((sm & 0x80u) << 8) | (ex << 7) | (sm & 0x7Fu));
        }
    } else {
        constexpr uint32_t W = P + 1;
        const uint8_t* packed = d.mant + sym0 * W / 8;
        const uint32_t B = d.block_size;
        for (uint32_t g = tid; g < groups; g += T) {
            const uint32_t e = g << 4;
            const uint32_t* er = exps_s + (e >> LOG2K) * RW + ((e & (K - 1)) >> 2);
            // 16 items = 2W bytes, MSB-first: gather big-endian into the top bits.
            uint64_t bits;
            if constexpr (W == 4) {
                const uint2 v = __ldcs(reinterpret_cast<const uint2*>(packed) + g);
                bits = ((uint64_t)__byte_perm(v.x, 0, 0x0123) << 32) | __byte_perm(v.y, 0, 0x0123);
            } else if constexpr (W == 2) {
                bits = (uint64_t)__byte_perm(__ldcs(reinterpret_cast<const uint32_t*>(packed) + g), 0, 0x0123) << 32;
            } else {
                bits = (uint64_t)__byte_perm(__ldcs(reinterpret_cast<const unsigned short*>(packed) + g), 0, 0x0144)
                       << 32;
            }
            const uint64_t gi = sym0 + e;
            const uint64_t b0 = gi / B;
            const float c0 = scale_coef(__ldg(d.scales + b0));
            const uint32_t split = (uint32_t)min((uint64_t)16, (b0 + 1) * B - gi);
            const float c1 = split < 16 ? scale_coef(__ldg(d.scales + b0 + 1)) : c0;
            uint32_t res[8];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t ex = (er[q >> 2] >> (8 * (q & 3))) & 0xFFu;
                const uint32_t item = (uint32_t)(bits >> (64 - (q + 1) * W)) & ((1u << W) - 1u);
                float c = q < (int)split ? c0 : c1;
                if (B < 16 && q >= (int)split) c = scale_coef(__ldg(d.scales + (gi + q) / B));
                const uint32_t h = lossy_rebuild(item, ex, P, c);
                if (q & 1) res[q >> 1] |= h << 16; else res[q >> 1] = h;
            }
            __stcs(out + 2 * g, make_uint4(res[0], res[1], res[2], res[3]));
            __stcs(out + 2 * g + 1, make_uint4(res[4], res[5], res[6], res[7]));
        }
        for (uint32_t i = groups * 16 + tid; i < tile_syms; i += T) {
            const uint32_t ex = (exps_s[(i >> LOG2K) * RW + ((i & (K - 1)) >> 2)] >> (8 * (i & 3))) & 0xFFu;
            const uint64_t gi = sym0 + i;
            const uint32_t item = packed_item(d.mant, gi, P);
            d.out[gi] = lossy_rebuild(item, ex, P, scale_coef(__ldg(d.scales + gi / B)));
        }
    }
}

// ------------------------------------------------------------------ K8 ---
// Sequential decode of whole chunks, one thread per chunk, with exactly the
// reference's checks (ans.hpp:229-256).  Used to (a) build the checkpoint
// index of streams that did not come from our encoder (e.g. produced by the
// CPU reference) and (b) decode streams with irregular chunk framing.
__global__ void __launch_bounds__(128) seq_decode_kernel(const uint8_t* __restrict__ stream,
                                                         const uint4* __restrict__ chunk_info,
                                                         const uint64_t* __restrict__ chunk_sym0,
                                                         uint32_t chunk_syms, uint64_t nchunks, const uint32_t* __restrict__ lut_g,
                                                         uint32_t flags, uint32_t log2k,
                                                         uint2* __restrict__ ckpt,
                                                         uint8_t* __restrict__ exps,
                                                         uint32_t* __restrict__ err) {
    __shared__ uint32_t lut[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) lut[i] = lut_g[i];
    __syncthreads();
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const uint4 ci = chunk_info[c];
    const uint8_t* pl = stream + chunk_offset(ci);
    const uint32_t len = ci.z, nsym = ci.w;
    const uint64_t base = chunk_sym0 ? chunk_sym0[c] : c * chunk_syms;
    if (len < 4) {  // ans.hpp:231-233
        atomicOr(err, kErrTruncated);
        return;
    }
    const uint32_t limit = len - 4;
    uint32_t x = ld_u32le_bytes(pl + limit);
    uint32_t pos = 0;
    const uint32_t kmask = (1u << log2k) - 1u;
    const bool single = flags & kFlagSingleSymbol;
    for (uint32_t i = 0; i < nsym; ++i) {
        if (ckpt && ((base + i) & kmask) == 0) ckpt[(base + i) >> log2k] = make_uint2(x, limit - pos);
        const uint32_t slot = x & (kProbScale - 1);
        const uint32_t v = lut[slot];
        const uint32_t f = single ? kProbScale : (v >> 20);
        x = f * (x >> kProbBits) + (single ? slot : ((v >> 8) & 0xFFFu));
        while (x < kStateLow) {
            if (pos >= limit) {  // ans.hpp:245-247
                atomicOr(err, kErrTruncated);
                return;
            }
            x = (x << 8) | pl[pos++];
        }
        if (exps) exps[base + i] = (uint8_t)(v & 0xFFu);
    }
    if (x != kStateLow || pos != limit) atomicOr(err, kErrDesync);  // ans.hpp:252-254
}

// Merge of a global exponent plane with the mantissa plane (irregular-
// framing fallback after seq_decode_kernel).
__global__ void merge_plane_kernel(const uint8_t* __restrict__ exps, const uint8_t* __restrict__ mant,
                                   const uint8_t* __restrict__ scales, uint64_t n, int k, uint32_t block,
                                   uint16_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = exps[i];
        if (k == 7) {
            const uint32_t sm = mant[i];
            out[i] = (uint16_t)(((sm & 0x80u) << 8) | (e << 7) | (sm & 0x7Fu));
        } else {
            out[i] = lossy_rebuild(packed_item(mant, i, k), e, k, scale_coef(scales[i / block]));
        }
    }
}

// Largest payload window any tile of a tensor needs (sizes dynamic smem).
template <int LOG2K>
__global__ void window_max_kernel(DecodeDesc d, uint32_t* __restrict__ out) {
    const uint64_t nsub = ceil_div(d.n, 1u << LOG2K);
    const uint64_t tiles = ceil_div(nsub, kDecodeThreads);
    uint32_t best = 0;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < tiles; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t sub0 = t * kDecodeThreads;
        const uint32_t subs = (uint32_t)min((uint64_t)kDecodeThreads, nsub - sub0);
        uint64_t a, b;
        tile_window(d, sub0, subs, LOG2K, nsub, a, b);
        const uint64_t bytes = ((b + 15) & ~15ull) - (a & ~15ull);
        best = max(best, (uint32_t)min(bytes, (uint64_t)0xFFFFFFFFu));
    }
    atomicMax(out, best);
}

// ------------------------------------------------------------ launchers --
template <int LOG2K, int P>
static cudaError_t launch_decode_t(const DecodeDesc* descs, int ndesc, const uint64_t* prefix, const DecodeDesc& one,
                                   uint64_t tiles, uint32_t win_cap, cudaStream_t s) {
    const uint32_t smem = decode_smem_bytes(LOG2K, win_cap);
    static uint32_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(decode_tiles_kernel<LOG2K, P>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    decode_tiles_kernel<LOG2K, P><<<(unsigned)tiles, kDecodeThreads, smem, s>>>(descs, ndesc, prefix, one, win_cap);
    return cudaGetLastError();
}

template <int LOG2K>
static cudaError_t launch_decode_k(int precision, const DecodeDesc* descs, int ndesc, const uint64_t* prefix,
                                   const DecodeDesc& one, uint64_t tiles, uint32_t win_cap, cudaStream_t s) {
    switch (precision) {
        case 7: return launch_decode_t<LOG2K, 7>(descs, ndesc, prefix, one, tiles, win_cap, s);
        case 3: return launch_decode_t<LOG2K, 3>(descs, ndesc, prefix, one, tiles, win_cap, s);
        case 1: return launch_decode_t<LOG2K, 1>(descs, ndesc, prefix, one, tiles, win_cap, s);
        case 0: return launch_decode_t<LOG2K, 0>(descs, ndesc, prefix, one, tiles, win_cap, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_decode(int log2k, int precision, const DecodeDesc* descs, int ndesc, const uint64_t* prefix,
                          const DecodeDesc& one, uint64_t tiles, uint32_t win_cap, cudaStream_t s) {
    if (tiles == 0) return cudaSuccess;
    switch (log2k) {
        case 6: return launch_decode_k<6>(precision, descs, ndesc, prefix, one, tiles, win_cap, s);
        case 7: return launch_decode_k<7>(precision, descs, ndesc, prefix, one, tiles, win_cap, s);
        case 8: return launch_decode_k<8>(precision, descs, ndesc, prefix, one, tiles, win_cap, s);
        default: return cudaErrorInvalidValue;
    }
}

uint32_t decode_smem_for(int log2k, uint32_t win_cap) { return decode_smem_bytes(log2k, win_cap); }

cudaError_t launch_window_max(int log2k, const DecodeDesc& d, uint32_t* out, cudaStream_t s) {
    switch (log2k) {
        case 6: window_max_kernel<6><<<148, 256, 0, s>>>(d, out); break;
        case 7: window_max_kernel<7><<<148, 256, 0, s>>>(d, out); break;
        case 8: window_max_kernel<8><<<148, 256, 0, s>>>(d, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace nzgpu
