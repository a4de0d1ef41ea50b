// decode_tiles.cu -- K5/K7: tiled rANS decode fused with bf16 reassembly.
//
// Replaces ans_decode (ans.hpp:273-293) + decompress_lossless's merge loop
// (tensorstore.hpp:119-123) / decompress_lossy's rebuild loop
// (tensorstore.hpp:229-236) with ONE kernel launch per layer (a plan groups
// many tensors).  A CTA of 128 threads decodes a tile of 128*kChains
// sub-ranges of K symbols (the checkpoint side index gives every sub-range
// its starting state and byte position):
//
//   1. thread 0 arms an mbarrier and issues TMA bulk copies (cp.async.bulk,
//      SASS UBLKCP) of the tensor's 16 KiB packed decode LUT and of the tile's
//      contiguous payload window; meanwhile every thread issues its 128-bit
//      loads of the tile's sign/mantissa plane into registers, so they are in
//      flight during the whole decode;
//   2. every thread runs kChains independent ANS lanes interleaved for ILP,
//      entirely out of shared memory: LUT lookup, state transition, a
//      predicated one-byte renormalisation and a predicated second byte.
//      Four exponents are packed per 32-bit word into a padded
//      (bank-conflict-free) exponent tile.  Every lane must land exactly on
//      the next checkpoint -- the reference's end-of-chunk desync check
//      (ans.hpp:252) applied to every sub-range;
//   3. the CTA merges exponents with the sign/mantissa plane in 16-element
//      groups: PRMT/LOP3 bit assembly, two 128-bit streaming stores per group.
//
// Byte format, ratio and every output bit are the reference's.
#include "decode_common.cuh"

namespace nzgpu {

namespace {

constexpr uint32_t kLutOff = kSmemHeader;
constexpr uint32_t kExpOff = kSmemHeader + kLutBytes;

template <int LOG2K>
__host__ __device__ constexpr uint32_t win_off() {
    return kExpOff + kTileSubs * exps_row_words(LOG2K) * 4;
}

// Sign/mantissa bytes of one 8-element group: lossless 8 B, lossy (k+1) B.
template <int P>
struct GroupBits;
template <>
struct GroupBits<7> {
    using T = uint2;
};
template <>
struct GroupBits<3> {
    using T = uint32_t;
};
template <>
struct GroupBits<1> {
    using T = unsigned short;
};
template <>
struct GroupBits<0> {
    using T = unsigned char;
};

}  // namespace

// Shared-memory loads on 32-bit shared-window addresses.  They are NOT
// volatile, so the compiler may interleave the independent ANS lanes of a
// thread freely; they stay behind the mbarrier wait because every address
// they use is derived from the wait's output token (see mbar_wait_token).
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// mbarrier wait that returns a data dependency (always 0) to thread the
// completion of the TMA copies into later (non-volatile) shared loads.
__device__ __forceinline__ uint32_t mbar_wait_token(uint64_t* bar, uint32_t parity) {
    uint32_t tok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "@!p bra WAITT_%=;\n"
        "mov.u32 %0, 0;\n"
        "}\n"
        : "=r"(tok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return tok;
}

// One decode step (ans.hpp:240-251).  `lut` is the shared address of the
// packed LUT, `p` the shared address of the next payload byte and `b` that
// byte, loaded one step ahead.  With v = f<<20 | (slot-cum)<<8 | sym:
//   f*(x>>12) + slot - cum  ==  f*((x>>12) - 4096) + (v>>8)   (mod 2^32),
// which saves the bias mask (the >>12 and -4096 fuse into one LEA.HI).
// Renormalisation is predicated, never divergent, and the byte reload is
// predicated on consumption: only the ~1/3 of lanes that consumed a byte
// touch shared memory, which cuts the bank-conflict wavefronts of the
// (random-address) byte loads -- shared-memory wavefronts, not issue slots,
// bound this loop (ncu: L1 data pipe 94% busy).
#define NZ_DECODE_STEP(lut, x, p, b, v)                                                      \
    do {                                                                                     \
        uint32_t a_;                                                                         \
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a_) : "r"((x) & 0xFFFu), "r"(lut));           \
        v = lds32(a_);                                                                       \
        x = ((v) >> 20) * (((x) >> kProbBits) - kProbScale) + ((v) >> 8);                    \
        asm(                                                                                 \
            "{\n\t.reg .pred q;\n\t"                                                         \
            "setp.lt.u32 q, %0, 8388608;\n\t"                                                \
            "@q mad.lo.u32 %0, %0, 256, %2;\n\t"                                             \
            "@q add.u32 %1, %1, 1;\n\t"                                                      \
            "@q ld.shared.u8 %2, [%1];\n\t"                                                  \
            "setp.lt.u32 q, %0, 8388608;\n\t"                                                \
            "@q mad.lo.u32 %0, %0, 256, %2;\n\t"                                             \
            "@q add.u32 %1, %1, 1;\n\t"                                                      \
            "@q ld.shared.u8 %2, [%1];\n\t}"                                                 \
            : "+r"(x), "+r"(p), "+r"(b));                                                    \
    } while (0)

// Same step with the renormalisation bytes served from a per-lane 8-byte
// register window {w, w2} = shared words [q, q+8): a byte at bit offset o8
// is one clamped funnel shift + one PRMT away, and the window only refills
// (one aligned 32-bit load) when a lane crosses a word -- ~8% of lanes per
// step instead of ~30% random byte loads, i.e. far fewer bank-conflict
// wavefronts in the L1 data pipe.
#define NZ_DECODE_STEP_W(lut, x, q, o8, w, w2, v)                                            \
    do {                                                                                     \
        uint32_t a_;                                                                         \
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a_) : "r"((x) & 0xFFFu), "r"(lut));           \
        v = lds32(a_);                                                                       \
        x = ((v) >> 20) * (((x) >> kProbBits) - kProbScale) + ((v) >> 8);                    \
        asm(                                                                                 \
            "{\n\t.reg .pred q;\n\t.reg .b32 t, u;\n\t"                                      \
            "setp.lt.u32 q, %0, 8388608;\n\t"                                                \
            "shf.r.clamp.b32 t, %3, %4, %2;\n\t"                                             \
            "@q prmt.b32 %0, %0, t, 0x2104;\n\t"                                             \
            "@q add.u32 %2, %2, 8;\n\t"                                                      \
            "setp.lt.and.u32 q, %0, 8388608, q;\n\t"                                         \
            "shf.r.clamp.b32 u, %3, %4, %2;\n\t"                                             \
            "@q prmt.b32 %0, %0, u, 0x2104;\n\t"                                             \
            "@q add.u32 %2, %2, 8;\n\t"                                                      \
            "setp.ge.u32 q, %2, 32;\n\t"                                                     \
            "@q mov.b32 %3, %4;\n\t"                                                         \
            "@q add.u32 %1, %1, 4;\n\t"                                                      \
            "@q sub.u32 %2, %2, 32;\n\t"                                                     \
            "@q ld.shared.u32 %4, [%1+4];\n\t}"                                              \
            : "+r"(x), "+r"(q), "+r"(o8), "+r"(w), "+r"(w2));                                \
    } while (0)

template <int LOG2K, int P>
__global__ void __launch_bounds__(kDecodeThreads, NZ_MINBLOCKS) decode_tiles_kernel(const DecodeDesc* __restrict__ descs,
                                                                      int ndesc,
                                                                      const uint64_t* __restrict__ tile_prefix,
                                                                      DecodeDesc one, uint32_t win_cap) {
    constexpr int T = kDecodeThreads;
    constexpr int CH = kChains;
    constexpr int TS = kTileSubs;
    constexpr int K = 1 << LOG2K;
    constexpr uint32_t RW = exps_row_words(LOG2K);
    constexpr uint32_t kWinOff = win_off<LOG2K>();
    constexpr int G = TS * K / 8 / T;           // 8-element merge groups per thread
    constexpr int PF = G < NZ_PF ? G : NZ_PF;   // groups prefetched into registers
    using GB = typename GroupBits<P>::T;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint32_t* exps_s = reinterpret_cast<uint32_t*>(smem + kExpOff);
    const int tid = threadIdx.x;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t lut = sbase + kLutOff;

    // Locate the tensor of this tile (plans group many tensors per launch).
    uint32_t tile = blockIdx.x;
    const DecodeDesc* dp = &one;
    if (descs) {
        int lo = 0, hi = ndesc - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(tile_prefix + mid) <= tile) lo = mid; else hi = mid - 1;
        }
        dp = descs + lo;
        tile -= (uint32_t)__ldg(tile_prefix + lo);
    }
    const DecodeDesc d = *dp;
    const uint32_t nsub = (uint32_t)ceil_div(d.n, K);
    const uint32_t sub0 = tile * TS;
    const uint32_t tile_subs = min((uint32_t)TS, nsub - sub0);
    const uint64_t sym0 = (uint64_t)sub0 << LOG2K;
    const uint32_t tile_syms = (uint32_t)min((uint64_t)TS * K, d.n - sym0);
    const uint32_t groups = tile_syms >> 3;
    const bool single = d.flags & kFlagSingleSymbol;
    const bool fast_lossy = d.block_size >= 8 && !(d.flags & kFlagSlowLossy);

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
            bulk_g2s(smem + kLutOff, d.lut, kLutBytes, bar);
            if (bytes) bulk_g2s(smem + kWinOff, d.stream + wa, (uint32_t)bytes, bar);
        }
        *reinterpret_cast<uint64_t*>(smem + 16) = wa;
        *reinterpret_cast<uint32_t*>(smem + 24) = st;
    }

    // Sign/mantissa plane of this tile: issue the loads now, use them after
    // the decode (group g = tid + i*T, coalesced across the CTA).
    const GB* gbits = reinterpret_cast<const GB*>(d.mant + sym0 * (P + 1) / 8);
    GB pre[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) {
        const uint32_t g = tid + i * T;
        if (g < groups) pre[i] = __ldcs(gbits + g);
    }
    __syncthreads();

    const uint64_t wa = *reinterpret_cast<const uint64_t*>(smem + 16);
    uint32_t errs = *reinterpret_cast<const uint32_t*>(smem + 24);    uint32_t x[CH], p[CH], xe[CH], pe[CH], cnt[CH];
    bool all_full = true;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint32_t r = c * T + tid;  // tile-local sub-range == exponent-tile row
        cnt[c] = 0;
        x[c] = xe[c] = kStateLow;
        p[c] = pe[c] = sbase + kWinOff;
        const uint32_t j = sub0 + r;
        const bool valid = r < tile_subs;
        uint32_t ch = 0, jin = 0;
        if (valid) sub_to_chunk(d, LOG2K, j, ch, jin);
        if (valid) {
            const uint4 ci = d.chunk_info[ch];
            const uint64_t off = chunk_offset(ci);
            const uint32_t len = ci.z, nsym = ci.w;
            const uint32_t sym_in = jin << LOG2K;
            cnt[c] = nsym > sym_in ? min((uint32_t)K, nsym - sym_in) : 0u;
            if (len < 4) errs |= kErrTruncated;  // ans.hpp:231-233
            const uint32_t limit = len >= 4 ? len - 4 : 0;
            if (jin == 0) {
                // The chunk's framing must agree with the index (ans.hpp:332-340),
                // and the chunk's first lane starts from the stream's own final
                // state (ans.hpp:235-236), not from the index.
                if (ld_u32le_bytes(d.stream + off - 8) != nsym || ld_u32le_bytes(d.stream + off - 4) != len)
                    errs |= kErrLength;
                x[c] = ld_u32le_bytes(d.stream + off + limit);
            }
            if (single) {
                // A one-symbol table keeps the state at 2^23 and consumes no
                // bytes: every chunk payload must be exactly LE32(2^23).
                if (jin == 0 && len >= 4 && (x[c] != kStateLow || len != 4))
                    errs |= x[c] < kStateLow ? kErrTruncated : kErrDesync;
            } else {
                // positions as in decode_persist.cu lane_job (nzgpu_internal.cuh)
                const uint32_t lane = j & 31u;
                const uint32_t ref = jin >= lane ? d.ck_base[j >> 5] : 0u;
                const uint32_t start = d.ck_off[j] + ref;
                const bool last = sym_in + K >= nsym;
                if (jin != 0) x[c] = d.ck_state[j];
                xe[c] = last ? kStateLow : d.ck_state[j + 1];
                const uint32_t end =
                    last ? limit : d.ck_off[j + 1] + (lane == 31u ? d.ck_base[(j >> 5) + 1] : ref);
                const int64_t p0 = (int64_t)(off + min(start, limit)) - (int64_t)wa;
                const int64_t p1 = (int64_t)(off + min(end, limit)) - (int64_t)wa;
                if (start > limit || end > limit || p0 < 0 || p1 > (int64_t)win_cap || p1 < p0)
                    errs |= kErrDesync;
                else {
                    p[c] = sbase + kWinOff + (uint32_t)p0;
                    pe[c] = sbase + kWinOff + (uint32_t)p1;
                }
            }
        }
        all_full &= cnt[c] == (uint32_t)K;
    }

    if (single) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            uint32_t* row = exps_s + (c * T + tid) * RW;
            const uint32_t w = d.single_symbol * 0x01010101u;
            for (uint32_t i = 0; i < (cnt[c] + 3) / 4; ++i) row[i] = w;
        }
    } else {
        // LUT + payload window landed (never exit with a TMA in flight); every
        // shared address below carries the wait's token.
        const uint32_t tok = mbar_wait_token(bar, 0);
        const uint32_t lutt = lut + tok;
        if (!errs) {
            uint32_t b[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                p[c] += tok;
                b[c] = lds8(p[c]);
            }
            if (all_full) {
                // Hot loop: CH independent ANS lanes interleaved per thread.
#if NZ_WINDOW
                uint32_t q[CH], o8[CH], w0[CH], w1[CH];
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    q[c] = p[c] & ~3u;
                    o8[c] = (p[c] & 3u) * 8;
                    w0[c] = lds32(q[c]);
                    w1[c] = lds32(q[c] + 4);
                }
#endif
#pragma unroll 1
                for (uint32_t w = 0; w < (uint32_t)K / 4; ++w) {
                    uint32_t v[CH][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
#if NZ_WINDOW
                            NZ_DECODE_STEP_W(lutt, x[c], q[c], o8[c], w0[c], w1[c], v[c][u]);
#else
                            NZ_DECODE_STEP(lutt, x[c], p[c], b[c], v[c][u]);
#endif
                        }
                    }
#pragma unroll
                    for (int c = 0; c < CH; ++c)
                        exps_s[(c * T + tid) * RW + w] = __byte_perm(__byte_perm(v[c][0], v[c][1], 0x0040),
                                                                     __byte_perm(v[c][2], v[c][3], 0x0040), 0x5410);
                }
#if NZ_WINDOW
#pragma unroll
                for (int c = 0; c < CH; ++c) p[c] = q[c] + (o8[c] >> 3);
#endif
            } else {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    uint32_t* row = exps_s + (c * T + tid) * RW;
                    uint32_t word = 0;
                    for (uint32_t i = 0; i < cnt[c]; ++i) {
                        uint32_t v;
                        NZ_DECODE_STEP(lutt, x[c], p[c], b[c], v);
                        word |= (v & 0xFFu) << (8 * (i & 3));
                        if ((i & 3) == 3 || i + 1 == cnt[c]) {
                            row[i >> 2] = word;
                            word = 0;
                        }
                    }
                }
            }
            // End of every lane: the next checkpoint, or the reference's
            // end-of-chunk condition (x == 2^23, pos == len-4).
#pragma unroll
            for (int c = 0; c < CH; ++c)
                if (cnt[c] && (x[c] != xe[c] || p[c] != pe[c])) errs |= p[c] > pe[c] ? kErrTruncated : kErrDesync;
        }
    }
    if (errs) atomicOr(d.err, errs);
    __syncthreads();

    // ---- merge: exponents (smem) + sign/mantissa plane -> bf16 ---------------
    uint4* out = reinterpret_cast<uint4*>(d.out + sym0);
    const uint32_t B = d.block_size;
    // Groups beyond the register prefetch are loaded in batches of PF so their
    // latencies overlap (no load waits on the previous group's store).
    GB nxt[PF];
#pragma unroll
    for (int i = 0; i < G; ++i) {
        if (i >= PF && i % PF == 0) {
#pragma unroll
            for (int j = 0; j < PF; ++j) {
                const uint32_t gj = tid + (i + j) * T;
                if (i + j < G && gj < groups) nxt[j] = __ldcs(gbits + gj);
            }
        }
        const uint32_t g = tid + i * T;  // 8-element group: one 16-byte store per lane, coalesced
        if (g >= groups) break;
        const GB s = i < PF ? pre[i % PF] : nxt[i % PF];
        const uint32_t e = g << 3;
        const uint32_t* er = exps_s + (e >> LOG2K) * RW + ((e & (K - 1)) >> 2);
        const uint32_t e0 = er[0], e1 = er[1];
        if constexpr (P == 7) {
            NZ_CHECK(sym0 + 8ull * g + 8 <= d.n);
            __stcs(out + g, merge8(e0, s.x, e1, s.y));
        } else if (fast_lossy) {
            const uint64_t gi = sym0 + e;
            uint32_t b0, split;
            if (d.log2_block != 0xFFFFFFFFu) {
                b0 = (uint32_t)(gi >> d.log2_block);
                split = min(8u, B - ((uint32_t)gi & (B - 1u)));
            } else {
                b0 = (uint32_t)(gi / B);
                split = (uint32_t)min((uint64_t)8, (uint64_t)(b0 + 1) * B - gi);
            }
            const uint32_t c0 = scale_coef_bf16(__ldg(d.scales + b0));
            const uint32_t c1 = split < 8 ? scale_coef_bf16(__ldg(d.scales + b0 + 1)) : c0;
            __stcs(out + g, lossy_merge8<P>(e0, e1, (uint32_t)s, c0, c1, split));
        } else {
            constexpr uint32_t W = P + 1;
            // 8 items of W bits, MSB-first: gather big-endian into the top bits.
            uint32_t bits;
            if constexpr (W == 4) {
                bits = __byte_perm(s, 0, 0x0123);
            } else if constexpr (W == 2) {
                bits = __byte_perm((uint32_t)s, 0, 0x0144) ;
            } else {
                bits = (uint32_t)s << 24;
            }
            const uint64_t gi = sym0 + e;
            const uint64_t b0 = gi / B;
            const float c0 = scale_coef(__ldg(d.scales + b0));
            const uint32_t split = (uint32_t)min((uint64_t)8, (b0 + 1) * B - gi);
            const float c1 = split < 8 ? scale_coef(__ldg(d.scales + b0 + 1)) : c0;
            const uint32_t ew[2] = {e0, e1};
            uint32_t res[4];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t ex = (ew[q >> 2] >> (8 * (q & 3))) & 0xFFu;
                const uint32_t item = (bits >> (32 - (q + 1) * W)) & ((1u << W) - 1u);
                float c = q < (int)split ? c0 : c1;
                if (B < 8 && q >= (int)split) c = scale_coef(__ldg(d.scales + (gi + q) / B));
                const uint32_t h = lossy_rebuild(item, ex, P, c);
                if (q & 1) res[q >> 1] |= h << 16; else res[q >> 1] = h;
            }
            __stcs(out + g, make_uint4(res[0], res[1], res[2], res[3]));
        }
    }
    // Tail of the tensor (n % 8 elements).
    for (uint32_t i = groups * 8 + tid; i < tile_syms; i += T) {
        const uint32_t ex = (exps_s[(i >> LOG2K) * RW + ((i & (K - 1)) >> 2)] >> (8 * (i & 3))) & 0xFFu;
        const uint64_t gi = sym0 + i;
        if constexpr (P == 7) {
            const uint32_t sm = __ldg(d.mant + gi);
            d.out[gi] = (uint16_t)(((sm & 0x80u) << 8) | (ex << 7) | (sm & 0x7Fu));
        } else {
            d.out[gi] = lossy_rebuild(packed_item(d.mant, gi, P), ex, P, scale_coef(__ldg(d.scales + gi / B)));
        }
    }
}

// Largest payload window any tile of a tensor needs (sizes dynamic smem).
template <int LOG2K>
__global__ void window_max_kernel(DecodeDesc d, uint32_t* __restrict__ out) {
    const uint32_t nsub = (uint32_t)ceil_div(d.n, 1u << LOG2K);
    const uint32_t tiles = (uint32_t)ceil_div(nsub, kTileSubs);
    uint32_t best = 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < tiles; t += gridDim.x * blockDim.x) {
        const uint32_t sub0 = t * kTileSubs;
        const uint32_t subs = min((uint32_t)kTileSubs, nsub - sub0);
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
    static SmemAttr attr;  // per device: one process may drive several GPUs
    if (cudaError_t e = attr.ensure((const void*)decode_tiles_kernel<LOG2K, P>, smem)) return e;
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
        default: return cudaErrorInvalidValue;
    }
}

uint32_t decode_smem_for(int log2k, uint32_t win_cap) {
    switch (log2k) {
        case 6: return decode_smem_bytes(6, win_cap);
        case 7: return decode_smem_bytes(7, win_cap);
        default: return decode_smem_bytes(8, win_cap);
    }
}

uint64_t decode_tiles_for(uint64_t nsub) { return ceil_div(nsub, kTileSubs); }
uint64_t decode_tile_subs() { return kTileSubs; }

cudaError_t launch_window_max(int log2k, const DecodeDesc& d, uint32_t* out, cudaStream_t s) {
    switch (log2k) {
        case 6: window_max_kernel<6><<<148, 256, 0, s>>>(d, out); break;
        case 7: window_max_kernel<7><<<148, 256, 0, s>>>(d, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace nzgpu
