// decode_persist.cu -- K5/K7, persistent warp-pipelined variant (default).
//
// Same contract and bit-exact output as decode_tiles.cu, different schedule:
//
//  * a CTA owns a contiguous range of work units of ONE tensor, so the
//    16 KiB packed decode LUT is TMA-loaded once per CTA (not per tile);
//  * a work unit is one warp's worth of sub-ranges: 32 lanes x K symbols;
//    every warp runs its own pipeline with no CTA-wide barrier: while it
//    decodes unit i from shared memory, the TMA bulk copy (UBLKCP, own
//    mbarrier per buffer) of unit i+1's payload window is already in flight
//    and the unit's sign/mantissa words are in registers;
//  * each lane decodes one sub-range (ANS lane) from a register byte window,
//    checks it lands on the next checkpoint (ans.hpp:252 applied per
//    sub-range), writes exponents into the warp's padded smem tile, and the
//    same warp then merges the unit with coalesced 16-byte stores -- so
//    decode (ALU/shared) of some warps overlaps merge (HBM) of others.
#include <algorithm>
#include <type_traits>

#include "decode_common.cuh"

#ifndef NZ_PWARPS
#define NZ_PWARPS 32  // warps per persistent CTA (one CTA per SM)
#endif
#ifndef NZ_PUNROLL
#define NZ_PUNROLL 16  // 4-step groups of the full-sub-range decode loop unrolled (16 = all of K=64)
#endif

#ifndef NZ_PMINB
#define NZ_PMINB 1  // resident CTAs per SM the register budget must allow
#endif

namespace nzgpu {

namespace {

#ifndef NZ_HALVES_UNROLL
#define NZ_HALVES_UNROLL 2
#endif
constexpr int kHalvesUnroll = NZ_HALVES_UNROLL;  // K = 128 in halves: unrolled halves (code size vs registers)
#ifndef NZ_K128_SPLIT
#define NZ_K128_SPLIT 0  // K = 128: 1 = two 64-symbol halves at NZ_PWARPS warps, 0 = one pass at NZ_K128_WARPS
#endif
#ifndef NZ_K128_WARPS
#define NZ_K128_WARPS 24  // a K = 128 unit's exponent tile is twice K = 64's: fewer warps fit
#endif
constexpr int kPWarps = NZ_PWARPS;
// warps per persistent CTA, and the log2 of the symbols per exponent-tile row
__host__ __device__ constexpr int p_warps(int log2k) { return (log2k == 7 && !NZ_K128_SPLIT) ? NZ_K128_WARPS : NZ_PWARPS; }
__host__ __device__ constexpr int tile_log2(int log2k) { return (log2k == 7 && NZ_K128_SPLIT) ? 6 : log2k; }
constexpr int kPUnroll = NZ_PUNROLL;
constexpr int kPThreads = kPWarps * 32;
constexpr uint32_t kPHeader = 128;  // LUT mbarrier

// exponent tile of a warp: 32 rows of (at most) 64 symbols (K = 128 is merged
// in two halves through the same tile)
__host__ __device__ constexpr uint32_t unit_words(int log2k) { return 32 * exps_row_words(tile_log2(log2k)); }

// Per-warp region: its 2 mbarriers (16 B), the exponent tile (32 padded
// rows) and 2 payload windows -- every per-warp address is the region base
// plus a constant, so register pressure never has to rematerialise more than
// one value.
constexpr uint32_t kPWarpBars = 16;
__host__ __device__ constexpr uint32_t warp_region(int log2k, uint32_t win_cap) {
    return (kPWarpBars + unit_words(log2k) * 4 + 2 * (win_cap + 2 * (1u << log2k) + 64) + 127) & ~127u;
}

__host__ __device__ constexpr uint32_t persist_smem(int log2k, uint32_t win_cap) {
    return kPHeader + kLutBytes + p_warps(log2k) * warp_region(log2k, win_cap);
}

template <int P>
struct HalfBits;
template <>
struct HalfBits<7> {
    using T = uint2;
};
template <>
struct HalfBits<3> {
    using T = uint32_t;
};
template <>
struct HalfBits<1> {
    using T = unsigned short;
};
template <>
struct HalfBits<0> {
    using T = unsigned char;
};

// Uniform accessors over the per-precision group words (a generic lambda
// instantiates every flavour for every precision).
__device__ __forceinline__ uint32_t hb_raw(uint32_t v) { return v; }
__device__ __forceinline__ uint32_t hb_raw(uint2 v) { return v.x; }
__device__ __forceinline__ uint32_t hb_lo(uint2 v) { return v.x; }
__device__ __forceinline__ uint32_t hb_hi(uint2 v) { return v.y; }
__device__ __forceinline__ uint32_t hb_lo(uint32_t) { return 0; }
__device__ __forceinline__ uint32_t hb_hi(uint32_t) { return 0; }

}  // namespace

__device__ __forceinline__ uint32_t p_lds32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t p_lds8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t p_wait_token(uint32_t bar, uint32_t parity) {
    uint32_t tok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "@!p bra PWAIT_%=;\n"
        "mov.u32 %0, 0;\n"
        "}\n"
        : "=r"(tok)
        : "r"(bar), "r"(parity)
        : "memory");
    return tok;
}
__device__ __forceinline__ void p_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void p_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Opaque constants passed as a kernel parameter so ptxas cannot fold the
// FMA-pipe forms below back into ALU instructions.
struct MulConsts {
    uint32_t one;
};

// The ANS step (ans.hpp:238-255) balanced across the two integer pipes.  ncu
// on the first version showed the half-rate ALU pipe 89% busy and the FMA
// pipe 25%, so everything that can be a multiply-add is one:
//   * slot address 4 (x & 0xFFF) + lut = 4x - 16384 (x >> 12) + lut, with
//     h' = (x >> 12) - 4096 (one LEA.HI) shared with the state update
//     x = (v >> 20) h' + (v >> 8), lutm = lut - 2^26 (two IMADs, no LOP3);
//   * the window shift w = w2 is a multiply by an opaque 1 (not a SEL);
//   * both renormalisation bytes come from ONE PRMT of the 8-byte register
//     window, and the window moves every second step (below).
// Measured on 218M symbols: 246 -> 200 us.  Tried and slower: mul.hi for the
// shifts (the FMA pipe's IMAD.HI is not cheaper than the ALU shift), a
// warp-uniform branch for the rare second byte (VOTE + reconvergence),
// reloading both window words instead of rotating them (one more LDS).
#ifndef NZ_EXP_LUTBANK
#define NZ_EXP_LUTBANK 0  // timing experiment only (wrong output): every LUT gather conflict-free
#endif

#if NZ_EXP_LUTBANK
#define NZP_TRANSITION(lut, x, v)                                                            \
    do {                                                                                     \
        uint32_t h_ = ((x) >> kProbBits) - kProbScale;                                       \
        v = p_lds32(lut_lane + ((x) & 0xF80u) * 4u);                                         \
        x = ((v) >> 20) * h_ + ((v) >> 8);                                                   \
    } while (0)
#else
#define NZP_TRANSITION(lut, x, v)                                                            \
    do {                                                                                     \
        uint32_t a_, h_ = ((x) >> kProbBits) - kProbScale;                                   \
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a_) : "r"(x), "r"(lutm));                      \
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a_) : "r"(h_), "r"(0xFFFFC000u), "r"(a_));    \
        v = p_lds32(a_);                                                                     \
        x = ((v) >> 20) * h_ + ((v) >> 8);                                                   \
    } while (0)
#endif

#ifndef NZ_PBYTES
#define NZ_PBYTES 0
#endif
#ifndef NZ_FLO
#define NZ_FLO 1  // measured: 200 -> 190 us per 218M-symbol layer vs the predicated PRMT pair
#endif

#if NZ_PBYTES
// Renormalisation bytes loaded from shared memory one at a time (q is the
// byte pointer): both "need a byte" predicates are known right after the
// transition (x < 2^23, x < 2^15), so the two loads issue together and the
// byte insertion runs on the FMA pipe (x*256 + b) -- fewer ALU ops, but the
// byte loads add ~1.5 shared-memory wavefronts per step to the LUT's ~3.7
// and the kernel turns LSU-bound (measured slower than the window).
#define NZP_STEP(lut, x, q, o8, w, w2, v)                                                    \
    do {                                                                                     \
        NZP_TRANSITION(lut, x, v);                                                           \
        asm("{\n\t.reg .pred p1, p2;\n\t.reg .b32 b0, b1;\n\t"                                 \
            "setp.lt.u32 p1, %0, 8388608;\n\t"                                               \
            "setp.lt.u32 p2, %0, 32768;\n\t"                                                 \
            "@p1 ld.shared.u8 b0, [%1];\n\t"                                                 \
            "@p2 ld.shared.u8 b1, [%1+1];\n\t"                                               \
            "@p1 mad.lo.u32 %0, %0, 256, b0;\n\t"                                            \
            "@p1 add.u32 %1, %1, 1;\n\t"                                                     \
            "@p2 mad.lo.u32 %0, %0, 256, b1;\n\t"                                            \
            "@p2 add.u32 %1, %1, 1;\n\t}"                                                    \
            : "+r"(x), "+r"(q));                                                             \
    } while (0)
#define NZP_STEP_A NZP_STEP
#elif NZ_FLO
// Renormalisation as one funnel shift: the byte count comes from the leading
// zeros (FLO, on the otherwise idle XU pipe), n8 = 8 * bytes =
// (clz(x) - 1) & 0x18 = ~msb(2x) & 0x18 for x in [2^11, 2^31) (2x on the FMA
// pipe, one LOP3); the next two stream bytes are
// PRMTed big-endian into the top of t (selector nibbles 3,2 = k, k+1), and
// x = (x:t) << n8.  The selector advances by n8 * 0x220 (0x1100 per byte).
#define NZP_RENORM_FLO                                                                       \
    "mul.lo.u32 c, %0, 2;\n\t"                                                                \
    "bfind.u32 c, c;\n\t"                                                                    \
    "not.b32 c, c;\n\t"                                                                      \
    "and.b32 c, c, 24;\n\t"                                                                  \
    "prmt.b32 t, %3, %4, %2;\n\t"                                                            \
    "shf.l.clamp.b32 %0, t, %0, c;\n\t"                                                      \
    "mad.lo.u32 %2, c, 0x220, %2;\n\t"
#define NZP_STEP_A(lut, x, q, o8, w, w2, v)                                                  \
    do {                                                                                     \
        NZP_TRANSITION(lut, x, v);                                                           \
        asm("{\n\t.reg .b32 t, c;\n\t" NZP_RENORM_FLO "}"                                      \
            : "+r"(x), "+r"(q), "+r"(o8), "+r"(w), "+r"(w2));                                \
    } while (0)
#ifndef NZ_WSHIFT_MOV
#define NZ_WSHIFT_MOV 0  // 1: measured no faster (182.3-184.3 us either way)
#endif
#if NZ_WSHIFT_MOV
// Window shift as plain predicated moves/adds: the kernel is issue-bound
// (a conflict-free LUT gather, timed with NZ_EXP_LUTBANK, is no faster), so
// the instruction count per step is what matters, not the ALU/FMA balance.
#define NZP_STEP(lut, x, q, o8, w, w2, v)                                                    \
    do {                                                                                     \
        NZP_TRANSITION(lut, x, v);                                                           \
        asm("{\n\t.reg .pred q;\n\t.reg .b32 t, c;\n\t" NZP_RENORM_FLO                        \
            "setp.ge.u32 q, %2, 0x4000;\n\t"                                                 \
            "@q mov.b32 %3, %4;\n\t"                                                         \
            "@q add.u32 %1, %1, 4;\n\t"                                                      \
            "@q sub.u32 %2, %2, 0x4400;\n\t"                                                 \
            "@q ld.shared.u32 %4, [%1+4];\n\t}"                                              \
            : "+r"(x), "+r"(q), "+r"(o8), "+r"(w), "+r"(w2));                                \
    } while (0)
#else
#define NZP_STEP(lut, x, q, o8, w, w2, v)                                                    \
    do {                                                                                     \
        NZP_TRANSITION(lut, x, v);                                                           \
        asm("{\n\t.reg .pred q;\n\t.reg .b32 t, c;\n\t" NZP_RENORM_FLO                        \
            "setp.ge.u32 q, %2, 0x4000;\n\t"                                                 \
            "@q mad.lo.u32 %3, %4, %5, 0;\n\t"                                                \
            "@q add.u32 %1, %1, 4;\n\t"                                                      \
            "@q sub.u32 %2, %2, 0x4400;\n\t"                                                 \
            "@q ld.shared.u32 %4, [%1+4];\n\t}"                                              \
            : "+r"(x), "+r"(q), "+r"(o8), "+r"(w), "+r"(w2) : "r"(mc.one));                  \
    } while (0)
#endif
#else
// The window position is a PRMT selector sel = k | (k+1) << 4 (k = byte
// offset into the 8-byte window w:w2) instead of a bit offset: one PRMT
// extracts the next two bytes wherever they sit in the 8 bytes, so the
// window only has to move once every TWO steps (after a shift k <= 3, two
// steps read at most bytes k..k+3 <= 6).  Step A has no window shift, step B
// shifts when k >= 4.
#define NZP_RENORM_SEL                                                                       \
    "setp.lt.u32 q, %0, 8388608;\n\t"                                                        \
    "setp.lt.u32 r, %0, 32768;\n\t"                                                          \
    "prmt.b32 t, %3, %4, %2;\n\t"                                                            \
    "@q prmt.b32 %0, %0, t, 0x2104;\n\t"                                                     \
    "@q add.u32 %2, %2, 0x11;\n\t"                                                           \
    "@r prmt.b32 %0, %0, t, 0x2105;\n\t"                                                     \
    "@r add.u32 %2, %2, 0x11;\n\t"
#define NZP_STEP_A(lut, x, q, o8, w, w2, v)                                                  \
    do {                                                                                     \
        NZP_TRANSITION(lut, x, v);                                                           \
        asm("{\n\t.reg .pred q, r;\n\t.reg .b32 t;\n\t" NZP_RENORM_SEL "}"                     \
            : "+r"(x), "+r"(q), "+r"(o8), "+r"(w), "+r"(w2));                                \
    } while (0)
#define NZP_STEP(lut, x, q, o8, w, w2, v)                                                    \
    do {                                                                                     \
        NZP_TRANSITION(lut, x, v);                                                           \
        asm("{\n\t.reg .pred q, r;\n\t.reg .b32 t;\n\t" NZP_RENORM_SEL                       \
            "setp.ge.u32 q, %2, 0x54;\n\t"                                                   \
            "@q mad.lo.u32 %3, %4, %5, 0;\n\t"                                                \
            "@q add.u32 %1, %1, 4;\n\t"                                                      \
            "@q sub.u32 %2, %2, 0x44;\n\t"                                                   \
            "@q ld.shared.u32 %4, [%1+4];\n\t}"                                              \
            : "+r"(x), "+r"(q), "+r"(o8), "+r"(w), "+r"(w2) : "r"(mc.one));                  \
    } while (0)
#endif

// Lane setup for one unit: the lane's sub-range (start state/position, end
// state/position, symbol count) and the unit's payload window.
struct LaneJob {
    uint32_t x0, xe, cnt, err;
    uint32_t p0, pe;  // stream offsets relative to the unit's first chunk (< 2^32 apart)
};

// Raw index records of a lane's sub-range, loaded one unit ahead so the
// global-memory latency never sits on a warp's critical path: the chunk
// record, the lane's state and the next sub-range's (its end state), and the
// terms of its chunk-relative start / end positions (nzgpu_internal.cuh: the
// offset plus the unit position for anchored lanes; the end is the next
// sub-range's start, for lane 31 the next unit's position).  The last
// sub-range of a chunk ends at len - 4 instead (lane_job).
struct RawRec {
    uint4 ci;
    uint32_t st, st1, off, off1, ref;
};

// 16-bit index load zero-extended by the load itself (a C++ u16 -> u32
// conversion made ptxas mask the value right after the load, which then
// waited on it: long-scoreboard stalls at ~8 % of the kernel).
__device__ __forceinline__ uint32_t ldg_u16(const uint16_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Only loads here (their results are consumed a unit later, in lane_job):
// the unit position comes from a predicated load rather than a select, so no
// instruction waits on a load in this function.  Lane 31's end is the next
// unit's position (the next sub-range is that unit's lane 0, offset 0), which
// it loads into `off1`.
template <int LOG2K>
__device__ __forceinline__ RawRec load_raw(const DecodeDesc& d, uint32_t j, uint32_t nsub) {
    RawRec r{make_uint4(0, 0, 0, 0), 0u, 0u, 0u, 0u, 0u};
    if (j >= nsub) return r;
    uint32_t ch, jin;
    sub_to_chunk(d, LOG2K, j, ch, jin);
    r.ci = __ldg(d.chunk_info + ch);
    if (d.ck_state) {  // null for single-symbol tables (no index)
        const uint32_t lane = j & 31u;
        r.st = __ldg(d.ck_state + j);
        r.off = ldg_u16(d.ck_off + j);
        if (jin >= lane) r.ref = __ldg(d.ck_base + (j >> 5));  // anchored: the unit position
        if (j + 1 < nsub) {
            r.st1 = __ldg(d.ck_state + j + 1);
            if (lane == 31u) r.off1 = __ldg(d.ck_base + (j >> 5) + 1);
            else r.off1 = ldg_u16(d.ck_off + j + 1);
        }
    }
    return r;
}

template <int LOG2K>
__device__ __forceinline__ LaneJob lane_job(const DecodeDesc& d, uint32_t j, uint32_t nsub, bool single,
                                            const RawRec& raw, uint32_t lo0) {
    constexpr int K = 1 << LOG2K;
    LaneJob L{kStateLow, kStateLow, 0u, 0u, 0u, 0u};
    if (j >= nsub) return L;
    uint32_t ch, jin;
    sub_to_chunk(d, LOG2K, j, ch, jin);
    const uint4 ci = raw.ci;
    const uint64_t off = chunk_offset(ci);
    const uint32_t len = ci.z, nsym = ci.w;
    const uint32_t sym_in = jin << LOG2K;
    L.cnt = nsym > sym_in ? min((uint32_t)K, nsym - sym_in) : 0u;
    if (len < 4) L.err |= kErrTruncated;  // ans.hpp:231-233
    const uint32_t limit = len >= 4 ? len - 4 : 0;
    if (jin == 0) {
        // framing must agree with the index (ans.hpp:332-340); the chunk's first
        // lane starts from the stream's own final state (ans.hpp:235-236)
        if (ld_u32le_bytes(d.stream + off - 8) != nsym || ld_u32le_bytes(d.stream + off - 4) != len)
            L.err |= kErrLength;
        L.x0 = ld_u32le_bytes(d.stream + off + limit);
    }
    if (single) {
        if (jin == 0 && len >= 4 && (L.x0 != kStateLow || len != 4)) L.err |= L.x0 < kStateLow ? kErrTruncated : kErrDesync;
        L.p0 = L.pe = ci.x - lo0 + limit;
        return L;
    }
    // The last sub-range of a chunk ends on the reference's end-of-chunk
    // condition (x == 2^23 at len - 4, ans.hpp:252); the others on the next
    // sub-range's state and position.
    const bool last = sym_in + K >= nsym;
    if (jin != 0) L.x0 = raw.st;
    L.xe = last ? kStateLow : raw.st1;
    const uint32_t start = raw.off + raw.ref;
    const uint32_t end = last ? limit : raw.off1 + ((j & 31u) == 31u ? 0u : raw.ref);
    if (start > limit || end > limit) L.err |= kErrDesync;
    L.p0 = ci.x - lo0 + min(start, limit);  // chunk offsets of one unit differ by < 2^32
    L.pe = ci.x - lo0 + min(end, limit);
    return L;
}

template <int LOG2K, int P>
__global__ void __launch_bounds__(p_warps(LOG2K) * 32, NZ_PMINB) decode_persist_kernel(const DecodeDesc* __restrict__ descs,
                                                                      int ndesc,
                                                                      const uint32_t* __restrict__ cta_prefix,
                                                                      DecodeDesc one, uint32_t upc,
                                                                      uint32_t win_cap, MulConsts mc) {
    constexpr int K = 1 << LOG2K;
    // K = 128 sub-ranges are decoded and merged in two 64-symbol halves
    // through one 64-symbol exponent tile (the unit's window and the lane's
    // ANS state carry over), so shared memory and the merge are those of K = 64
    // while the per-unit work (index records, window TMA, hand-out) is spread
    // over twice the symbols.
    constexpr int KH = 1 << tile_log2(LOG2K);
    constexpr int HALVES = K / KH;
    constexpr int kPWarps = p_warps(LOG2K);  // shadows the default for this K
    constexpr uint32_t RW = exps_row_words(tile_log2(LOG2K));
    constexpr int G = KH / 8;  // 8-element merge groups per lane per half
    using HB = typename HalfBits<P>::T;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t lut_bar = sbase;
    const uint32_t lut = sbase + kPHeader;
    const uint32_t wregion = warp_region(LOG2K, win_cap);
    const uint32_t region = sbase + kPHeader + kLutBytes + warp * wregion;
    const uint32_t my_bar0 = region;  // two mbarriers per warp
    uint32_t* exps = reinterpret_cast<uint32_t*>(smem + (region - sbase) + kPWarpBars);
    const uint32_t winbuf0 = region + kPWarpBars + unit_words(LOG2K) * 4;  // 16-B aligned
    const uint32_t winstride = win_cap + 2 * K + 64;

    // ---- which tensor / unit range this CTA owns
    uint32_t cta = blockIdx.x;
    const DecodeDesc* dp = &one;
    if (descs) {
        int lo = 0, hi = ndesc - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(cta_prefix + mid) <= cta) lo = mid; else hi = mid - 1;
        }
        dp = descs + lo;
        cta -= __ldg(cta_prefix + lo);
    }
    const DecodeDesc d = *dp;
    const uint32_t nsub = (uint32_t)ceil_div(d.n, K);
    const uint32_t units = (nsub + 31) / 32;
    const uint32_t ubeg = cta * upc, uend = min(units, ubeg + upc);
    const bool single = d.flags & kFlagSingleSymbol;
    const bool fast_lossy = d.block_size >= 8 && !(d.flags & kFlagSlowLossy);
    // lossy, power-of-two B >= 32K/8: the unit's scale bytes come from one
    // load issued with the sign/mantissa prefetch (merge flavours 4..7)
    const int unit_scales = (P != 7 && fast_lossy && d.log2_block != 0xFFFFFFFFu &&
                             d.log2_block >= (uint32_t)LOG2K + 2)
                                ? min((int)d.log2_block - (LOG2K + 2), 3)
                                : -1;

    // Prologue: thread 0 arms the CTA's LUT copy; every warp's lane 0 inits
    // the warp's own two window barriers, so each warp can load its first
    // index records and issue its first window TMA before the CTA barrier
    // (a lone launch -- a small tensor -- pays this latency once, unhidden).
    if (threadIdx.x == 0) {
        *reinterpret_cast<uint32_t*>(smem + 16) = ubeg + 2 * kPWarps;  // dynamic unit counter
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(lut_bar));
        fence_mbar_init();
        if (!single) {
            p_expect_tx(lut_bar, kLutBytes);
            p_bulk(lut, d.lut, kLutBytes, lut_bar);
        }
    }
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(my_bar0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(my_bar0 + 8));
        fence_mbar_init();
    }
    __syncwarp();
    if (ubeg >= uend) {
        __syncthreads();
        if (!single) p_wait_token(lut_bar, 0);
        return;
    }

    // ---- per-warp pipeline over units u = ubeg + warp + i * kPWarps
    uint32_t err = 0;
    // stage unit u into buffer b: returns this lane's job, issues the window TMA
    // Positions are 32-bit offsets from the unit's first chunk (lane 0's,
    // whose 64-bit offset only lane 0 needs, for the TMA source).
    auto stage = [&](uint32_t u, int b, uint32_t& wa_out, const RawRec& raw) -> LaneJob {
        const uint32_t lo0 = __shfl_sync(0xFFFFFFFFu, raw.ci.x, 0);
        LaneJob L = lane_job<LOG2K>(d, u * 32 + lane, nsub, single, raw, lo0);
        const uint32_t a = __shfl_sync(0xFFFFFFFFu, L.p0, 0);
        const uint32_t last_lane = min(31u, nsub - u * 32 - 1);
        const uint32_t e = __shfl_sync(0xFFFFFFFFu, L.pe, last_lane);
        const uint32_t wa = a - ((lo0 + a) & 15u);             // 16-B aligned absolute start
        const uint32_t eb = e + ((0u - (lo0 + e)) & 15u);      // 16-B aligned absolute end
        uint32_t bytes = single ? 0u : eb - wa;
        if (!single && (e < a || bytes > win_cap)) {
            L.err |= kErrDesync;
            bytes = 0;
        }
        if (!single && lane == 0) {
            const uint32_t bar = my_bar0 + 8 * b;
            p_expect_tx(bar, bytes);
            if (bytes) p_bulk(winbuf0 + b * winstride, d.stream + (int64_t)chunk_offset(raw.ci) + (int32_t)wa, bytes, bar);
        }
        wa_out = wa;
        return L;
    };

    // Units are handed out dynamically: each warp starts with units
    // ubeg + warp and ubeg + kPWarps + warp, then takes the next free unit
    // of the CTA's range from a shared counter, so warps that drew cheaper
    // units take more and the CTA ends within about one unit of its average
    // (a static round-robin left ~7 % of SM time idle in the tail).
    // One predicated ATOMS by lane 0.  With a warp-uniform address ptxas
    // rewrites any shared atomic into a warp-aggregated one (vote, popc,
    // shuffle, reconvergence: ~20 instructions per unit); the address gets
    // a lane term that is zero at run time (mc.one == 1) but opaque to it.
    const uint32_t s_next = sbase + 16 + lane * (mc.one - 1u);
    auto grab = [&]() -> uint32_t {
        uint32_t v = 0;
        asm volatile(
            "{\n.reg .pred p;\nsetp.eq.u32 p, %1, 0;\n@p atom.shared.add.u32 %0, [%2], 1;\n}\n"
            : "+r"(v)
            : "r"(lane), "r"(s_next)
            : "memory");
        return __shfl_sync(0xFFFFFFFFu, v, 0);
    };
    uint32_t u = ubeg + warp, un = ubeg + kPWarps + warp, unn = 0;
    uint32_t wa_cur = 0, wa_nxt = 0;
    LaneJob cur{}, nxt{};
    RawRec raw_n{};  // index records of unit `un` (loaded one iteration early)
    if (u < uend) {
        const RawRec r0 = load_raw<LOG2K>(d, u * 32 + lane, nsub);
        if (un < uend) raw_n = load_raw<LOG2K>(d, un * 32 + lane, nsub);
        cur = stage(u, 0, wa_cur, r0);
    }
    __syncthreads();  // the LUT barrier is initialised (and the unit counter set)
    uint32_t tok = 0;
    if (!single) tok = p_wait_token(lut_bar, 0);
    const uint32_t lutt = lut + tok;
    const uint32_t lutm = lutt - (1u << 26);
    (void)lutm;
#if NZ_EXP_LUTBANK
    const uint32_t lut_lane = lutt + lane * 4u;  // (x & 0xF80) * 4 is a multiple of 128: bank = lane
#endif

    for (uint32_t i = 0; u < uend; ++i) {
        const int b = i & 1;
        if (un < uend) {
            nxt = stage(un, b ^ 1, wa_nxt, raw_n);
            unn = grab();
            if (unn < uend) raw_n = load_raw<LOG2K>(d, unn * 32 + lane, nsub);
        } else {
            unn = uend;
        }
        if constexpr (HALVES == 1) {
            const uint64_t sym0 = (uint64_t)u * 32 * K;
            const uint32_t unit_syms = (uint32_t)min((uint64_t)32 * K, d.n - sym0);
            const uint32_t groups = unit_syms >> 3;
            // sign/mantissa words of this unit: in flight during the decode
            const HB* gb = reinterpret_cast<const HB*>(d.mant + sym0 * (P + 1) / 8);
            const bool full = unit_syms == 32u * K;  // every unit but a tensor's last
            HB pre[G];
            uint2 sw = make_uint2(0u, 0u);  // this unit's scale bytes (unit_scales >= 0)
            if constexpr (P != 7) {
                if (unit_scales >= 0) {
                    const uint64_t idx0 = sym0 >> d.log2_block;
                    if (unit_scales == 0) sw = __ldg(reinterpret_cast<const uint2*>(d.scales + idx0));
                    else if (unit_scales == 1) sw.x = __ldg(reinterpret_cast<const uint32_t*>(d.scales + idx0));
                    else if (unit_scales == 2) sw.x = __ldg(reinterpret_cast<const uint32_t*>(d.scales + (idx0 & ~3ull))) >>
                                                      (8u * (uint32_t)(idx0 & 2u));
                    else sw.x = __ldg(d.scales + idx0);
                }
            }
            if (full) {
    #pragma unroll
                for (int gi = 0; gi < G; ++gi) pre[gi] = __ldcs(gb + lane + gi * 32);
            } else {
    #pragma unroll
                for (int gi = 0; gi < G; ++gi) {
                    const uint32_t g = lane + gi * 32;
                    if (g < groups) pre[gi] = __ldcs(gb + g);
                }
            }
            err |= cur.err;
            uint32_t* row = exps + lane * RW;
            if (single) {
                const uint32_t wv = d.single_symbol * 0x01010101u;
                for (uint32_t k = 0; k < (cur.cnt + 3) / 4; ++k) row[k] = wv;
            } else {
                const uint32_t t2 = p_wait_token(my_bar0 + 8 * b, (i >> 1) & 1);
                if (!cur.err && cur.cnt) {
                    const uint32_t wbase = winbuf0 + b * winstride + t2;
                    uint32_t x = cur.x0;
                    const uint32_t p = wbase + (cur.p0 - wa_cur);
    #if NZ_PBYTES
                    uint32_t q = p, o8 = 0, w0 = 0, w1 = 0;
    #elif NZ_FLO
                    uint32_t q = p & ~3u, o8 = (p & 3u) * 0x1100u + 0x100u;  // PRMT selector nibbles 3,2 = k, k+1
                    uint32_t w0 = p_lds32(q), w1 = p_lds32(q + 4);
    #else
                    uint32_t q = p & ~3u, o8 = (p & 3u) * 0x11u + 0x10u;  // PRMT selector k | (k+1) << 4
                    uint32_t w0 = p_lds32(q), w1 = p_lds32(q + 4);
    #endif
                    if (cur.cnt == (uint32_t)K) {
    #pragma unroll kPUnroll
                        for (uint32_t k = 0; k < (uint32_t)K / 4; ++k) {
                            uint32_t v0, v1, v2, v3;
                            NZP_STEP_A(lutt, x, q, o8, w0, w1, v0);
                            NZP_STEP(lutt, x, q, o8, w0, w1, v1);
                            NZP_STEP_A(lutt, x, q, o8, w0, w1, v2);
                            NZP_STEP(lutt, x, q, o8, w0, w1, v3);
                            row[k] = __byte_perm(__byte_perm(v0, v1, 0x0040), __byte_perm(v2, v3, 0x0040), 0x5410);
                        }
                    } else {
                        uint32_t word = 0;
                        for (uint32_t k = 0; k < cur.cnt; ++k) {
                            uint32_t v;
                            NZP_STEP(lutt, x, q, o8, w0, w1, v);
                            word |= (v & 0xFFu) << (8 * (k & 3));
                            if ((k & 3) == 3 || k + 1 == cur.cnt) {
                                row[k >> 2] = word;
                                word = 0;
                            }
                        }
                    }
                    const uint32_t pend = wbase + (cur.pe - wa_cur);
    #if NZ_PBYTES
                    const uint32_t pos = q;
    #elif NZ_FLO
                    const uint32_t pos = q + (o8 >> 12);
    #else
                    const uint32_t pos = q + (o8 & 0xFu);
    #endif
                    NZ_CHECK(q + 8 <= winbuf0 + b * winstride + winstride && q >= winbuf0 + b * winstride);
                if (x != cur.xe || pos != pend) err |= pos > pend ? kErrTruncated : kErrDesync;
                }
            }
            __syncwarp();
            // ---- merge this unit: 8-element groups, one coalesced 16-B store per lane
            // group g = lane + 32 gi starts at element 8g: row (8g) / K, word ((8g) % K) / 4,
            // i.e. a per-lane base plus a compile-time stride per gi (K <= 256)
            uint4* out = reinterpret_cast<uint4*>(d.out + sym0);
            const uint32_t* erow = exps + (lane >> (LOG2K - 3)) * RW + (lane & ((K >> 3) - 1)) * 2;
            // one fully unrolled loop per merge flavour, chosen once per unit
            auto merge_groups = [&](auto flavour, auto full_unit) {
                // 0 lossless, 1 lossy pow2 B, 2 lossy any B, 3 float path,
                // 4..7 lossy pow2 B with 8/4/2/1 scale bytes per unit (B >= 32K/8)
                constexpr int M = decltype(flavour)::value;
                constexpr bool FULL = decltype(full_unit)::value;
                uint32_t blk0 = 0, rem0 = 0;
                if constexpr (M == 1) {
                    blk0 = (uint32_t)(sym0 >> d.log2_block);
                    rem0 = (uint32_t)sym0 & (d.block_size - 1u);
                }
                // M >= 4: a unit (32K elements, 32K-aligned) spans NB whole blocks
                // and merge group gi (elements 256 gi .. +255 of the unit) lies in
                // block gi * NB / G -- one broadcast load for the unit (`sw`, issued
                // with the sign/mantissa prefetch before the decode), then each
                // group's bf16x2 coefficient 0x3F80|s is one PRMT with a constant
                // selector (scale bytes are < 128 on this path).  The load stays
                // inside the scale section: it starts NB-aligned and sections are
                // padded to 256 bytes.
                uint32_t sw0 = 0, sw1 = 0;
                if constexpr (M >= 4) {
                    sw0 = sw.x | 0x80808080u;
                    sw1 = sw.y | 0x80808080u;
                }
    #pragma unroll
                for (int gi = 0; gi < G; ++gi) {
                    const uint32_t g = lane + gi * 32;
                    if (!FULL && g >= groups) break;
                    const HB s = pre[gi];
                    const uint32_t e = g << 3;
                    const uint32_t* er = erow + gi * ((256 >> LOG2K) * RW);
                    const uint32_t e0 = er[0], e1 = er[1];
                    if constexpr (M == 0) {
                        NZ_CHECK(sym0 + 8ull * g + 8 <= d.n);
                    __stcs(out + g, merge8(e0, hb_lo(s), e1, hb_hi(s)));
                    } else if constexpr (M >= 4) {
                        constexpr int NB = 8 >> (M - 4);
                        const uint32_t k = (uint32_t)(gi * NB / G);  // constant after unrolling
                        const uint32_t cp = __byte_perm(k < 4 ? sw0 : sw1, 0x3F3F3F3Fu, 0x4040u | (k & 3u) | ((k & 3u) << 8));
                        NZ_CHECK(sym0 + 8ull * g + 8 <= d.n);
                    __stcs(out + g, lossy_merge8_cp<P>(e0, e1, hb_raw(s), cp));
                    } else if constexpr (M == 1) {
                        // power-of-two B >= 8: an aligned 8-group never straddles a block
                        const uint32_t c = scale_coef_bf16(__ldg(d.scales + blk0 + ((rem0 + e) >> d.log2_block)));
                        __stcs(out + g, lossy_merge8<P>(e0, e1, hb_raw(s), c, c, 8));
                    } else if constexpr (M == 2) {
                        const uint64_t gidx = sym0 + e;
                        const uint64_t b0 = gidx / d.block_size;
                        const uint32_t split = (uint32_t)min((uint64_t)8, (b0 + 1) * d.block_size - gidx);
                        const uint32_t c0 = scale_coef_bf16(__ldg(d.scales + b0));
                        const uint32_t c1 = split < 8 ? scale_coef_bf16(__ldg(d.scales + b0 + 1)) : c0;
                        __stcs(out + g, lossy_merge8<P>(e0, e1, hb_raw(s), c0, c1, split));
                    } else {
                        constexpr uint32_t W = P + 1;
                        uint32_t bits;
                        if constexpr (W == 4) bits = __byte_perm(hb_raw(s), 0, 0x0123);
                        else if constexpr (W == 2) bits = __byte_perm(hb_raw(s), 0, 0x0144);
                        else bits = hb_raw(s) << 24;
                        const uint32_t B = d.block_size;
                        const uint64_t gidx = sym0 + e;
                        const uint64_t b0 = gidx / B;
                        const float c0 = scale_coef(__ldg(d.scales + b0));
                        const uint32_t split = (uint32_t)min((uint64_t)8, (b0 + 1) * B - gidx);
                        const float c1 = split < 8 ? scale_coef(__ldg(d.scales + b0 + 1)) : c0;
                        const uint32_t ew[2] = {e0, e1};
                        uint32_t res[4];
    #pragma unroll
                        for (int qq = 0; qq < 8; ++qq) {
                            const uint32_t ex = (ew[qq >> 2] >> (8 * (qq & 3))) & 0xFFu;
                            const uint32_t item = (bits >> (32 - (qq + 1) * W)) & ((1u << W) - 1u);
                            float c = qq < (int)split ? c0 : c1;
                            if (B < 8 && qq >= (int)split) c = scale_coef(__ldg(d.scales + (gidx + qq) / B));
                            const uint32_t h = lossy_rebuild(item, ex, P, c);
                            if (qq & 1) res[qq >> 1] |= h << 16; else res[qq >> 1] = h;
                        }
                        __stcs(out + g, make_uint4(res[0], res[1], res[2], res[3]));
                    }
                }
            };
            auto merge_unit = [&](auto flavour) {
                if (full) merge_groups(flavour, std::true_type{});
                else merge_groups(flavour, std::false_type{});
            };
            if constexpr (P == 7) {
                merge_unit(std::integral_constant<int, 0>{});
            } else if (!fast_lossy) {
                merge_unit(std::integral_constant<int, 3>{});
            } else if (unit_scales >= 0) {
                // scale bytes per unit: 32K / B = 2^(3 - unit_scales) (1 when B >= 32K)
                if (unit_scales == 0) merge_unit(std::integral_constant<int, 4>{});
                else if (unit_scales == 1) merge_unit(std::integral_constant<int, 5>{});
                else if (unit_scales == 2) merge_unit(std::integral_constant<int, 6>{});
                else merge_unit(std::integral_constant<int, 7>{});
            } else if (d.log2_block != 0xFFFFFFFFu) {
                merge_unit(std::integral_constant<int, 1>{});
            } else {
                merge_unit(std::integral_constant<int, 2>{});
            }
            for (uint32_t ii = groups * 8 + lane; ii < unit_syms; ii += 32) {  // tensor tail (n % 8)
                const uint32_t ex = (exps[(ii >> LOG2K) * RW + ((ii & (K - 1)) >> 2)] >> (8 * (ii & 3))) & 0xFFu;
                const uint64_t gidx = sym0 + ii;
            NZ_CHECK(gidx < d.n);
                if constexpr (P == 7) {
                    const uint32_t sm = __ldg(d.mant + gidx);
                    d.out[gidx] = (uint16_t)(((sm & 0x80u) << 8) | (ex << 7) | (sm & 0x7Fu));
                } else {
                    d.out[gidx] = lossy_rebuild(packed_item(d.mant, gidx, P), ex, P,
                                                scale_coef(__ldg(d.scales + gidx / d.block_size)));
                }
            }
            __syncwarp();
        } else {
            const uint64_t sym0 = (uint64_t)u * 32 * K;
            const uint32_t unit_syms = (uint32_t)min((uint64_t)32 * K, d.n - sym0);
            // sign/mantissa words of this unit: in flight during the decode
            const HB* gb = reinterpret_cast<const HB*>(d.mant + sym0 * (P + 1) / 8);
            const bool full = unit_syms == 32u * K;  // every unit but a tensor's last
            uint2 sw = make_uint2(0u, 0u);  // this unit's scale bytes (unit_scales >= 0)
            if constexpr (P != 7) {
                if (unit_scales >= 0) {
                    const uint64_t idx0 = sym0 >> d.log2_block;
                    if (unit_scales == 0) sw = __ldg(reinterpret_cast<const uint2*>(d.scales + idx0));
                    else if (unit_scales == 1) sw.x = __ldg(reinterpret_cast<const uint32_t*>(d.scales + idx0));
                    else if (unit_scales == 2) sw.x = __ldg(reinterpret_cast<const uint32_t*>(d.scales + (idx0 & ~3ull))) >>
                                                      (8u * (uint32_t)(idx0 & 2u));
                    else sw.x = __ldg(d.scales + idx0);
                }
            }
            err |= cur.err;
            uint32_t* row = exps + lane * RW;
            // Element offset (within the unit) of merge group gi of this lane in
            // half h: group g = lane + 32 gi covers 8 elements of sub-range row
            // r = g / 8 (lane = row of the exponent tile), KH-symbol half h.  For
            // K = 64 (one half) this is simply 8 g.
            auto grp = [&](int gi, int h) -> uint32_t {  // element offset / 8
                if constexpr (HALVES == 1) return (uint32_t)(lane + 32 * gi);
                else return (uint32_t)(((lane >> 3) + 4 * gi) * (K / 8) + h * (KH / 8) + (lane & 7));
            };
            const uint32_t groups = unit_syms >> 3;
            // decoder state, carried across the halves of a K = 128 unit
            bool dec = false;
            uint32_t x = 0, q = 0, o8 = 0, w0 = 0, w1 = 0, wbase = 0;
            if (!single) {
                const uint32_t t2 = p_wait_token(my_bar0 + 8 * b, (i >> 1) & 1);
                dec = !cur.err && cur.cnt;
                if (dec) {
                    wbase = winbuf0 + b * winstride + t2;
                    x = cur.x0;
                    const uint32_t p = wbase + (cur.p0 - wa_cur);
    #if NZ_PBYTES
                    q = p;
    #elif NZ_FLO
                    q = p & ~3u;
                    o8 = (p & 3u) * 0x1100u + 0x100u;  // PRMT selector nibbles 3,2 = k, k+1
                    w0 = p_lds32(q);
                    w1 = p_lds32(q + 4);
    #else
                    q = p & ~3u;
                    o8 = (p & 3u) * 0x11u + 0x10u;  // PRMT selector k | (k+1) << 4
                    w0 = p_lds32(q);
                    w1 = p_lds32(q + 4);
    #endif
                }
            }
#pragma unroll kHalvesUnroll
            for (int h = 0; h < HALVES; ++h) {
                HB pre[G];
                if (full) {
    #pragma unroll
                    for (int gi = 0; gi < G; ++gi) pre[gi] = __ldcs(gb + grp(gi, h));
                } else {
    #pragma unroll
                    for (int gi = 0; gi < G; ++gi) {
                        const uint32_t g = grp(gi, h);
                        if (g < groups) pre[gi] = __ldcs(gb + g);
                    }
                }
                // this lane's symbols in half h
                const uint32_t hcnt = cur.cnt > (uint32_t)(h * KH) ? min((uint32_t)KH, cur.cnt - (uint32_t)(h * KH)) : 0u;
                if (single) {
                    const uint32_t wv = d.single_symbol * 0x01010101u;
                    for (uint32_t k = 0; k < (hcnt + 3) / 4; ++k) row[k] = wv;
                } else if (dec) {
#if NZ_FLO && !NZ_PBYTES
                    // the register window is the two words at q (an invariant of
                    // NZP_STEP): reload rather than keep it live across the merge
                    if (h > 0) {
                        w0 = p_lds32(q);
                        w1 = p_lds32(q + 4);
                    }
#endif
                    if (hcnt == (uint32_t)KH) {
    #pragma unroll kPUnroll
                        for (uint32_t k = 0; k < (uint32_t)KH / 4; ++k) {
                            uint32_t v0, v1, v2, v3;
                            NZP_STEP_A(lutt, x, q, o8, w0, w1, v0);
                            NZP_STEP(lutt, x, q, o8, w0, w1, v1);
                            NZP_STEP_A(lutt, x, q, o8, w0, w1, v2);
                            NZP_STEP(lutt, x, q, o8, w0, w1, v3);
                            row[k] = __byte_perm(__byte_perm(v0, v1, 0x0040), __byte_perm(v2, v3, 0x0040), 0x5410);
                        }
                    } else if (hcnt) {
                        uint32_t word = 0;
                        for (uint32_t k = 0; k < hcnt; ++k) {
                            uint32_t v;
                            NZP_STEP(lutt, x, q, o8, w0, w1, v);
                            word |= (v & 0xFFu) << (8 * (k & 3));
                            if ((k & 3) == 3 || k + 1 == hcnt) {
                                row[k >> 2] = word;
                                word = 0;
                            }
                        }
                    }
                    if (h == HALVES - 1) {
                        const uint32_t pend = wbase + (cur.pe - wa_cur);
    #if NZ_PBYTES
                        const uint32_t pos = q;
    #elif NZ_FLO
                        const uint32_t pos = q + (o8 >> 12);
    #else
                        const uint32_t pos = q + (o8 & 0xFu);
    #endif
                        NZ_CHECK(q + 8 <= winbuf0 + b * winstride + winstride && q >= winbuf0 + b * winstride);
                if (x != cur.xe || pos != pend) err |= pos > pend ? kErrTruncated : kErrDesync;
                    }
                }
                __syncwarp();
            // ---- merge this half: 8-element groups, one coalesced 16-B store per lane
            // group g = lane + 32 gi: exponent-tile row g / 8, words 2 (g % 8), +1,
            // i.e. a per-lane base plus a compile-time stride per gi
            uint4* out = reinterpret_cast<uint4*>(d.out + sym0);
            const uint32_t* erow = exps + (lane >> 3) * RW + (lane & 7) * 2;
            // one fully unrolled loop per merge flavour, chosen once per unit
            auto merge_groups = [&](auto flavour, auto full_unit) {
                // 0 lossless, 1 lossy pow2 B, 2 lossy any B, 3 float path,
                // 4..7 lossy pow2 B with 8/4/2/1 scale bytes per unit (B >= 128K)
                constexpr int M = decltype(flavour)::value;
                constexpr bool FULL = decltype(full_unit)::value;
                uint32_t blk0 = 0, rem0 = 0;
                if constexpr (M == 1) {
                    blk0 = (uint32_t)(sym0 >> d.log2_block);
                    rem0 = (uint32_t)sym0 & (d.block_size - 1u);
                }
                // M >= 4: a unit (32K elements, 32K-aligned) spans NB whole blocks
                // and merge group gi (tile rows 4 gi .. 4 gi + 3, i.e. unit elements
                // 4 gi K .. 4 (gi + 1) K - 1 with B >= 4K) lies in block gi * NB / G
                // -- one broadcast load for the unit (`sw`, issued with the
                // sign/mantissa prefetch before the decode), then each group's
                // bf16x2 coefficient 0x3F80|s is one PRMT with a constant selector
                // (scale bytes are < 128 on this path).  The load stays inside the
                // scale section: it starts NB-aligned and sections are padded to
                // 256 bytes.
                uint32_t sw0 = 0, sw1 = 0;
                if constexpr (M >= 4) {
                    sw0 = sw.x | 0x80808080u;
                    sw1 = sw.y | 0x80808080u;
                }
    #pragma unroll
                for (int gi = 0; gi < G; ++gi) {
                    const uint32_t g = grp(gi, h);
                    if (!FULL && g >= groups) continue;
                    const uint32_t e = g << 3;
                    const HB s = pre[gi];
                    const uint32_t* er = erow + gi * (4 * RW);
                    const uint32_t e0 = er[0], e1 = er[1];
                    if constexpr (M == 0) {
                        NZ_CHECK(sym0 + 8ull * g + 8 <= d.n);
                    __stcs(out + g, merge8(e0, hb_lo(s), e1, hb_hi(s)));
                    } else if constexpr (M >= 4) {
                        constexpr int NB = 8 >> (M - 4);
                        const uint32_t k = (uint32_t)(gi * NB / G);  // constant after unrolling
                        const uint32_t cp = __byte_perm(k < 4 ? sw0 : sw1, 0x3F3F3F3Fu, 0x4040u | (k & 3u) | ((k & 3u) << 8));
                        NZ_CHECK(sym0 + 8ull * g + 8 <= d.n);
                    __stcs(out + g, lossy_merge8_cp<P>(e0, e1, hb_raw(s), cp));
                    } else if constexpr (M == 1) {
                        // power-of-two B >= 8: an aligned 8-group never straddles a block
                        const uint32_t c = scale_coef_bf16(__ldg(d.scales + blk0 + ((rem0 + e) >> d.log2_block)));
                        __stcs(out + g, lossy_merge8<P>(e0, e1, hb_raw(s), c, c, 8));
                    } else if constexpr (M == 2) {
                        const uint64_t gidx = sym0 + e;
                        const uint64_t b0 = gidx / d.block_size;
                        const uint32_t split = (uint32_t)min((uint64_t)8, (b0 + 1) * d.block_size - gidx);
                        const uint32_t c0 = scale_coef_bf16(__ldg(d.scales + b0));
                        const uint32_t c1 = split < 8 ? scale_coef_bf16(__ldg(d.scales + b0 + 1)) : c0;
                        __stcs(out + g, lossy_merge8<P>(e0, e1, hb_raw(s), c0, c1, split));
                    } else {
                        constexpr uint32_t W = P + 1;
                        uint32_t bits;
                        if constexpr (W == 4) bits = __byte_perm(hb_raw(s), 0, 0x0123);
                        else if constexpr (W == 2) bits = __byte_perm(hb_raw(s), 0, 0x0144);
                        else bits = hb_raw(s) << 24;
                        const uint32_t B = d.block_size;
                        const uint64_t gidx = sym0 + e;
                        const uint64_t b0 = gidx / B;
                        const float c0 = scale_coef(__ldg(d.scales + b0));
                        const uint32_t split = (uint32_t)min((uint64_t)8, (b0 + 1) * B - gidx);
                        const float c1 = split < 8 ? scale_coef(__ldg(d.scales + b0 + 1)) : c0;
                        const uint32_t ew[2] = {e0, e1};
                        uint32_t res[4];
    #pragma unroll
                        for (int qq = 0; qq < 8; ++qq) {
                            const uint32_t ex = (ew[qq >> 2] >> (8 * (qq & 3))) & 0xFFu;
                            const uint32_t item = (bits >> (32 - (qq + 1) * W)) & ((1u << W) - 1u);
                            float c = qq < (int)split ? c0 : c1;
                            if (B < 8 && qq >= (int)split) c = scale_coef(__ldg(d.scales + (gidx + qq) / B));
                            const uint32_t h = lossy_rebuild(item, ex, P, c);
                            if (qq & 1) res[qq >> 1] |= h << 16; else res[qq >> 1] = h;
                        }
                        __stcs(out + g, make_uint4(res[0], res[1], res[2], res[3]));
                    }
                }
            };
            auto merge_unit = [&](auto flavour) {
                if (full) merge_groups(flavour, std::true_type{});
                else merge_groups(flavour, std::false_type{});
            };
            if constexpr (P == 7) {
                merge_unit(std::integral_constant<int, 0>{});
            } else if (!fast_lossy) {
                merge_unit(std::integral_constant<int, 3>{});
            } else if (unit_scales >= 0) {
                // scale bytes per unit: 32K / B = 2^(3 - unit_scales) (1 when B >= 32K)
                if (unit_scales == 0) merge_unit(std::integral_constant<int, 4>{});
                else if (unit_scales == 1) merge_unit(std::integral_constant<int, 5>{});
                else if (unit_scales == 2) merge_unit(std::integral_constant<int, 6>{});
                else merge_unit(std::integral_constant<int, 7>{});
            } else if (d.log2_block != 0xFFFFFFFFu) {
                merge_unit(std::integral_constant<int, 1>{});
            } else {
                merge_unit(std::integral_constant<int, 2>{});
            }
            for (uint32_t ii = (unit_syms & ~7u) + lane; ii < unit_syms; ii += 32) {  // tensor tail (n % 8)
                if ((int)((ii & (K - 1)) / KH) != h) continue;  // lies in the other half
                const uint32_t ex = (exps[(ii >> LOG2K) * RW + ((ii & (KH - 1)) >> 2)] >> (8 * (ii & 3))) & 0xFFu;
                const uint64_t gidx = sym0 + ii;
            NZ_CHECK(gidx < d.n);
                if constexpr (P == 7) {
                    const uint32_t sm = __ldg(d.mant + gidx);
                    d.out[gidx] = (uint16_t)(((sm & 0x80u) << 8) | (ex << 7) | (sm & 0x7Fu));
                } else {
                    d.out[gidx] = lossy_rebuild(packed_item(d.mant, gidx, P), ex, P,
                                                scale_coef(__ldg(d.scales + gidx / d.block_size)));
                }
            }
            __syncwarp();
            }  // halves
        }
        cur = nxt;
        wa_cur = wa_nxt;
        u = un;
        un = unn;
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
#if NZ_EXP_LUTBANK
    err = 0;
#endif
    if (lane == 0 && err) atomicOr(d.err, err);
}

// Largest per-unit payload window (32 sub-ranges) of a tensor.
template <int LOG2K>
__global__ void unit_window_max_kernel(DecodeDesc d, uint32_t* __restrict__ out) {
    const uint32_t nsub = (uint32_t)ceil_div(d.n, 1u << LOG2K);
    const uint32_t units = (nsub + 31) / 32;
    uint32_t best = 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < units; t += gridDim.x * blockDim.x) {
        const uint32_t sub0 = t * 32;
        uint64_t a, b;
        tile_window(d, sub0, min(32u, nsub - sub0), LOG2K, nsub, a, b);
        const uint64_t bytes = (uint64_t)(((b + 15) & ~15ull) - (a & ~15ull));
        best = max(best, (uint32_t)min(bytes, (uint64_t)0xFFFFFFFFu));
    }
    atomicMax(out, best);
}

// Both window maxima (per 32-sub-range unit for the persistent kernel, per
// `tile_subs`-sub-range tile for the tiles kernel) of many tensors in one
// launch: blockIdx.y picks the tensor, out[2y] / out[2y + 1] receive them
// (zeroed by the caller).
template <int LOG2K>
__global__ void windows_batch_kernel(const DecodeDesc* __restrict__ descs, uint32_t tile_subs,
                                     uint32_t* __restrict__ out) {
    const DecodeDesc d = descs[blockIdx.y];
    const uint32_t nsub = (uint32_t)ceil_div(d.n, 1u << LOG2K);
    const uint32_t units = (nsub + 31) / 32, tiles = (nsub + tile_subs - 1) / tile_subs;
    uint32_t bu = 0, bt = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < units; t += stride) {
        uint64_t a, b;
        tile_window(d, t * 32, min(32u, nsub - t * 32), LOG2K, nsub, a, b);
        bu = max(bu, (uint32_t)min((uint64_t)(((b + 15) & ~15ull) - (a & ~15ull)), (uint64_t)0xFFFFFFFFu));
    }
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < tiles; t += stride) {
        uint64_t a, b;
        tile_window(d, t * tile_subs, min(tile_subs, nsub - t * tile_subs), LOG2K, nsub, a, b);
        bt = max(bt, (uint32_t)min((uint64_t)(((b + 15) & ~15ull) - (a & ~15ull)), (uint64_t)0xFFFFFFFFu));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        bu = max(bu, __shfl_xor_sync(0xFFFFFFFFu, bu, o));
        bt = max(bt, __shfl_xor_sync(0xFFFFFFFFu, bt, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (bu) atomicMax(out + 2 * blockIdx.y, bu);
        if (bt) atomicMax(out + 2 * blockIdx.y + 1, bt);
    }
}

cudaError_t launch_windows_batch(int log2k, const DecodeDesc* descs, int count, uint32_t tile_subs, uint64_t max_units,
                                 uint32_t* out, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    const dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(max_units, 256), 148)), (unsigned)count);
    switch (log2k) {
        case 6: windows_batch_kernel<6><<<grid, 256, 0, s>>>(descs, tile_subs, out); break;
        case 7: windows_batch_kernel<7><<<grid, 256, 0, s>>>(descs, tile_subs, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------ launchers --
template <int LOG2K, int P>
static cudaError_t launch_p(const DecodeDesc* descs, int ndesc, const uint32_t* cta_prefix, const DecodeDesc& one,
                            uint32_t ctas, uint32_t upc, uint32_t win_cap, cudaStream_t s) {
    const uint32_t smem = persist_smem(LOG2K, win_cap);
    static SmemAttr attr;  // per device: one process may drive several GPUs
    if (cudaError_t e = attr.ensure((const void*)decode_persist_kernel<LOG2K, P>, smem)) return e;
    const MulConsts mc{1u};
    decode_persist_kernel<LOG2K, P><<<ctas, p_warps(LOG2K) * 32, smem, s>>>(descs, ndesc, cta_prefix, one, upc, win_cap,
                                                                          mc);
    return cudaGetLastError();
}

template <int LOG2K>
static cudaError_t launch_pk(int precision, const DecodeDesc* descs, int ndesc, const uint32_t* cta_prefix,
                             const DecodeDesc& one, uint32_t ctas, uint32_t upc, uint32_t win_cap, cudaStream_t s) {
    switch (precision) {
        case 7: return launch_p<LOG2K, 7>(descs, ndesc, cta_prefix, one, ctas, upc, win_cap, s);
        case 3: return launch_p<LOG2K, 3>(descs, ndesc, cta_prefix, one, ctas, upc, win_cap, s);
        case 1: return launch_p<LOG2K, 1>(descs, ndesc, cta_prefix, one, ctas, upc, win_cap, s);
        case 0: return launch_p<LOG2K, 0>(descs, ndesc, cta_prefix, one, ctas, upc, win_cap, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_decode_persist(int log2k, int precision, const DecodeDesc* descs, int ndesc,
                                  const uint32_t* cta_prefix, const DecodeDesc& one, uint32_t ctas, uint32_t upc,
                                  uint32_t win_cap, cudaStream_t s) {
    if (ctas == 0) return cudaSuccess;
    switch (log2k) {
        case 6: return launch_pk<6>(precision, descs, ndesc, cta_prefix, one, ctas, upc, win_cap, s);
        case 7: return launch_pk<7>(precision, descs, ndesc, cta_prefix, one, ctas, upc, win_cap, s);
        default: return cudaErrorInvalidValue;
    }
}

bool persist_fits(int log2k, uint32_t win_cap) {
    static thread_local int dev_cached = -1, optin = 0;  // queried once per device, not per launch
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        dev_cached = dev;
    }
    return persist_smem(log2k, win_cap) <= (uint32_t)optin;
}

// CTAs of the persistent kernel that fit on the device at once.
uint32_t persist_resident_ctas(int log2k, uint32_t win_cap) {
    const uint32_t smem = persist_smem(log2k, win_cap);
    int dev = 0, sms = 148, per_sm_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    uint32_t per_sm = smem ? (uint32_t)per_sm_smem / (smem + 1024) : 1;
    const uint32_t by_threads = 2048u / (uint32_t)(p_warps(log2k) * 32);
    if (per_sm > by_threads) per_sm = by_threads;
    if (per_sm < 1) per_sm = 1;
    return (uint32_t)sms * per_sm;
}

cudaError_t launch_unit_window_max(int log2k, const DecodeDesc& d, uint32_t* out, cudaStream_t s) {
    switch (log2k) {
        case 6: unit_window_max_kernel<6><<<148, 256, 0, s>>>(d, out); break;
        case 7: unit_window_max_kernel<7><<<148, 256, 0, s>>>(d, out); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace nzgpu
