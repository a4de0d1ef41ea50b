// encode.cu -- K3 (chunked rANS encode) and K4 (stream compaction) of the
// B200 NeuZip codec.
//
// K3 restates ans_encode_chunk (ans.hpp:202-225) one chunk per thread: the
// state is a single serial chain per chunk (format-inherent: one 32-bit
// state per 65,536-symbol chunk), so parallelism comes from chunks and the
// step is built for latency.  The reference's `state / f` and `state % f`
// become one exact Granlund-Montgomery division, q = (x m) >> (31 + l) for
// x < 2^31 (tests/test_oracle.py::test_encoder_exact_division_identity), and
// x/f << 12 + x%f = x + q (4096 - f).
// Renormalisation bytes are emitted in reverse consumption order, so they
// are written backwards from the end of a per-chunk scratch slot; the
// payload (ans.hpp:222-223) is then contiguous and in decoder order.
// Every K symbols the encoder also records the side index that lets the
// decoder split a chunk into independent sub-ranges (nzgpu_internal.cuh):
// the state, and the decoder byte positions -- known only once the chunk is
// done, so the backward pass records each sub-range's consumed bytes (emitted
// since the previous checkpoint, which in reverse order is the NEXT
// sub-range) and a forward pass over the chunk's sub-ranges turns them into
// unit positions and offsets at the end.
//
// K4 restates serialize_stream (ans.hpp:306-316): an exclusive scan of
// (8 + len) over chunks, then a copy of every payload behind its header.
#include <algorithm>

#include "nzgpu_internal.cuh"

#ifndef NZ_ENC_NOSTORE
#define NZ_ENC_NOSTORE 0
#endif
#ifndef NZ_ENC_PF
#define NZ_ENC_PF 1
#endif
#ifndef NZ_ENC_PTXSTORE
#define NZ_ENC_PTXSTORE 1
#endif
#ifndef NZ_ENC_PTXRENORM
#define NZ_ENC_PTXRENORM 1
#endif
#ifndef NZ_ENC_PTXOFF
#define NZ_ENC_PTXOFF 1
#endif
#ifndef NZ_ENC_PTXQUEUE
#define NZ_ENC_PTXQUEUE 1
#endif
#ifndef NZ_ENC_PF_WIN
#define NZ_ENC_PF_WIN 4096  // symbols per L2 prefetch step (power of two, multiple of 16)
#endif

namespace nzgpu {

// Task of CTA `blk`: the last task whose first CTA is <= blk (tasks are in
// launch order); `one` stands in for a device array when ntasks == 1.
__device__ __forceinline__ const EncTask& task_of(const EncTask* tasks, int ntasks, const EncTask& one, uint32_t blk) {
    if (!tasks) return one;
    int lo = 0, hi = ntasks - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tasks[mid].cta0 <= blk) lo = mid; else hi = mid - 1;
    }
    return tasks[lo];
}

// Stores of the encoder's outputs (scratch bytes/words, side index) as
// explicit global stores: through a generic pointer ptxas must assume a store
// may alias the shared-memory encoder table and cannot hoist the next
// steps' table loads above it.
#ifndef NZ_ENC_STG
#define NZ_ENC_STG 0  // measured slower (C1 2.48-2.64 vs 2.34 ms)
#endif
template <class T>
__device__ __forceinline__ void st_g(T* p, T v) {
#if NZ_ENC_STG
    __stcg(p, v);
#else
    *p = v;
#endif
}

// One encoder chain: the state of ans_encode_chunk (ans.hpp:202-225) for one
// chunk, plus where its renormalisation bytes go.
struct EncChain {
    uint32_t x;
    uint32_t emitted;
    uint8_t* out;     // direct byte stores: next byte goes to out[-1]
    uint8_t* base;    // slot start; with off: out = base + off (the PTX step's form)
    uint32_t off;
    uint32_t* wo;     // QUEUE: next word goes to wo[-1]
    uint32_t qlo, qhi, qc;
    uint64_t begin;   // first symbol of the chunk
};

// QUEUE: word stores from the byte queue (throughput: many chains per SM,
// where per-lane byte stores saturate L1); otherwise direct byte stores,
// fewer instructions per step for latency-bound launches of few chains.
//
// One warp per CTA (NZ_ENC_THREADS), and the launch bounds say so: with the
// register budget of a 32-thread, one-CTA bound ptxas schedules the step
// with 84 registers instead of 62, and a lone chain runs 2.23 instead of
// 2.88 ms on C1 (in-order issue: the stall cycles per step are what it
// saves).  Two chains per thread, interleaved, measured 2x slower.  The
// byte-queue kernel (many chains, throughput-bound) keeps the default
// bound: with the tight one it took 15.3 instead of 14.3 ms on 8 layers.
// CHECK: test every symbol's frequency (ans.hpp:210-212) -- needed for a
// caller's table (nzgpu_ans_encode); a table built from the data's own
// histogram gives every present symbol a nonzero frequency (ans.hpp:71-90).
template <bool QUEUE, bool CHECK>
__global__ void __launch_bounds__(QUEUE ? 128 : NZ_ENC_THREADS, QUEUE ? 0 : 1) ans_encode_kernel(const EncTask* __restrict__ tasks, int ntasks,
                                                         const __grid_constant__ EncTask one) {
    __shared__ EncSym enc[256];
    const EncTask& t = task_of(tasks, ntasks, one, blockIdx.x);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) enc[i] = t.enc[i];
    __syncthreads();
    const uint64_t n = t.n;
    const uint32_t chunk_syms = t.chunk_syms, log2_interval = t.log2k;
    uint32_t* const ck_state = t.ck_state;
    uint32_t* const ck_base = t.ck_base;
    uint16_t* const ck_off = t.ck_off;
    const uint64_t nchunks = ceil_div(n, chunk_syms);
    const uint64_t c = (blockIdx.x - t.cta0) * (uint64_t)blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    bool bad = false;
    const uint32_t kmask = (1u << log2_interval) - 1u;
    auto init = [&](EncChain& ch, uint64_t cc) {
        ch.x = kStateLow;
        ch.emitted = 0;
        ch.begin = cc * chunk_syms;
        // Renormalisation bytes go backwards from the slot's end - 4.  Every
        // lane writes a different chunk, so a byte store costs one L2 sector
        // per lane: with QUEUE the bytes are queued in a 64-bit register pair
        // (newest at the top, pulled in by funnel shifts) and leave as
        // aligned 32-bit words.
        uint8_t* const slot_end = t.scratch + (cc + 1) * t.slot_bytes;  // 16-byte aligned
        ch.out = slot_end - 4;
        ch.base = slot_end - t.slot_bytes;
        ch.off = (uint32_t)t.slot_bytes - 4;
        ch.wo = reinterpret_cast<uint32_t*>(slot_end - 4);
        ch.qlo = ch.qhi = ch.qc = 0;
    };
    // Branch-free step (lanes of a warp encode different chunks, so any
    // data-dependent branch diverges).  The serial chain is
    // x -> compare -> select -> IMAD.WIDE -> shift -> IMAD -> x; the byte
    // queue and the checkpoint record hang off it.
    auto step = [&](EncChain& ch, const EncSym& e, uint32_t i, bool may_ckpt) {
        uint32_t x = ch.x;
        const uint32_t limit = e.freq << 19;
        if constexpr (CHECK) bad |= e.freq == 0;  // ans.hpp:210-212
#if NZ_ENC_PTXQUEUE
        if constexpr (QUEUE) {
            // The byte queue as one branch-free PTX block: the renormalising
            // compares, the queue shift (two wrap funnel shifts), and -- when
            // four bytes are queued -- the word store at slot base + 32-bit
            // offset, all predicated (the C++ form branched per lane)
            uint32_t nb;
            NZ_CHECK(ch.off >= 4);
            asm volatile(
                "{\n\t.reg .pred p, q, w;\n\t.reg .b32 t, s8, sh, wd;\n\t.reg .b64 a;\n\t"
                "shr.u32 t, %1, 8;\n\t"
                "setp.ge.u32 p, %1, %6;\n\t"
                "setp.ge.u32 q, t, %6;\n\t"
                "selp.u32 %5, 1, 0, p;\n\t"
                "@q add.u32 %5, %5, 1;\n\t"
                "shl.b32 s8, %5, 3;\n\t"
                "shf.r.wrap.b32 %2, %2, %3, s8;\n\t"
                "shf.r.wrap.b32 %3, %3, %1, s8;\n\t"
                "add.u32 %4, %4, %5;\n\t"
                "setp.ge.u32 w, %4, 4;\n\t"
                "shl.b32 sh, %4, 3;\n\t"
                "sub.u32 sh, 64, sh;\n\t"
                "shf.r.clamp.b32 wd, %2, %3, sh;\n\t"
                "prmt.b32 wd, wd, 0, 0x0123;\n\t"
                "mad.wide.u32 a, %0, 1, %7;\n\t"
                "@w st.u32 [a+-4], wd;\n\t"
                "@w sub.u32 %0, %0, 4;\n\t"
                "@w sub.u32 %4, %4, 4;\n\t"
                "@p mov.b32 %1, t;\n\t"
                "@q shr.u32 %1, t, 8;\n\t}"
                : "+r"(ch.off), "+r"(x), "+r"(ch.qlo), "+r"(ch.qhi), "+r"(ch.qc), "=r"(nb)
                : "r"(limit), "l"(ch.base)
                : "memory");
            ch.emitted += nb;
        } else
#endif
#if NZ_ENC_PTXRENORM
        if constexpr (!QUEUE) {
            // ans.hpp:214-218 as one PTX block: emit x & 0xFF while
            // x >= f << 19 (at most twice) -- compares, predicated byte stores
            // at immediate offsets, the renormalised state, the byte count
            // and the pointer decrement (one IMAD.WIDE)
            uint32_t nb;
#if NZ_ENC_PTXOFF
            // the store address as slot base + 32-bit offset: one unsigned
            // IMAD.WIDE, where a 64-bit pointer decrement costs four
            NZ_CHECK(ch.off >= 2);
            asm volatile(
                "{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t.reg .b64 a;\n\t"
                "mad.wide.u32 a, %0, 1, %4;\n\t"
                "shr.u32 t, %1, 8;\n\t"
                "setp.ge.u32 p, %1, %3;\n\t"
                "setp.ge.u32 q, t, %3;\n\t"
                "@p st.u8 [a+-1], %1;\n\t"
                "@q st.u8 [a+-2], t;\n\t"
                "selp.u32 %2, 1, 0, p;\n\t"
                "@p mov.b32 %1, t;\n\t"
                "@q shr.u32 %1, t, 8;\n\t"
                "@q add.u32 %2, %2, 1;\n\t"
                "sub.u32 %0, %0, %2;\n\t}"
                : "+r"(ch.off), "+r"(x), "=r"(nb)
                : "r"(limit), "l"(ch.base)
                : "memory");
#else
            NZ_CHECK(ch.out - 2 >= t.scratch + (ch.begin / chunk_syms) * t.slot_bytes);
            asm volatile(
                "{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
                "shr.u32 t, %1, 8;\n\t"
                "setp.ge.u32 p, %1, %3;\n\t"
                "setp.ge.u32 q, t, %3;\n\t"
                "@p st.u8 [%0+-1], %1;\n\t"
                "@q st.u8 [%0+-2], t;\n\t"
                "selp.u32 %2, 1, 0, p;\n\t"
                "@p mov.b32 %1, t;\n\t"
                "@q shr.u32 %1, t, 8;\n\t"
                "@q add.u32 %2, %2, 1;\n\t"
                "mad.wide.s32 %0, %2, -1, %0;\n\t}"
                : "+l"(ch.out), "+r"(x), "=r"(nb)
                : "r"(limit)
                : "memory");
#endif
            ch.emitted += nb;
        } else
#endif
        {
        // ans.hpp:214-218: emit x & 0xFF while x >= f << 19 -- at most twice.
        const bool n1 = x >= limit, n2 = (x >> 8) >= limit;
        const uint32_t nb = (uint32_t)n1 + (uint32_t)n2;
        if constexpr (QUEUE) {
            ch.qlo = __funnelshift_r(ch.qlo, ch.qhi, 8 * nb);
            ch.qhi = __funnelshift_r(ch.qhi, x, 8 * nb);  // x & 0xFF first, then (x >> 8) & 0xFF
            ch.qc += nb;
            if (ch.qc >= 4) {  // the 4 oldest queued bytes, oldest at the highest address
                NZ_CHECK(reinterpret_cast<uint8_t*>(ch.wo - 1) >= t.scratch + (ch.begin / chunk_syms) * t.slot_bytes);
                st_g(--ch.wo, __byte_perm(__funnelshift_rc(ch.qlo, ch.qhi, 64 - 8 * ch.qc), 0, 0x0123));
                ch.qc -= 4;
            }
        } else {
            NZ_CHECK(ch.out - nb >= t.scratch + (ch.begin / chunk_syms) * t.slot_bytes);
#if NZ_ENC_PTXSTORE
            // both predicated byte stores at immediate offsets from the
            // pointer and its decrement as one IMAD.WIDE (ptxas otherwise
            // rebuilds each store address in 64-bit arithmetic)
            asm volatile(
                "{\n\t.reg .pred p, q;\n\t"
                "setp.ne.u32 p, %2, 0;\n\t"
                "setp.ne.u32 q, %3, 0;\n\t"
                "@p st.u8 [%0+-1], %1;\n\t"
                "@q st.u8 [%0+-2], %4;\n\t"
                "mad.wide.s32 %0, %5, -1, %0;\n\t}"
                : "+l"(ch.out)
                : "r"(x), "r"((uint32_t)n1), "r"((uint32_t)n2), "r"(x >> 8), "r"(nb)
                : "memory");
#else
#if !NZ_ENC_NOSTORE  // timing experiment only: the chain without its byte stores
            if (n1) st_g(ch.out - 1, (uint8_t)x);
            if (n2) st_g(ch.out - 2, (uint8_t)(x >> 8));
#endif
            ch.out -= nb;
#endif
        }
        ch.emitted += nb;
        x = n2 ? x >> 16 : (n1 ? x >> 8 : x);
        }
        // ans.hpp:219: (x/f << 12) + x%f + cum = x + (x/f)(4096 - f) + cum,
        // with x/f exact from one 64-bit multiply and shift (x < 2^31 here)
        const uint32_t q = (uint32_t)(((uint64_t)x * e.rcp) >> e.pad);
        x = q * (kProbScale - e.freq) + (x + e.cum);
        ch.x = x;
        if (may_ckpt && ck_state && (i & kmask) == 0) {
            const uint64_t j = (ch.begin + i) >> log2_interval;
            st_g(ck_state + j, x);
            // positions are final only once the chunk's length is known:
            // record -E_j (mod 2^16) and, for unit starts, E_j itself;
            // index_finalize_kernel adds the right reference (E_32u or len-4)
            st_g(ck_off + j, (uint16_t)(0u - ch.emitted));
            if ((j & 31) == 0) st_g(ck_base + (j >> 5), ch.emitted);
        }
    };
    auto finish = [&](EncChain& ch, uint64_t cc) {
        uint8_t* const slot_end = t.scratch + (cc + 1) * t.slot_bytes;
        // The last 1-3 queued bytes: one word whose low (4 - qc) bytes lie
        // below the payload start, inside the slot.
#if NZ_ENC_PTXQUEUE
        if (QUEUE) ch.wo = reinterpret_cast<uint32_t*>(ch.base + ch.off);  // the PTX queue step's position
#endif
        if (QUEUE && ch.qc) *--ch.wo = __byte_perm(ch.qhi, 0, 0x0123) << (32 - 8 * ch.qc);
        // ans.hpp:223: final state little-endian at the tail (aligned store).
        *reinterpret_cast<uint32_t*>(slot_end - 4) = ch.x;
        t.plen[cc] = ch.emitted + 4;
    };
#if NZ_ENC_PF
    // A lone chain (few chunks: one warp per SM) cannot hide the load of
    // its next 16-symbol block: ncu put 22 % of C1's stall samples on the
    // block's first use.  The chunk's symbols are pulled into L2 in one
    // bulk prefetch up front, and the block load is pinned where it is
    // issued (asm volatile: the compiler otherwise sinks it next to its
    // use, a whole block later than intended).
    auto ldblk = [](const uint8_t* p) {
        uint4 v;
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(p));
        return v;
    };
#else
    auto ldblk = [](const uint8_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); };
#endif
    auto sym_of = [](const uint32_t (&w)[4], int b) { return (w[b >> 2] >> (8 * (b & 3))) & 0xFFu; };


    EncChain ch;
    init(ch, c);
    const uint32_t len = (uint32_t)min((uint64_t)chunk_syms, n - ch.begin);
    const uint8_t* src = t.exps + ch.begin;
    uint32_t i = len;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (!ck_state || (kmask & 15) == 15)) {
        // 16 symbols per aligned load, walked backwards in registers; with
        // K a multiple of 16 only the block's first symbol can be a checkpoint
        for (const uint32_t top = len & ~15u; i > top;) {
            --i;
            step(ch, enc[__ldg(src + i)], i, true);
        }
#if NZ_ENC_PF
        // A rolling window: the 2W symbols below the walk are in (or on their
        // way to) L2.  Prefetching whole chunks up front overflows L2 once
        // there are thousands of chains (a layer's 3,328 chunks are 218 MB):
        // one layer 3.26 -> 2.85 ms, C1 2.24 -> 2.28 ms.  Keeping the whole-
        // chunk prefetch for launches that fit in L2 measured slower on both.
        constexpr uint32_t kPfWin = NZ_ENC_PF_WIN;
        if (i >= 16) {
            const uint32_t lo = i > 2 * kPfWin ? i - 2 * kPfWin : 0;
            prefetch_l2(src + lo, i - lo);
        }
#endif
        // table entries are loaded one step ahead so the shared-memory
        // latency stays off the state chain
        uint4 blk4 = i ? ldblk(src + i - 16) : make_uint4(0, 0, 0, 0);
        while (i) {
            i -= 16;
            const uint32_t w[4] = {blk4.x, blk4.y, blk4.z, blk4.w};
            if (i) blk4 = ldblk(src + i - 16);
#if NZ_ENC_PF
            if ((i & (kPfWin - 1)) == 0 && i >= 2 * kPfWin) prefetch_l2(src + i - 2 * kPfWin, kPfWin);
#endif
            EncSym cur = enc[w[3] >> 24];
#pragma unroll
            for (int b = 15; b >= 0; --b) {
                EncSym nxt;
                if (b > 0) nxt = enc[sym_of(w, b - 1)];
                step(ch, cur, i + b, b == 0);
                if (b > 0) cur = nxt;
            }
        }
    } else {
        while (i) {
            --i;
            step(ch, enc[__ldg(src + i)], i, true);
        }
    }
    if (bad) {
        atomicOr(t.err, kErrZeroFreq);
        return;
    }
    finish(ch, c);
}

// Side index positions after K3 (nzgpu_internal.cuh).  The encoder walks a
// chunk backwards, so it records E_j (renormalisation bytes from sub-range j
// to the chunk end) as -E_j mod 2^16 in off[j] and E_32u in base[u]; with
// the chunk lengths known, one warp per unit turns them into
//   base[u] = (len - 4) - E_32u                  (position of sub-range 32u)
//   off[j]  = E_32u - E_j       anchored lanes   (position - base[u])
//   off[j]  = (len' - 4) - E_j  other lanes      (position in their chunk)
// -- independent per unit, so the serial encoder chains carry none of it.
__global__ void __launch_bounds__(256) index_finalize_kernel(const EncTask* __restrict__ tasks, int ntasks,
                                                             const __grid_constant__ EncTask one,
                                                             uint64_t total_units) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < total_units; w += warps) {
        const EncTask* tp = &one;
        if (tasks) {
            int lo = 0, hi = ntasks - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (tasks[mid].unit0 <= w) lo = mid; else hi = mid - 1;
            }
            tp = tasks + lo;
        }
        const EncTask& t = *tp;
        const uint64_t u = w - t.unit0;
        const uint64_t nsub = ceil_div(t.n, 1ull << t.log2k);
        const uint64_t j = (u << 5) + lane;
        const uint32_t log2_spc_k = t.log2k;  // symbols -> chunk via the symbol index
        const uint64_t c0 = ((u << 5) << log2_spc_k) / t.chunk_syms;
        const uint32_t e32 = t.ck_base[u];
        const uint32_t total0 = t.plen[c0] - 4u;
        if (j < nsub) {
            const uint64_t c = (j << log2_spc_k) / t.chunk_syms;
            const uint32_t add = c == c0 ? e32 : t.plen[c] - 4u;
            t.ck_off[j] = (uint16_t)(t.ck_off[j] + add);
        }
        __syncwarp();
        if (lane == 0) t.ck_base[u] = total0 - e32;
    }
}

// Exclusive scan of (8 + len) over chunks -> chunk_info {off_lo, off_hi,
// len, nsym}; writes the stream's leading u32 chunk count and the total
// stream length.  One CTA of 1024 threads per task (blockIdx.x).
__global__ void __launch_bounds__(1024) stream_scan_kernel(const EncTask* __restrict__ tasks,
                                                           const __grid_constant__ EncTask one) {
    const EncTask& t = tasks ? tasks[blockIdx.x] : one;
    const uint32_t* __restrict__ payload_len = t.plen;
    const uint64_t n = t.n;
    const uint32_t chunk_syms = t.chunk_syms;
    const uint64_t nchunks = ceil_div(n, chunk_syms);
    uint4* __restrict__ chunk_info = t.chunk_info;
    uint8_t* __restrict__ stream = t.hdr;
    unsigned long long* __restrict__ total_out = t.total;
    __shared__ unsigned long long warp_sums[32];
    __shared__ unsigned long long carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 4;  // leading u32 chunk count
    __syncthreads();
    for (uint64_t base = 0; base < nchunks; base += blockDim.x) {
        const uint64_t c = base + tid;
        const unsigned long long v = c < nchunks ? 8ull + payload_len[c] : 0ull;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = warp_sums[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= o) w += y;
            }
            warp_sums[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long excl = carry + (warp ? warp_sums[warp - 1] : 0ull) + incl - v;
        if (c < nchunks) {
            const uint64_t off = excl + 8;  // payload start
            const uint32_t nsym = (uint32_t)min((uint64_t)chunk_syms, n - c * chunk_syms);
            chunk_info[c] = make_uint4((uint32_t)off, (uint32_t)(off >> 32), payload_len[c], nsym);
        }
        __syncthreads();
        if (tid == 0) carry += warp_sums[31];
        __syncthreads();
    }
    if (tid == 0) {
        const uint32_t cnt = (uint32_t)nchunks;
        stream[0] = cnt & 0xFF;
        stream[1] = (cnt >> 8) & 0xFF;
        stream[2] = (cnt >> 16) & 0xFF;
        stream[3] = cnt >> 24;
        *total_out = carry;
    }
}

// One CTA per chunk: header [nsym][len] + payload copy from the scratch slot.
__global__ void __launch_bounds__(256) stream_copy_kernel(const uint8_t* __restrict__ scratch,
                                                          uint64_t slot_bytes,
                                                          const uint4* __restrict__ chunk_info,
                                                          uint8_t* __restrict__ stream) {
    const uint64_t c = blockIdx.x;
    const uint4 ci = chunk_info[c];
    const uint64_t off = (uint64_t)ci.x | ((uint64_t)ci.y << 32);
    const uint32_t len = ci.z;
    const uint8_t* src = scratch + (c + 1) * slot_bytes - len;
    uint8_t* dst = stream + off;
    if (threadIdx.x < 8) {
        const uint32_t v = threadIdx.x < 4 ? ci.w : len;
        dst[-8 + (int)threadIdx.x] = (uint8_t)(v >> (8 * (threadIdx.x & 3)));
    }
    // Byte-granular head until dst is 4-aligned, then word copies assembled
    // from the (differently aligned) source with funnel shifts.
    const uint32_t head = (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3);
    for (uint32_t i = threadIdx.x; i < min(head, len); i += blockDim.x) dst[i] = src[i];
    if (len <= head) return;
    const uint32_t body = (len - head) / 4;
    const uint8_t* s = src + head;
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + head);
    const uint32_t mis = (uint32_t)((uintptr_t)s & 3);
    const uint32_t* sa = reinterpret_cast<const uint32_t*>(s - mis);
    for (uint32_t w = threadIdx.x; w < body; w += blockDim.x) {
        const uint32_t lo = __ldg(sa + w);
        const uint32_t hi = mis ? __ldg(sa + w + 1) : 0u;
        d[w] = mis ? __funnelshift_r(lo, hi, 8 * mis) : lo;
    }
    for (uint32_t i = head + body * 4 + threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
}

// K4 copy of many tensors in one launch: block b copies chunk b - chunk0 of
// the job whose chunk range holds it (binary search); a tensor's first block
// also writes its stream's leading u32 chunk count.
struct StreamCopyJob {
    const uint8_t* scratch;
    const uint4* chunk_info;
    uint8_t* stream;
    const uint8_t* hdr;
    uint64_t chunk0;
};

__global__ void __launch_bounds__(256) stream_copy_batch_kernel(const StreamCopyJob* __restrict__ jobs, int njobs,
                                                                uint64_t slot_bytes) {
    int lo = 0, hi = njobs - 1;
    const uint64_t blk = blockIdx.x;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].chunk0 <= blk) lo = mid; else hi = mid - 1;
    }
    const StreamCopyJob j = jobs[lo];
    const uint64_t c = blk - j.chunk0;
    if (c == 0 && threadIdx.x < 4) j.stream[threadIdx.x] = j.hdr[threadIdx.x];
    const uint4 ci = j.chunk_info[c];
    const uint64_t off = (uint64_t)ci.x | ((uint64_t)ci.y << 32);
    const uint32_t len = ci.z;
    const uint8_t* src = j.scratch + (c + 1) * slot_bytes - len;
    uint8_t* dst = j.stream + off;
    if (threadIdx.x < 8) {
        const uint32_t v = threadIdx.x < 4 ? ci.w : len;
        dst[-8 + (int)threadIdx.x] = (uint8_t)(v >> (8 * (threadIdx.x & 3)));
    }
    const uint32_t head = (uint32_t)((4 - ((uintptr_t)dst & 3)) & 3);
    for (uint32_t i = threadIdx.x; i < min(head, len); i += blockDim.x) dst[i] = src[i];
    if (len <= head) return;
    const uint32_t body = (len - head) / 4;
    const uint8_t* sb = src + head;
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + head);
    const uint32_t mis = (uint32_t)((uintptr_t)sb & 3);
    const uint32_t* sa = reinterpret_cast<const uint32_t*>(sb - mis);
    for (uint32_t w = threadIdx.x; w < body; w += blockDim.x) {
        const uint32_t lo32 = __ldg(sa + w);
        const uint32_t hi32 = mis ? __ldg(sa + w + 1) : 0u;
        d[w] = mis ? __funnelshift_r(lo32, hi32, 8 * mis) : lo32;
    }
    for (uint32_t i = head + body * 4 + threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
}

cudaError_t launch_stream_copy_batch(const void* jobs, int njobs, uint64_t total_chunks, uint64_t slot_bytes,
                                     cudaStream_t s) {
    if (!total_chunks) return cudaSuccess;
    stream_copy_batch_kernel<<<(unsigned)total_chunks, 256, 0, s>>>(static_cast<const StreamCopyJob*>(jobs), njobs,
                                                                   slot_bytes);
    return cudaGetLastError();
}
size_t stream_copy_job_bytes() { return sizeof(StreamCopyJob); }
void stream_copy_job_fill(void* at, const uint8_t* scratch, const uint4* chunk_info, uint8_t* stream,
                          const uint8_t* hdr, uint64_t chunk0) {
    *static_cast<StreamCopyJob*>(at) = StreamCopyJob{scratch, chunk_info, stream, hdr, chunk0};
}

cudaError_t launch_index_finalize(const EncTask* tasks, int ntasks, const EncTask& one, uint64_t total_units,
                                  cudaStream_t s) {
    if (!total_units) return cudaSuccess;
    const uint64_t blocks = std::min<uint64_t>(ceil_div(total_units, 8), 148 * 16);
    index_finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(tasks, ntasks, one, total_units);
    return cudaGetLastError();
}

// K3 launcher (the template kernels stay in this translation unit).
cudaError_t launch_encode(bool queue, bool check, unsigned ctas, unsigned threads, const EncTask* tasks, int ntasks,
                          const EncTask& one, cudaStream_t s) {
    if (queue && check)
        ans_encode_kernel<true, true><<<ctas, threads, 0, s>>>(tasks, ntasks, one);
    else if (queue)
        ans_encode_kernel<true, false><<<ctas, threads, 0, s>>>(tasks, ntasks, one);
    else if (check)
        ans_encode_kernel<false, true><<<ctas, threads, 0, s>>>(tasks, ntasks, one);
    else
        ans_encode_kernel<false, false><<<ctas, threads, 0, s>>>(tasks, ntasks, one);
    return cudaGetLastError();
}

// dst[i] = *src[i]: one readback of scattered per-tensor result words.
__global__ void gather_u32_kernel(const uint32_t* const* __restrict__ src, uint32_t* __restrict__ dst, int count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) dst[i] = *src[i];
}

}  // namespace nzgpu
