// nzgpu_internal.cuh -- shared definitions of the B200 NeuZip codec kernels.
//
// Stream format (unchanged from the reference, ans.hpp:304-316):
//   [u32 nchunks] then per chunk [u32 nsym][u32 len][payload(len)]
//   payload = renormalisation bytes in decoder order || LE32(final state)
// Table: 256 x u16 frequencies summing to 4096 (ans.hpp:111-118).
//
// Side index (ours; NOT part of the reference format or the ratio), one
// record set per sub-range j of K symbols (global symbols [jK, jK+K)) and per
// warp unit u of 32 consecutive sub-ranges:
//   st[j]   u32  decoder state before symbol jK (= the encoder state after
//                encoding it);
//   base[u] u32  decoder byte position (from its chunk's payload start) of
//                sub-range 32u;
//   off[j]  u16  decoder byte position of sub-range j relative to base[u]
//                when sub-range 32u lies in j's chunk ("anchored"), else
//                relative to j's chunk start (a unit that straddles chunks).
// So a lane's position is one load and one add -- no warp scan -- and its end
// position is the next sub-range's (off[j+1], or base[u+1] for lane 31).
// Offsets stay below 31 * (1.5K + 2) < 2^16.  A sub-range must end on the
// next sub-range's state and position; the last one of a chunk on
// (2^23, len-4), the reference's end-of-chunk check (ans.hpp:252).  6 bytes
// per K symbols + 4 per 32K: 0.096 B/element at K = 64, 0.048 at K = 128.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace nzgpu {

constexpr uint32_t kProbBits = 12;          // ans.hpp:30
constexpr uint32_t kProbScale = 1u << 12;   // ans.hpp:31
constexpr uint32_t kStateLow = 1u << 23;    // ans.hpp:32
constexpr uint32_t kDefaultChunk = 65536;   // ans.hpp:33

// Device error word bits (sticky, OR-ed by kernels).
enum : uint32_t {
    kErrTruncated = 1u << 0,   // ans.hpp:232, :246
    kErrDesync = 1u << 1,      // ans.hpp:253
    kErrLength = 1u << 2,      // framing / count mismatch
    kErrZeroFreq = 1u << 3,    // ans.hpp:210-212 (invalid_argument)
    kErrNonFinite = 1u << 4,   // tensorstore.hpp:153-157
    kErrTable = 1u << 5,       // ans.hpp:99-101
};

// Packed decode LUT entry: sym | (slot - cum) << 8 | freq << 20.
// freq == 4096 (single-symbol table) does not fit; such tensors take the
// constant path (flag kFlagSingleSymbol).
__host__ __device__ inline uint32_t lut_entry(uint32_t sym, uint32_t bias, uint32_t freq) {
    return sym | (bias << 8) | (freq << 20);
}

// kFlagHas255: the table gives symbol 255 (exponent of Inf/NaN) a nonzero
// frequency, so decoded values may be non-finite; kFlagWideScale: a lossy
// scale byte >= 128 (never produced by compress_lossy, whose scales are 7-bit
// mantissas, but legal in an imported blob).  Either sends the lossy merge to
// the float path.
enum : uint32_t { kFlagSingleSymbol = 1u, kFlagHas255 = 4u, kFlagWideScale = 8u };
constexpr uint32_t kFlagSlowLossy = kFlagHas255 | kFlagWideScale;

// Per-symbol encoder constants (ans.hpp:209-219): x / f as one exact
// multiply-shift (Granlund-Montgomery), valid for the encoder's x < 2^31.
struct EncSym {
    uint32_t freq;
    uint32_t cum;
    uint32_t rcp;  // m = ceil(2^(31+l) / f), l = ceil(log2 f)
    uint32_t pad;  // shift 31 + l: x / f = (x * m) >> shift for x < 2^31
};

// K3 threads per CTA: chains are latency-bound and their byte stores cost one
// transaction per active lane (every lane writes a different chunk), so few
// lanes per warp, spread over many SMs.
#ifndef NZ_ENC_THREADS
#define NZ_ENC_THREADS 32
#endif

// One tensor of a (batched) encode launch: K3 encodes its chunks into
// per-chunk scratch slots, K4 scans and compacts them.  A launch covers many
// tensors so that their chunk chains run concurrently (one chain per thread).
struct EncTask {
    const uint8_t* exps;     // exponent symbols, n bytes
    const EncSym* enc;       // 256 encoder constants
    uint8_t* scratch;        // nchunks slots of slot_bytes (16-B aligned)
    uint32_t* plen;          // payload length per chunk
    uint32_t* ck_state;      // side index (st[], cnt[], base[]), or nullptr
    uint32_t* ck_base;
    uint16_t* ck_off;
    uint32_t* err;           // sticky error word
    uint4* chunk_info;       // K4 out: {off lo, off hi, len, nsym}
    uint8_t* hdr;            // K4 out: the stream's leading u32 chunk count
    unsigned long long* total;  // K4 out: serialized stream length
    uint64_t n;
    uint64_t slot_bytes;
    uint32_t chunk_syms;
    uint32_t log2k;
    uint32_t cta0;           // first K3 CTA of this tensor in the launch
    uint32_t pad_;
    uint64_t unit0;          // first warp unit of this tensor in the index-finalize launch
};

// One tensor of a batched table build (K2): histogram in, tables out.
struct TableTask {
    const unsigned long long* counts;
    uint16_t* freqs;
    EncSym* enc;
    uint32_t* lut;
    uint32_t* info;
};

// Device view of one compressed tensor, as the decode kernels consume it.
struct DecodeDesc {
    const uint8_t* stream;        // serialized stream (reference layout), 16-B aligned + 16 B pad
    const uint8_t* mant;          // lossless: n bytes (s<<7|m); lossy: packed (k+1)-bit items
    const uint8_t* scales;        // lossy block scale bytes
    const uint32_t* ck_state;     // side index: state per sub-range
    const uint32_t* ck_base;      //   position of sub-range 32u in its chunk
    const uint16_t* ck_off;       //   sub-range position within the unit / chunk
    const uint4* chunk_info;      // {payload offset lo, hi, len, nsym} per chunk
    const uint32_t* lut;          // 4096 packed decode entries
    uint16_t* out;                // bf16 output, 16-B aligned
    uint32_t* err;                // sticky error word
    uint64_t n;                   // elements
    uint32_t chunk_syms;          // uniform chunk size S (multiple of K)
    uint32_t flags;               // kFlagSingleSymbol | kFlagHas255
    uint32_t single_symbol;       // the exponent when kFlagSingleSymbol
    int32_t precision;            // 7 lossless, 0/1/3 lossy
    uint32_t block_size;          // lossy block size B
    uint32_t log2_spc;            // log2(S/K) when S/K is a power of two, else 0xFFFFFFFF
    uint32_t log2_block;          // log2(B) when B is a power of two, else 0xFFFFFFFF
};

// ------------------------------------------------------------------ PTX --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// TMA bulk copy global -> shared (cp.async.bulk, SASS UBLKCP); dst/src
// 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a global range (cp.async.bulk.prefetch.L2); 16-byte
// aligned address, size a multiple of 16.
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint32_t ld_u32le_bytes(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Bf16::from_float, bitfloat.hpp:25-32.
__device__ __forceinline__ uint16_t bf16_from_float(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x0040u);
    return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Lane-private 16-bit exponent counters in shared memory (K1 and the fused
// lossy kernel): counter (warp, bin, lane) at u16 index (warp*256 + bin)*32 +
// lane, so a warp's 32 increments touch at most two lanes per bank and need
// no match/atomic.  A lane counts at most kLaneMax elements (grids are sized
// for it), so 16 bits cannot overflow.
constexpr int kLaneHistWarps = 4;
constexpr uint32_t kLaneHistSmem = kLaneHistWarps * 256 * 32 * 2;  // 64 KiB
constexpr uint64_t kLaneMax = 65000;

// Sum every warp's and lane's counters of the CTA into the global histogram
// (call after a __syncthreads that follows the last increment).
__device__ __forceinline__ void lane_hist_flush(const uint32_t* lh, unsigned long long* counts) {
    for (int bin = threadIdx.x; bin < 256; bin += blockDim.x) {
        uint32_t sum = 0;
#pragma unroll
        for (int wp = 0; wp < kLaneHistWarps; ++wp) {
            const uint32_t* row = lh + (wp * 256 + bin) * 16;  // 32 u16 counters = 16 words
#pragma unroll
            for (int k = 0; k < 16; ++k) sum += (row[(k + bin) & 15] & 0xFFFFu) + (row[(k + bin) & 15] >> 16);
        }
        if (sum) atomicAdd(counts + bin, (unsigned long long)sum);
    }
}

// Bounds assertions of the checked build (NZ_CHECKS=1, libnzgpu_checks.so;
// tools/checked_suite.sh runs the GPU tests against it): a violated bound
// traps the kernel, so the launch fails loudly instead of touching memory
// it does not own.  Compiled out of the product library.
#ifndef NZ_CHECKS
#define NZ_CHECKS 0
#endif
#if NZ_CHECKS
#define NZ_CHECK(cond)      \
    do {                    \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define NZ_CHECK(cond) \
    do {               \
    } while (0)
#endif

// Per-device, thread-safe record of the dynamic shared-memory opt-in of one
// kernel: the attribute is per (device, function), so a process that drives
// several GPUs (one host thread per device) must set it on each of them.
// Raising it concurrently from two threads is harmless (same call twice).
#ifndef NZ_CARVEOUT
#define NZ_CARVEOUT 0
#endif
struct SmemAttr {
    static constexpr int kMaxDevices = 64;
    std::atomic<uint32_t> configured[kMaxDevices] = {};

    cudaError_t ensure(const void* func, uint32_t smem) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
        if (smem <= configured[dev].load(std::memory_order_acquire)) return cudaSuccess;
        e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
#if NZ_CARVEOUT
        // prefer the largest shared-memory carveout so a launch after a kernel
        // that used the default split need not wait for the SMs to reconfigure
        cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#endif
        uint32_t cur = configured[dev].load(std::memory_order_relaxed);
        while (cur < smem && !configured[dev].compare_exchange_weak(cur, smem, std::memory_order_acq_rel)) {
        }
        return cudaSuccess;
    }
};

}  // namespace nzgpu
