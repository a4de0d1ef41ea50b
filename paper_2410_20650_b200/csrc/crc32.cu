// crc32.cu -- K9: CRC-32 (IEEE 802.3, reflected polynomial 0xEDB88320) of
// device-resident byte ranges, for the NZT container (crc32.hpp:26-43,
// tensorstore.hpp:339-343 / :449-457).
//
// The reference updates one 32-bit register byte by byte.  The register
// update is linear over GF(2), so with the register starting at 0 ("raw"
// CRC, no final xor):
//   raw(A || B) = raw(A) * x^(8|B|) mod P  xor  raw(B)
//   raw(zeros || B) = raw(B)
//   crc32(D) = raw(D) xor (0xFFFFFFFF * x^(8|D|) mod P) xor 0xFFFFFFFF.
// K9a: the data is conceptually front-padded with zeros to whole 16 KiB
// blocks; each warp computes one block's raw CRC -- every lane runs a
// slicing-by-4 table CRC over its own 512 contiguous bytes (16-byte loads),
// then a 5-level shuffle tree joins the lanes with the constants
// x^(8*512*2^k).  K9b joins the block CRCs with a tree over a power-of-two
// count (front-padded with zero blocks) using x^(8*16384*2^k).  The host
// joins sections (table, scales, stream, mantissas) and applies the
// init/xorout term -- a few GF(2) multiplies.
#include <mutex>

#include "nzgpu_internal.cuh"

namespace nzgpu {

constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr uint32_t kCrcLane = 512;               // bytes per lane
constexpr uint32_t kCrcBlock = 32 * kCrcLane;    // bytes per warp block (16 KiB)

struct CrcConsts {
    uint32_t lane[5];    // x^(8 * 512 * 2^k) mod P, k = 0..4
    uint32_t block[40];  // x^(8 * 16384 * 2^k) mod P
};

// a * b mod P in the reflected representation (x^0 = bit 31), as zlib's
// multmodp.
__host__ __device__ inline uint32_t gf2_mulmod(uint32_t a, uint32_t b) {
    uint32_t p = 0;
    for (uint32_t m = 1u << 31; m; m >>= 1) {
        if (a & m) p ^= b;
        b = (b & 1u) ? (b >> 1) ^ kCrcPoly : b >> 1;
    }
    return p;
}

// x^(8n) mod P (square-and-multiply over the bits of n).
__host__ __device__ inline uint32_t gf2_x8n(uint64_t n) {
    uint32_t r = 1u << 31;       // x^0
    uint32_t sq = 1u << 23;      // x^8
    while (n) {
        if (n & 1) r = gf2_mulmod(sq, r);
        sq = gf2_mulmod(sq, sq);
        n >>= 1;
    }
    return r;
}

__global__ void __launch_bounds__(256) crc_raw_blocks_kernel(const uint8_t* __restrict__ data, uint64_t len,
                                                             uint64_t pad, uint64_t nblocks,
                                                             const uint32_t* __restrict__ tables_g,
                                                             CrcConsts cc, uint32_t* __restrict__ out) {
    __shared__ uint32_t T[4][256];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) T[i >> 8][i & 255] = tables_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t wblock = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    if (wblock >= nblocks) return;
    // this lane's padded range -> data range [s, e)
    const uint64_t ps = wblock * kCrcBlock + (uint64_t)lane * kCrcLane;
    const uint64_t pe = ps + kCrcLane;
    const uint64_t s = ps > pad ? ps - pad : 0, e = pe > pad ? pe - pad : 0;
    uint32_t c = 0;
    auto byte_step = [&](uint32_t b) { c = T[0][(c ^ b) & 0xFFu] ^ (c >> 8); };
    auto word_step = [&](uint32_t w) {
        c ^= w;
        c = T[3][c & 0xFFu] ^ T[2][(c >> 8) & 0xFFu] ^ T[1][(c >> 16) & 0xFFu] ^ T[0][c >> 24];
    };
    if (e > s) {
        uint64_t i = s;
        const uint64_t base = reinterpret_cast<uintptr_t>(data);
        const uint64_t al = ((base + s + 15) & ~15ull) - base;  // first 16-B aligned data index
        const uint64_t head_end = e < al ? e : al;
        for (; i < head_end; ++i) byte_step(__ldg(data + i));
        for (; i + 16 <= e; i += 16) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(data + i));
            word_step(v.x);
            word_step(v.y);
            word_step(v.z);
            word_step(v.w);
        }
        for (; i < e; ++i) byte_step(__ldg(data + i));
    }
    // join lanes: raw(L || R) = raw(L) * x^(8|R|) ^ raw(R), |R| = 512 * 2^k
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint32_t r = __shfl_down_sync(0xFFFFFFFFu, c, 1 << k);
        if ((lane & ((2 << k) - 1)) == 0) c = gf2_mulmod(cc.lane[k], c) ^ r;
    }
    if (lane == 0) out[wblock] = c;
}

// Same result for large inputs, conflict-free: the four 256-entry tables
// are replicated per bank (word (t*256 + e)*32 + lane, 128 KiB), so every
// warp-wide lookup is one shared-memory wavefront instead of ~3.5; a
// persistent grid (one 512-thread CTA per SM) amortises the table fill.
constexpr int kCrcWideThreads = 512;
constexpr uint32_t kCrcWideSmem = 4 * 256 * 32 * 4;

__global__ void __launch_bounds__(kCrcWideThreads) crc_raw_blocks_wide_kernel(
    const uint8_t* __restrict__ data, uint64_t len, uint64_t pad, uint64_t nblocks,
    const uint32_t* __restrict__ tables_g, CrcConsts cc, uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t Tw[];
    for (int w = threadIdx.x; w < 4 * 256 * 32; w += blockDim.x) Tw[w] = __ldg(tables_g + (w >> 5));
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t tb = (uint32_t)__cvta_generic_to_shared(Tw) + lane * 4;  // bank = lane
    auto lk = [&](int t, uint32_t e) {
        uint32_t v;
        asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(tb + ((uint32_t)t << 15) + (e << 7)));
        return v;
    };
    const uint64_t warps = (uint64_t)gridDim.x * (kCrcWideThreads / 32);
    for (uint64_t wblock = blockIdx.x * (uint64_t)(kCrcWideThreads / 32) + (threadIdx.x >> 5); wblock < nblocks;
         wblock += warps) {
        const uint64_t ps = wblock * kCrcBlock + (uint64_t)lane * kCrcLane;
        const uint64_t pe = ps + kCrcLane;
        const uint64_t s = ps > pad ? ps - pad : 0, e = pe > pad ? pe - pad : 0;
        uint32_t c = 0;
        if (e > s) {
            uint64_t i = s;
            const uint64_t base = reinterpret_cast<uintptr_t>(data);
            const uint64_t al = ((base + s + 15) & ~15ull) - base;
            const uint64_t head_end = e < al ? e : al;
            for (; i < head_end; ++i) c = lk(0, (c ^ __ldg(data + i)) & 0xFFu) ^ (c >> 8);
            auto word = [&](uint32_t w) {
                const uint32_t x = c ^ w;
                c = lk(3, x & 0xFFu) ^ lk(2, __byte_perm(x, 0, 0x4441)) ^ lk(1, __byte_perm(x, 0, 0x4442)) ^
                    lk(0, x >> 24);
            };
            // 8 loads (128 B) in flight per lane before the serial CRC chain
            for (; i + 128 <= e; i += 128) {
                uint4 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = __ldg(reinterpret_cast<const uint4*>(data + i) + q);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    word(v[q].x);
                    word(v[q].y);
                    word(v[q].z);
                    word(v[q].w);
                }
            }
            for (; i + 16 <= e; i += 16) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(data + i));
                word(v.x);
                word(v.y);
                word(v.z);
                word(v.w);
            }
            for (; i < e; ++i) c = lk(0, (c ^ __ldg(data + i)) & 0xFFu) ^ (c >> 8);
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const uint32_t r = __shfl_down_sync(0xFFFFFFFFu, c, 1 << k);
            if ((lane & ((2 << k) - 1)) == 0) c = gf2_mulmod(cc.lane[k], c) ^ r;
        }
        if (lane == 0) out[wblock] = c;
    }
}

// Tree over v[0 .. 2^levels): the data's blocks occupy the tail, the front
// entries are zero blocks (raw CRC 0).  One CTA; v[0] holds the result.
__global__ void __launch_bounds__(1024) crc_join_kernel(uint32_t* __restrict__ v, int levels, CrcConsts cc) {
    const uint64_t nb2 = 1ull << levels;
    for (int k = 0; k < levels; ++k) {
        const uint64_t step = 1ull << (k + 1), half = 1ull << k;
        for (uint64_t i = threadIdx.x * step; i < nb2; i += (uint64_t)blockDim.x * step) {
            const uint32_t L = v[i];
            v[i] = (L ? gf2_mulmod(cc.block[k], L) : 0u) ^ v[i + half];
        }
        __syncthreads();
    }
}

}  // namespace nzgpu

// ------------------------------------------------------------------ host --
namespace nzgpu {

namespace {
struct CrcTables {
    uint32_t* d[64] = {};
};
CrcTables g_crc_tables;

void host_tables(uint32_t* t) {
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? kCrcPoly ^ (c >> 1) : c >> 1;
        t[i] = c;
    }
    for (int j = 1; j < 4; ++j)
        for (uint32_t i = 0; i < 256; ++i) t[j * 256 + i] = (t[(j - 1) * 256 + i] >> 8) ^ t[t[(j - 1) * 256 + i] & 0xFFu];
}

CrcConsts make_consts() {
    CrcConsts cc{};
    for (int k = 0; k < 5; ++k) cc.lane[k] = gf2_x8n((uint64_t)kCrcLane << k);
    for (int k = 0; k < 40; ++k) cc.block[k] = gf2_x8n((uint64_t)kCrcBlock << k);
    return cc;
}
}  // namespace

uint32_t crc_combine_raw(uint32_t raw_a, uint32_t raw_b, uint64_t len_b) {
    return gf2_mulmod(gf2_x8n(len_b), raw_a) ^ raw_b;
}

uint32_t crc_finalize(uint32_t raw, uint64_t len) { return raw ^ gf2_mulmod(gf2_x8n(len), 0xFFFFFFFFu) ^ 0xFFFFFFFFu; }

uint32_t crc_raw_from_final(uint32_t crc, uint64_t len) {
    return crc ^ 0xFFFFFFFFu ^ gf2_mulmod(gf2_x8n(len), 0xFFFFFFFFu);
}

// Raw CRC of a device byte range; synchronises `s`.
cudaError_t crc_raw_device(const uint8_t* d, uint64_t len, cudaStream_t s, uint32_t* raw) {
    *raw = 0;
    if (len == 0) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!g_crc_tables.d[dev]) {
        uint32_t t[1024];
        host_tables(t);
        if ((e = cudaMalloc(&g_crc_tables.d[dev], sizeof t)) != cudaSuccess) return e;
        if ((e = cudaMemcpy(g_crc_tables.d[dev], t, sizeof t, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    }
    static const CrcConsts cc = make_consts();
    const uint64_t nblocks = (len + kCrcBlock - 1) / kCrcBlock;
    const uint64_t pad = nblocks * kCrcBlock - len;
    int levels = 0;
    while ((1ull << levels) < nblocks) ++levels;
    const uint64_t nb2 = 1ull << levels, lead = nb2 - nblocks;
    // grow-only scratch per device (a stream-ordered allocation per call costs
    // milliseconds when the pool trims at every synchronisation)
    static std::mutex mu;
    static uint32_t* scratch[64] = {};
    static uint64_t scratch_n[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (scratch_n[dev] < nb2) {
        if (scratch[dev]) cudaFree(scratch[dev]);
        scratch[dev] = nullptr;
        scratch_n[dev] = 0;
        if ((e = cudaMalloc(&scratch[dev], nb2 * sizeof(uint32_t))) != cudaSuccess) return e;
        scratch_n[dev] = nb2;
    }
    uint32_t* v = scratch[dev];
    if (lead) cudaMemsetAsync(v, 0, lead * sizeof(uint32_t), s);
    if (len >= (64ull << 20)) {
        static bool attr[64] = {};
        if (!attr[dev]) {
            if ((e = cudaFuncSetAttribute(crc_raw_blocks_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kCrcWideSmem)) != cudaSuccess)
                return e;
            attr[dev] = true;
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        crc_raw_blocks_wide_kernel<<<(unsigned)sms, kCrcWideThreads, kCrcWideSmem, s>>>(
            d, len, pad, nblocks, g_crc_tables.d[dev], cc, v + lead);
    } else {
        const uint64_t threads = nblocks * 32;
        crc_raw_blocks_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(d, len, pad, nblocks,
                                                                               g_crc_tables.d[dev], cc, v + lead);
    }
    if (levels) crc_join_kernel<<<1, 1024, 0, s>>>(v, levels, cc);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(raw, v, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // before the scratch can be reused
    return e;
}

}  // namespace nzgpu
