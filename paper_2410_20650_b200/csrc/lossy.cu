// lossy.cu -- K6: NeuZip lossy inference variant, block normalisation +
// round-to-nearest mantissa truncation + (k+1)-bit packing
// (compress_lossy, tensorstore.hpp:141-208; bitfloat.hpp:82-143).
//
// Per block of B elements: argmax of |bits| (first index on ties,
// tensorstore.hpp:168-174), scale byte = its mantissa, c = 1 + s/128;
// every element is divided by c in FP32 (__fdiv_rn; bit-identical to the
// reference's double path for every finite bf16 and scale, see
// tests/test_oracle.py::test_lossy_fp32_arithmetic_is_exact_vs_double),
// rounded to bf16 (RNE), its mantissa rounded to k bits (RNE with carry into
// the exponent; exponent 254 truncates instead).  Exponents go to the ANS
// coder, (sign, k-bit mantissa) items to the packer.
#include <algorithm>

#include "nzgpu_internal.cuh"

namespace nzgpu {

// |x| / c correctly rounded to FP32, given rc = RN(1/c): one multiply and a
// Markstein correction (r = |x| - q0 c exactly, by FMA; q = RN(q0 + r rc))
// instead of the IEEE division subroutine -- the fused kernel was bound by
// the division.  Bit-identical to __fdiv_rn for every finite bf16 magnitude
// and every scale byte (tests/test_gpu_parity.py::
// test_gpu_lossy_elementwise_exhaustive checks all 65,280 x 256 pairs).
#ifndef NZ_LOSSY_FASTDIV
#define NZ_LOSSY_FASTDIV 1
#endif
__device__ __forceinline__ float div_coef(float ax, float c, float rc) {
#if NZ_LOSSY_FASTDIV
    const float q0 = __fmul_rn(ax, rc);
    const float r = __fmaf_rn(-q0, c, ax);
    return __fmaf_rn(r, rc, q0);
#else
    (void)rc;
    return __fdiv_rn(ax, c);
#endif
}

#ifndef NZ_LOSSY_FUSED
#define NZ_LOSSY_FUSED 1
#endif

// round_mantissa (bitfloat.hpp:82-98) + carry rule (tensorstore.hpp:184-194).
// The division runs on the magnitude; c > 0, so the sign is the input's and
// the quotient is finite and non-negative (inputs are finite), so the FP32 ->
// bf16 RNE needs no NaN case.  Rounding to k mantissa bits is one add:
// m + (half - 1) + lsb carries exactly when RNE rounds up, and a carry out of
// the mantissa lands in the exponent (e + 1, m = 0) by itself; only a carry
// out of exponent 254 (to the Inf pattern) is replaced by the truncation the
// reference applies there.
__device__ __forceinline__ void lossy_normalize(uint32_t bits, float c, float rc, int k, uint32_t& exponent,
                                                uint32_t& item) {
    const uint32_t u = __float_as_uint(div_coef(__uint_as_float((bits & 0x7FFFu) << 16), c, rc));
    const uint32_t nbm = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;  // Bf16::from_float, bitfloat.hpp:25-32
    const uint32_t drop = 7 - k;
    const uint32_t mask = (1u << drop) - 1u;
    // the tie-break bit is the kept mantissa's lsb: bit `drop` of m, which
    // for k = 0 (drop = 7) lies outside m -- kept is 0, even
    uint32_t r = (nbm + (mask >> 1) + ((nbm >> drop) & (k != 0 ? 1u : 0u))) & ~mask;
    if (r >= 0x7F80u) r = nbm & ~mask;  // truncate_mantissa, bitfloat.hpp:102-105
    exponent = r >> 7;
    item = ((bits >> 15) << k) | ((r & 0x7Fu) >> drop);
}

__device__ __forceinline__ float lossy_coef(uint32_t s) { return 1.0f + (float)s * (1.0f / 128.0f); }
__device__ __forceinline__ float lossy_rcoef(float c) { return __frcp_rn(c); }

// One warp per block (grid-stride over blocks).
__global__ void __launch_bounds__(256) lossy_normalize_kernel(const uint16_t* __restrict__ v, uint64_t n, int k,
                                                              uint32_t block, uint8_t* __restrict__ scales,
                                                              uint8_t* __restrict__ exps,
                                                              uint8_t* __restrict__ items,
                                                              uint32_t* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t nblocks = ceil_div(n, block);
    for (uint64_t b = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); b < nblocks; b += warps) {
        const uint64_t begin = b * block;
        const uint32_t len = (uint32_t)min((uint64_t)block, n - begin);
        // argmax of magnitude bits, first index wins (strict >).
        uint64_t key = 0;
        bool nonfinite = false;
        for (uint32_t i = lane; i < len; i += 32) {
            const uint32_t bits = __ldg(v + begin + i);
            nonfinite |= (bits & 0x7F80u) == 0x7F80u;
            const uint64_t kk = ((uint64_t)(bits & 0x7FFFu) << 32) | (0xFFFFFFFFu - i);
            key = kk > key ? kk : key;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, key, o);
            key = other > key ? other : key;
        }
        if (__any_sync(0xFFFFFFFFu, nonfinite)) {
            if (lane == 0) atomicOr(err, kErrNonFinite);
            continue;
        }
        const uint32_t max_at = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
        const uint32_t scale = __ldg(v + begin + max_at) & 0x7Fu;
        if (lane == 0) scales[b] = (uint8_t)scale;
        const float c = lossy_coef(scale), rc = lossy_rcoef(c);
        for (uint32_t i = lane; i < len; i += 32) {
            uint32_t e, item;
            lossy_normalize(__ldg(v + begin + i), c, rc, k, e, item);
            exps[begin + i] = (uint8_t)e;
            items[begin + i] = (uint8_t)item;
        }
    }
}

// pack_signed_mantissas (bitfloat.hpp:124-143): one thread per output byte.
__global__ void pack_items_kernel(const uint8_t* __restrict__ items, uint64_t n, int k, uint8_t* __restrict__ out,
                                  uint64_t nbytes) {
    const uint32_t w = (uint32_t)k + 1;
    const uint32_t per = 8 / w;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < nbytes; j += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t byte = 0;
        const uint64_t i0 = j * per;
        for (uint32_t q = 0; q < per; ++q) {
            const uint64_t i = i0 + q;
            const uint32_t val = i < n ? items[i] : 0u;
            byte |= val << (8 - w * (q + 1));
        }
        out[j] = (uint8_t)byte;
    }
}

// unpack_signed_mantissas (bitfloat.hpp:145-164): one thread per item.
__global__ void unpack_items_kernel(const uint8_t* __restrict__ packed, uint64_t n, int k, uint8_t* __restrict__ items) {
    const uint32_t w = (uint32_t)k + 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bit = i * w;
        const uint32_t shift = 8 - w - (uint32_t)(bit & 7);
        items[i] = (uint8_t)((packed[bit >> 3] >> shift) & ((1u << w) - 1u));
    }
}

// K6 fused: normalisation + exponent histogram + item packing for the full
// blocks of a tensor whose block size is B = 32*E (E in {8, 16, 32, 64}).
// One warp per block; lane l holds elements q*256 + 8l .. 8l+7 of the block
// (q < E/8), so every load and store is warp-coalesced.  The bf16 block is
// read once (the three-kernel path reads it twice and round-trips an item
// plane through HBM).  Per element: 2 B read, 1 B exponent + (k+1)/8 B
// packed written.  Exponents are counted in lane-private shared counters.
constexpr int kFusedLoads = 8;  // uint4 loads in flight per lane

// One tensor's share of K6 (the single launch and the batched one below).
struct LossyTask {
    const uint16_t* v;
    uint64_t nfull;
    uint8_t* scales;
    uint8_t* exps;
    uint8_t* packed;
    unsigned long long* counts;
    uint32_t* err;
};

template <int E, int K>
__device__ __forceinline__ void lossy_fused_body(const uint16_t* __restrict__ v, uint64_t nfull,
                                                 uint8_t* __restrict__ scales, uint8_t* __restrict__ exps,
                                                 uint8_t* __restrict__ packed, unsigned long long* __restrict__ counts,
                                                 uint32_t* __restrict__ err, uint32_t bx, uint32_t gx) {
    constexpr int Q = E / 8;                                      // uint4 per lane per block
    constexpr int U = kFusedLoads / Q > 0 ? kFusedLoads / Q : 1;  // blocks per warp iteration
    constexpr uint64_t B = 32 * E;
    constexpr uint32_t W = K + 1;
    extern __shared__ uint32_t lh[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < (int)(kLaneHistSmem / 4); i += blockDim.x) lh[i] = 0;
    __syncthreads();
    uint16_t* h = reinterpret_cast<uint16_t*>(lh) + warp * 256 * 32 + lane;
    const uint64_t nw = (uint64_t)gx * kLaneHistWarps;
    for (uint64_t g = bx * (uint64_t)kLaneHistWarps + warp; g * U < nfull; g += nw) {
        uint4 w[U][Q];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t b = g * U + u;
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (b < nfull) w[u][q] = __ldcs(reinterpret_cast<const uint4*>(v + b * B) + q * 32 + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t b = g * U + u;
            if (b >= nfull) break;
            // the block's largest magnitude (tensorstore.hpp:168-174: the
            // argmax's index only breaks ties between equal magnitudes, which
            // share their mantissa, so the scale byte is the max's mantissa);
            // an exponent-255 element is the max iff the block is non-finite
            uint32_t m2 = 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                m2 = __vmaxu2(m2, w[u][q].x & 0x7FFF7FFFu);
                m2 = __vmaxu2(m2, w[u][q].y & 0x7FFF7FFFu);
                m2 = __vmaxu2(m2, w[u][q].z & 0x7FFF7FFFu);
                m2 = __vmaxu2(m2, w[u][q].w & 0x7FFF7FFFu);
            }
            const uint32_t mmax = __reduce_max_sync(0xFFFFFFFFu, max(m2 & 0xFFFFu, m2 >> 16));
            if (mmax >= 0x7F80u) {
                if (lane == 0) atomicOr(err, kErrNonFinite);
                continue;
            }
            const uint32_t scale = mmax & 0x7Fu;
            if (lane == 0) scales[b] = (uint8_t)scale;
            const float c = lossy_coef(scale), rc = lossy_rcoef(c);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const uint32_t in[4] = {w[u][q].x, w[u][q].y, w[u][q].z, w[u][q].w};
                uint32_t e8[2] = {0, 0}, acc = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t e, item;
                    lossy_normalize((in[j >> 1] >> (16 * (j & 1))) & 0xFFFFu, c, rc, K, e, item);
                    h[e * 32] += 1;
                    e8[j >> 2] |= e << (8 * (j & 3));
                    acc = (acc << W) | item;  // pack_signed_mantissas: first item in the high bits
                }
                const uint64_t i0 = b * B + q * 256 + lane * 8;
                NZ_CHECK(i0 + 8 <= nfull * B);
                __stcs(reinterpret_cast<uint2*>(exps + i0), make_uint2(e8[0], e8[1]));
                if constexpr (K == 3) {
                    __stcs(reinterpret_cast<uint32_t*>(packed + i0 / 2), __byte_perm(acc, 0, 0x0123));
                } else if constexpr (K == 1) {
                    *reinterpret_cast<uint16_t*>(packed + i0 / 4) = (uint16_t)__byte_perm(acc, 0, 0x0001);
                } else {
                    packed[i0 / 8] = (uint8_t)acc;
                }
            }
        }
    }
    __syncthreads();
    lane_hist_flush(lh, counts);
}

template <int E, int K>
__global__ void __launch_bounds__(kLaneHistWarps * 32) lossy_fused_kernel(const uint16_t* __restrict__ v,
                                                                          uint64_t nfull,
                                                                          uint8_t* __restrict__ scales,
                                                                          uint8_t* __restrict__ exps,
                                                                          uint8_t* __restrict__ packed,
                                                                          unsigned long long* __restrict__ counts,
                                                                          uint32_t* __restrict__ err) {
    lossy_fused_body<E, K>(v, nfull, scales, exps, packed, counts, err, blockIdx.x, gridDim.x);
}

// K6 of a whole compress batch in one launch (blockIdx.y = tensor).
template <int E, int K>
__global__ void __launch_bounds__(kLaneHistWarps * 32) lossy_fused_batch_kernel(const LossyTask* __restrict__ tasks) {
    const LossyTask t = tasks[blockIdx.y];
    lossy_fused_body<E, K>(t.v, t.nfull, t.scales, t.exps, t.packed, t.counts, t.err, blockIdx.x, gridDim.x);
}

__global__ void zero_lossy_tasks_kernel(const LossyTask* __restrict__ tasks) {
    const LossyTask t = tasks[blockIdx.x];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) t.counts[i] = 0ull;
    if (threadIdx.x < 16) t.err[threadIdx.x] = 0u;
}

template <int E, int K>
static cudaError_t launch_fused(const uint16_t* v, uint64_t nfull, uint8_t* scales, uint8_t* exps, uint8_t* packed,
                                unsigned long long* counts, uint32_t* err, cudaStream_t s) {
    static SmemAttr attr;
    if (cudaError_t e = attr.ensure((const void*)lossy_fused_kernel<E, K>, kLaneHistSmem)) return e;
    constexpr uint64_t U = kFusedLoads / (E / 8) > 0 ? kFusedLoads / (E / 8) : 1;
    const uint64_t per_warp = kLaneMax / E;  // blocks a warp may count (16-bit lane counters)
    const uint64_t need = ceil_div(ceil_div(nfull, per_warp), kLaneHistWarps);
    const uint64_t want = ceil_div(ceil_div(nfull, U), kLaneHistWarps);
    const uint64_t grid = std::max<uint64_t>(need, std::min<uint64_t>(want, 148 * 3));
    lossy_fused_kernel<E, K><<<(unsigned)grid, kLaneHistWarps * 32, kLaneHistSmem, s>>>(v, nfull, scales, exps, packed,
                                                                                     counts, err);
    return cudaGetLastError();
}

template <int E>
static cudaError_t launch_fused_k(int k, const uint16_t* v, uint64_t nfull, uint8_t* scales, uint8_t* exps,
                                  uint8_t* packed, unsigned long long* counts, uint32_t* err, cudaStream_t s) {
    switch (k) {
        case 0: return launch_fused<E, 0>(v, nfull, scales, exps, packed, counts, err, s);
        case 1: return launch_fused<E, 1>(v, nfull, scales, exps, packed, counts, err, s);
        default: return launch_fused<E, 3>(v, nfull, scales, exps, packed, counts, err, s);
    }
}

template <int E, int K>
static cudaError_t launch_fused_batch(const LossyTask* tasks, int count, uint64_t max_nfull, cudaStream_t s) {
    static SmemAttr attr;
    if (cudaError_t e = attr.ensure((const void*)lossy_fused_batch_kernel<E, K>, kLaneHistSmem)) return e;
    constexpr uint64_t U = kFusedLoads / (E / 8) > 0 ? kFusedLoads / (E / 8) : 1;
    const uint64_t per_warp = kLaneMax / E;
    const uint64_t need = ceil_div(ceil_div(max_nfull, per_warp), kLaneHistWarps);
    const uint64_t want = ceil_div(ceil_div(max_nfull, U), kLaneHistWarps);
    const uint64_t gx = std::max<uint64_t>(need, std::min<uint64_t>(want, 148 * 3));
    zero_lossy_tasks_kernel<<<count, 256, 0, s>>>(tasks);
    lossy_fused_batch_kernel<E, K><<<dim3((unsigned)gx, (unsigned)count), kLaneHistWarps * 32, kLaneHistSmem, s>>>(tasks);
    return cudaGetLastError();
}

template <int E>
static cudaError_t launch_fused_batch_k(int k, const LossyTask* tasks, int count, uint64_t max_nfull, cudaStream_t s) {
    switch (k) {
        case 0: return launch_fused_batch<E, 0>(tasks, count, max_nfull, s);
        case 1: return launch_fused_batch<E, 1>(tasks, count, max_nfull, s);
        default: return launch_fused_batch<E, 3>(tasks, count, max_nfull, s);
    }
}

size_t lossy_task_bytes() { return sizeof(LossyTask); }
void lossy_task_fill(void* at, const uint16_t* v, uint64_t nfull, uint8_t* scales, uint8_t* exps, uint8_t* packed,
                     unsigned long long* counts, uint32_t* err) {
    *static_cast<LossyTask*>(at) = LossyTask{v, nfull, scales, exps, packed, counts, err};
}
bool lossy_batchable(uint64_t n, int k, uint32_t block) {
    return NZ_LOSSY_FUSED && (block == 256 || block == 512 || block == 1024 || block == 2048) &&
           (k == 0 || k == 1 || k == 3) && n % block == 0;
}
// K6 (with the histograms and error words zeroed) of every tensor of a
// lossy batch in one launch; every tensor must be lossy_batchable.
cudaError_t launch_lossy_prep_batch(const void* tasks, int count, int k, uint32_t block, uint64_t max_nfull,
                                    cudaStream_t s) {
    const auto* t = static_cast<const LossyTask*>(tasks);
    switch (block) {
        case 256: return launch_fused_batch_k<8>(k, t, count, max_nfull, s);
        case 512: return launch_fused_batch_k<16>(k, t, count, max_nfull, s);
        case 1024: return launch_fused_batch_k<32>(k, t, count, max_nfull, s);
        default: return launch_fused_batch_k<64>(k, t, count, max_nfull, s);
    }
}

__global__ void byte_hist_kernel(const uint8_t*, uint64_t, unsigned long long*);


// K6 launcher: scales, exponent plane + histogram, packed (sign, mantissa)
// items.  Full blocks of B in {256, 512, 1024, 2048} take the fused kernel;
// the remaining blocks (a ragged last block, or every block of another B)
// take normalise -> histogram -> pack through the `items` scratch plane.
cudaError_t launch_lossy_prep(const uint16_t* v, uint64_t n, int k, uint32_t block, uint8_t* scales, uint8_t* exps,
                              uint8_t* items, uint8_t* packed, uint64_t packed_len, unsigned long long* counts,
                              uint32_t* err, cudaStream_t s) {
    uint64_t nfull = 0;
    if (NZ_LOSSY_FUSED && (block == 256 || block == 512 || block == 1024 || block == 2048) && (k == 0 || k == 1 || k == 3)) {
        nfull = n / block;
        if (nfull) {
            const int E = (int)(block / 32);
            cudaError_t e = E == 8    ? launch_fused_k<8>(k, v, nfull, scales, exps, packed, counts, err, s)
                            : E == 16 ? launch_fused_k<16>(k, v, nfull, scales, exps, packed, counts, err, s)
                            : E == 32 ? launch_fused_k<32>(k, v, nfull, scales, exps, packed, counts, err, s)
                                      : launch_fused_k<64>(k, v, nfull, scales, exps, packed, counts, err, s);
            if (e != cudaSuccess) return e;
        }
    }
    const uint64_t begin = nfull * block;  // a multiple of 256: byte- and 16-byte aligned planes
    if (begin == n) return cudaSuccess;
    const uint64_t rest = n - begin, pbegin = begin * (uint64_t)(k + 1) / 8;
    auto grid = [](uint64_t work) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(work, 256), 148 * 16)); };
    lossy_normalize_kernel<<<grid(ceil_div(rest, block) * 32), 256, 0, s>>>(v + begin, rest, k, block, scales + nfull,
                                                                           exps + begin, items, err);
    byte_hist_kernel<<<grid(rest / 16 + 1), 256, 0, s>>>(exps + begin, rest, counts);
    pack_items_kernel<<<grid(packed_len - pbegin), 256, 0, s>>>(items, rest, k, packed + pbegin, packed_len - pbegin);
    return cudaGetLastError();
}

// Elementwise lossy round trip under an explicit scale byte (the exhaustive
// parity harness; mirrors oracles.hpp:129-153 / tensorstore.hpp:179-198, 229-236).
__global__ void lossy_roundtrip_kernel(const uint16_t* __restrict__ v, const uint8_t* __restrict__ sc, uint64_t n,
                                       int k, uint16_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float c = lossy_coef(sc[i]);
        uint32_t e, item;
        lossy_normalize(v[i], c, lossy_rcoef(c), k, e, item);
        const uint32_t s = item >> k, m = item & ((1u << k) - 1u);
        const uint32_t normalized = (s << 15) | (e << 7) | (m << (7 - k));
        out[i] = bf16_from_float(__fmul_rn(__uint_as_float(normalized << 16), c));
    }
}

}  // namespace nzgpu
