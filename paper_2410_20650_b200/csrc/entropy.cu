// entropy.cu -- K10: per-component histograms of bf16 tensors for the
// entropy report (entropy.hpp:17-94).
//
// One pass over the tensor (8 bf16 per 16-byte load): sign counts by ballot
// + popcount, exponent counts with warp-aggregated shared atomics (the
// exponent histogram of trained weights has a handful of hot bins), mantissa
// counts with plain shared atomics in 4 bank-spread copies (near-uniform),
// then one u64 global atomic per bin and CTA.  The entropies themselves are
// computed on the host from the 386 counts with the reference's formulas.
#include "nzgpu_internal.cuh"

namespace nzgpu {

constexpr int kMantCopies = 4;

__device__ __forceinline__ void exp_add(uint32_t* h, uint32_t e) {
    const uint32_t peers = __match_any_sync(__activemask(), e);
    if ((__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(h + e, (uint32_t)__popc(peers));
}

__global__ void __launch_bounds__(256) component_hist_kernel(const uint16_t* __restrict__ v, uint64_t n,
                                                             unsigned long long* __restrict__ counts) {
    __shared__ uint32_t he[256];
    __shared__ uint32_t hm[kMantCopies][128];
    __shared__ uint32_t neg;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) he[i] = 0;
    for (int i = threadIdx.x; i < kMantCopies * 128; i += blockDim.x) (&hm[0][0])[i] = 0;
    if (threadIdx.x == 0) neg = 0;
    __syncthreads();
    uint32_t* m = hm[(threadIdx.x >> 5) & (kMantCopies - 1)];
    uint32_t my_neg = 0;
    const uint64_t groups = n / 8;
    const uint4* v4 = reinterpret_cast<const uint4*>(v);
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 w = __ldcs(v4 + g);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            my_neg += __popc(ws[q] & 0x80008000u);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t b = (ws[q] >> (16 * h)) & 0xFFFFu;
                exp_add(he, (b >> 7) & 0xFFu);
                atomicAdd(m + (b & 0x7Fu), 1u);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) {  // tail
        const uint32_t b = v[groups * 8 + threadIdx.x];
        my_neg += b >> 15;
        atomicAdd(he + ((b >> 7) & 0xFFu), 1u);
        atomicAdd(m + (b & 0x7Fu), 1u);
    }
    // warp-reduce the sign count, one shared atomic per warp
    for (int o = 16; o; o >>= 1) my_neg += __shfl_xor_sync(0xFFFFFFFFu, my_neg, o);
    if ((threadIdx.x & 31) == 0 && my_neg) atomicAdd(&neg, my_neg);
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (he[b]) atomicAdd(counts + 2 + b, (unsigned long long)he[b]);
    for (int b = threadIdx.x; b < 128; b += blockDim.x) {
        uint32_t s = 0;
#pragma unroll
        for (int c = 0; c < kMantCopies; ++c) s += hm[c][b];
        if (s) atomicAdd(counts + 258 + b, (unsigned long long)s);
    }
    if (threadIdx.x == 0 && neg) atomicAdd(counts + 1, (unsigned long long)neg);
}

}  // namespace nzgpu
