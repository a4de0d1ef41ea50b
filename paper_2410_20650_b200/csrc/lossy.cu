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
#include "nzgpu_internal.cuh"

namespace nzgpu {

// round_mantissa (bitfloat.hpp:82-98) + carry rule (tensorstore.hpp:184-194).
__device__ __forceinline__ void lossy_normalize(uint32_t bits, float c, int k, uint32_t& exponent,
                                                uint32_t& item) {
    const uint32_t nb = bf16_from_float(__fdiv_rn(__uint_as_float(bits << 16), c));
    const uint32_t s = nb >> 15;
    uint32_t e = (nb >> 7) & 0xFFu;
    uint32_t m = nb & 0x7Fu;
    const uint32_t drop = 7 - k;
    const uint32_t rem = m & ((1u << drop) - 1u);
    const uint32_t half = 1u << (drop - 1);
    uint32_t kept = m >> drop;
    if (rem > half || (rem == half && (kept & 1u))) kept += 1;
    if (kept >= (1u << k)) {       // carry
        if (e == 254) {
            m = (m >> drop) << drop;  // truncate_mantissa, bitfloat.hpp:102-105
        } else {
            e += 1;
            m = 0;
        }
    } else {
        m = kept << drop;
    }
    exponent = e;
    item = (s << k) | (m >> drop);
}

__device__ __forceinline__ float lossy_coef(uint32_t s) { return 1.0f + (float)s * (1.0f / 128.0f); }

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
        const float c = lossy_coef(scale);
        for (uint32_t i = lane; i < len; i += 32) {
            uint32_t e, item;
            lossy_normalize(__ldg(v + begin + i), c, k, e, item);
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

// Elementwise lossy round trip under an explicit scale byte (the exhaustive
// parity harness; mirrors oracles.hpp:129-153 / tensorstore.hpp:179-198, 229-236).
__global__ void lossy_roundtrip_kernel(const uint16_t* __restrict__ v, const uint8_t* __restrict__ sc, uint64_t n,
                                       int k, uint16_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float c = lossy_coef(sc[i]);
        uint32_t e, item;
        lossy_normalize(v[i], c, k, e, item);
        const uint32_t s = item >> k, m = item & ((1u << k) - 1u);
        const uint32_t normalized = (s << 15) | (e << 7) | (m << (7 - k));
        out[i] = bf16_from_float(__fmul_rn(__uint_as_float(normalized << 16), c));
    }
}

}  // namespace nzgpu
