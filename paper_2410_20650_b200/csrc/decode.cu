// decode.cu -- K8: sequential chunk decode.
//
// One thread per reference chunk runs exactly the reference's decoder loop
// and checks (ans_decode_chunk, ans.hpp:229-256).  Used to
//   (a) build the checkpoint side index of streams that did not come from our
//       encoder (e.g. produced by the CPU reference), validating them fully;
//   (b) decode streams whose chunk framing is irregular (chunk sizes that are
//       not a uniform multiple of the checkpoint stride), followed by
//       merge_plane_kernel.
// The hot path is decode_persist.cu (decode_tiles.cu when its unit windows
// do not fit in shared memory).
#include "decode_common.cuh"

namespace nzgpu {

__global__ void __launch_bounds__(128) seq_decode_kernel(const uint8_t* __restrict__ stream,
                                                         const uint4* __restrict__ chunk_info,
                                                         const uint64_t* __restrict__ chunk_sym0,
                                                         uint32_t chunk_syms, uint64_t nchunks,
                                                         const uint32_t* __restrict__ lut_g, uint32_t flags,
                                                         uint32_t log2k, uint32_t* __restrict__ ck_state,
                                                         uint32_t* __restrict__ ck_base, uint16_t* __restrict__ ck_off,
                                                         uint8_t* __restrict__ exps, uint32_t* __restrict__ err) {
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
    // side index (nzgpu_internal.cuh): state, unit position and offset of
    // every sub-range, recorded as the chunk decodes forward
    const uint64_t j0 = base >> log2k;  // the chunk's first sub-range
    for (uint32_t i = 0; i < nsym; ++i) {
        if (ck_state && ((base + i) & kmask) == 0) {
            const uint64_t j = (base + i) >> log2k, u = j >> 5;
            ck_state[j] = x;
            if ((j & 31) == 0) ck_base[u] = pos;
            const bool anchored = (u << 5) >= j0;
            ck_off[j] = (uint16_t)(pos - (anchored ? ck_base[u] : 0u));
        }
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

}  // namespace nzgpu
