// split_table.cu -- K1 (bit split + exponent histogram) and K2 (frequency
// table build) of the B200 NeuZip codec.
//
// K1 replaces the serial split/count loop of compress_lossless
// (tensorstore.hpp:93-102): bf16 -> exponent plane + (s<<7|m) byte plane,
// 256-bin u64 histogram.  HBM-bound: 2 B read + 2 B written per element.
//
// K2 restates FrequencyTable::from_counts (ans.hpp:52-93) exactly in one CTA
// and also emits the derived tables the coder needs: cumulative starts and
// reciprocals for the encoder (ans.hpp:209-219) and the packed 4096-slot
// decode LUT (ans.hpp:137-147 slot_to_symbol, plus freq and slot-cum).
#include <algorithm>

#include "nzgpu_internal.cuh"

namespace nzgpu {

// ------------------------------------------------------------------ K1 ---
constexpr int kHistCopies = 8;

__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t e) {
    // Aggregate equal exponents across the warp first: weight-sharing
    // Gaussians put most lanes on a handful of bins.
    const uint32_t peers = __match_any_sync(__activemask(), e);
    const int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(&h[e], __popc(peers));
}

// Split 8 bf16 (one uint4) into 8 exponent bytes + 8 sign/mantissa bytes.
__device__ __forceinline__ void split8(uint4 w, uint2& e8, uint2& s8) {
    const uint32_t in[4] = {w.x, w.y, w.z, w.w};
    uint32_t e[4], s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t v = in[i];
        e[i] = ((v >> 7) & 0xFFu) | (((v >> 23) & 0xFFu) << 8);
        s[i] = (((v >> 8) & 0x80u) | (v & 0x7Fu)) | ((((v >> 24) & 0x80u) | ((v >> 16) & 0x7Fu)) << 8);
    }
    e8.x = e[0] | (e[1] << 16);
    e8.y = e[2] | (e[3] << 16);
    s8.x = s[0] | (s[1] << 16);
    s8.y = s[2] | (s[3] << 16);
}

__global__ void __launch_bounds__(256) split_hist_kernel(const uint16_t* __restrict__ v, uint64_t n,
                                                         uint8_t* __restrict__ exps,
                                                         uint8_t* __restrict__ signmant,
                                                         unsigned long long* __restrict__ counts) {
    __shared__ uint32_t hist[kHistCopies][256];
    for (int i = threadIdx.x; i < kHistCopies * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
    uint32_t* h = hist[(threadIdx.x >> 5) & (kHistCopies - 1)];

    const uint64_t groups = n / 8;
    const uint4* v4 = reinterpret_cast<const uint4*>(v);
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 w = __ldcs(v4 + g);
        uint2 e8, s8;
        split8(w, e8, s8);
        if (exps) reinterpret_cast<uint2*>(exps)[g] = e8;
        if (signmant) reinterpret_cast<uint2*>(signmant)[g] = s8;
        if (counts) {
#pragma unroll
            for (int b = 0; b < 4; ++b) hist_add(h, (e8.x >> (8 * b)) & 0xFFu);
#pragma unroll
            for (int b = 0; b < 4; ++b) hist_add(h, (e8.y >> (8 * b)) & 0xFFu);
        }
    }
    // Tail (n % 8 elements) in block 0.
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) {
        const uint64_t i = groups * 8 + threadIdx.x;
        const uint32_t b = v[i];
        const uint32_t e = (b >> 7) & 0xFFu;
        if (exps) exps[i] = (uint8_t)e;
        if (signmant) signmant[i] = (uint8_t)(((b >> 8) & 0x80u) | (b & 0x7Fu));
        if (counts) atomicAdd(&h[e], 1u);
    }
    if (!counts) return;
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        uint32_t sum = 0;
#pragma unroll
        for (int c = 0; c < kHistCopies; ++c) sum += hist[c][b];
        if (sum) atomicAdd(counts + b, (unsigned long long)sum);
    }
}

// K1 with per-lane private 16-bit counters in shared memory instead of
// warp-aggregated atomics (layout: kLaneHistWarps, nzgpu_internal.cuh).
constexpr int kLaneUnroll = 8;

// K1 body over one tensor for CTA `bx` of `gx` (the single-tensor launch and
// the batched launch below share it).
__device__ __forceinline__ void split_hist_lane_body(const uint16_t* __restrict__ v, uint64_t n,
                                                     uint8_t* __restrict__ exps, uint8_t* __restrict__ signmant,
                                                     unsigned long long* __restrict__ counts, uint32_t bx,
                                                     uint32_t gx) {
    extern __shared__ uint32_t lh[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < (int)(kLaneHistSmem / 4); i += blockDim.x) lh[i] = 0;
    __syncthreads();
    uint16_t* h = reinterpret_cast<uint16_t*>(lh) + warp * 256 * 32 + lane;
    const uint64_t groups = n / 8;
    const uint4* v4 = reinterpret_cast<const uint4*>(v);
    // Only 12 warps fit per SM (64 KiB of counters per CTA), so each thread
    // keeps kLaneUnroll 16-byte loads in flight to cover HBM latency.
    // The next batch's loads are issued before this batch is processed, so a
    // warp's loads stay in flight while it splits and counts.
    const uint64_t stride = (uint64_t)gx * blockDim.x;
    uint4 nx[kLaneUnroll];
    const uint64_t gfirst = bx * (uint64_t)blockDim.x + tid;
#pragma unroll
    for (int k = 0; k < kLaneUnroll; ++k)
        if (gfirst + k * stride < groups) nx[k] = __ldcs(v4 + gfirst + k * stride);
    for (uint64_t g0 = gfirst; g0 < groups; g0 += kLaneUnroll * stride) {
        uint4 w[kLaneUnroll];
#pragma unroll
        for (int k = 0; k < kLaneUnroll; ++k) w[k] = nx[k];
        const uint64_t gn = g0 + kLaneUnroll * stride;
#pragma unroll
        for (int k = 0; k < kLaneUnroll; ++k)
            if (gn + k * stride < groups) nx[k] = __ldcs(v4 + gn + k * stride);
#pragma unroll
        for (int k = 0; k < kLaneUnroll; ++k) {
            const uint64_t g = g0 + k * stride;
            if (g >= groups) break;
            uint2 e8, s8;
            split8(w[k], e8, s8);
            __stcs(reinterpret_cast<uint2*>(exps) + g, e8);
            __stcs(reinterpret_cast<uint2*>(signmant) + g, s8);
#pragma unroll
            for (int b = 0; b < 4; ++b) h[((e8.x >> (8 * b)) & 0xFFu) * 32] += 1;
#pragma unroll
            for (int b = 0; b < 4; ++b) h[((e8.y >> (8 * b)) & 0xFFu) * 32] += 1;
        }
    }
    if (bx == 0 && tid < (n & 7)) {  // tail (n % 8 elements)
        const uint64_t i = groups * 8 + tid;
        const uint32_t b = v[i];
        const uint32_t e = (b >> 7) & 0xFFu;
        exps[i] = (uint8_t)e;
        signmant[i] = (uint8_t)(((b >> 8) & 0x80u) | (b & 0x7Fu));
        h[e * 32] += 1;
    }
    __syncthreads();
    lane_hist_flush(lh, counts);
}

__global__ void __launch_bounds__(kLaneHistWarps * 32) split_hist_lane_kernel(const uint16_t* __restrict__ v,
                                                                              uint64_t n,
                                                                              uint8_t* __restrict__ exps,
                                                                              uint8_t* __restrict__ signmant,
                                                                              unsigned long long* __restrict__ counts) {
    split_hist_lane_body(v, n, exps, signmant, counts, blockIdx.x, gridDim.x);
}

// K1 of a whole compress batch in one launch (blockIdx.y = tensor): the
// small tensors (norms, the k/v projections) no longer cost a launch each.
struct SplitTask {
    const uint16_t* v;
    uint64_t n;
    uint8_t* exps;
    uint8_t* signmant;
    unsigned long long* counts;
    uint32_t* err;
};

__global__ void __launch_bounds__(kLaneHistWarps * 32) split_hist_lane_batch_kernel(const SplitTask* __restrict__ tasks) {
    const SplitTask t = tasks[blockIdx.y];
    split_hist_lane_body(t.v, t.n, t.exps, t.signmant, t.counts, blockIdx.x, gridDim.x);
}

// The batch's histograms and error words zeroed in one launch (block = task).
__global__ void zero_split_tasks_kernel(const SplitTask* __restrict__ tasks) {
    const SplitTask t = tasks[blockIdx.x];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) t.counts[i] = 0ull;
    if (threadIdx.x < 16) t.err[threadIdx.x] = 0u;
}

size_t split_task_bytes() { return sizeof(SplitTask); }
void split_task_fill(void* at, const uint16_t* v, uint64_t n, uint8_t* exps, uint8_t* signmant,
                     unsigned long long* counts, uint32_t* err) {
    *static_cast<SplitTask*>(at) = SplitTask{v, n, exps, signmant, counts, err};
}

cudaError_t launch_split_hist_batch(const void* tasks, int count, uint64_t max_n, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    static SmemAttr attr;
    if (cudaError_t e = attr.ensure((const void*)split_hist_lane_batch_kernel, kLaneHistSmem)) return e;
    const auto* t = static_cast<const SplitTask*>(tasks);
    zero_split_tasks_kernel<<<count, 256, 0, s>>>(t);
    const uint64_t threads = kLaneHistWarps * 32;
    const uint64_t want = ceil_div(max_n / 8 + 1, threads);
    const uint64_t need = ceil_div(max_n, threads * kLaneMax);  // 16-bit counters
    const uint64_t gx = std::max<uint64_t>(need, std::min<uint64_t>(want, 148 * 3));
    split_hist_lane_batch_kernel<<<dim3((unsigned)gx, (unsigned)count), (unsigned)threads, kLaneHistSmem, s>>>(t);
    return cudaGetLastError();
}

#ifndef NZ_HIST_LANE
#define NZ_HIST_LANE 1
#endif

// K1 launcher: exponent plane + sign/mantissa plane + exponent histogram.
cudaError_t launch_split_hist(const uint16_t* v, uint64_t n, uint8_t* exps, uint8_t* signmant,
                              unsigned long long* counts, cudaStream_t s) {
    if (NZ_HIST_LANE && exps && signmant && counts) {
        // per call: the attribute is per device, and the call is cheap
        cudaError_t e = cudaFuncSetAttribute(split_hist_lane_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kLaneHistSmem);
        if (e != cudaSuccess) return e;
        const uint64_t threads = kLaneHistWarps * 32;
        const uint64_t want = ceil_div(n / 8 + 1, threads);
        const uint64_t need = ceil_div(n, threads * kLaneMax);  // 16-bit counters
        const uint64_t grid = std::max<uint64_t>(need, std::min<uint64_t>(want, 148 * 3));
        split_hist_lane_kernel<<<(unsigned)grid, (unsigned)threads, kLaneHistSmem, s>>>(v, n, exps, signmant, counts);
        return cudaGetLastError();
    }
    const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n / 8 + 1, 256), 148 * 16));
    split_hist_kernel<<<(unsigned)grid, 256, 0, s>>>(v, n, exps, signmant, counts);
    return cudaGetLastError();
}

// Histogram of an exponent plane (lossy path: post-normalisation exponents,
// tensorstore.hpp:201-203).
__global__ void __launch_bounds__(256) byte_hist_kernel(const uint8_t* __restrict__ x, uint64_t n,
                                                        unsigned long long* __restrict__ counts) {
    __shared__ uint32_t hist[kHistCopies][256];
    for (int i = threadIdx.x; i < kHistCopies * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
    uint32_t* h = hist[(threadIdx.x >> 5) & (kHistCopies - 1)];
    const uint64_t groups = n / 16;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 w = reinterpret_cast<const uint4*>(x)[g];
        const uint32_t in[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int b = 0; b < 4; ++b) hist_add(h, (in[i] >> (8 * b)) & 0xFFu);
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 15)) atomicAdd(&h[x[groups * 16 + threadIdx.x]], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        uint32_t sum = 0;
#pragma unroll
        for (int c = 0; c < kHistCopies; ++c) sum += hist[c][b];
        if (sum) atomicAdd(counts + b, (unsigned long long)sum);
    }
}

// ------------------------------------------------------------------ K2 ---
// One CTA of 256 threads; thread s owns symbol s.
//   info[0] = flags (kFlagSingleSymbol), info[1] = that symbol,
//   info[2] |= error bits.
__device__ __forceinline__ void build_table_body(const unsigned long long* __restrict__ counts,
                                                 const uint16_t* __restrict__ given_freqs,
                                                 uint16_t* __restrict__ freqs_out,
                                                 EncSym* __restrict__ enc,
                                                 uint32_t* __restrict__ lut,
                                                 uint32_t* __restrict__ info) {
    __shared__ unsigned long long rem[256];
    __shared__ uint32_t freq[256];
    __shared__ uint32_t cum[257];
    __shared__ unsigned long long red[8];
    __shared__ uint32_t redf[8];
    const int s = threadIdx.x;
    const int lane = s & 31, warp = s >> 5;

    uint32_t f;
    if (given_freqs) {
        // FrequencyTable::from_frequencies (ans.hpp:96-103): sum must be 4096.
        f = given_freqs[s];
    } else {
        // ans.hpp:56-70: total, floor(c*4096/T), remainders.
        const unsigned long long c = counts[s];
        unsigned long long t = c;
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
        if (lane == 0) red[warp] = t;
        __syncthreads();
        unsigned long long total = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) total += red[w];
        if (total == 0) {  // ans.hpp:58-60 -> invalid_argument
            if (s == 0) atomicOr(info + 2, kErrZeroFreq);
            return;
        }
        const unsigned long long scaled = c * (unsigned long long)kProbScale;
        f = (uint32_t)(scaled / total);
        rem[s] = scaled % total;
        // ans.hpp:72-80: stable sort by remainder desc, +1 to the first
        // `deficit` entries.  Restated as a rank: the stable position of s.
        uint32_t a = f;
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
        if (lane == 0) redf[warp] = a;
        __syncthreads();
        uint32_t assigned = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) assigned += redf[w];
        const uint32_t deficit = kProbScale - assigned;
        const unsigned long long mine = rem[s];
        uint32_t rank = 0;
        for (int j = 0; j < 256; ++j) {
            const unsigned long long r = rem[j];
            rank += (r > mine) || (r == mine && j < s);
        }
        f += rank < deficit ? 1u : 0u;
        freq[s] = f;
        __syncthreads();
        // ans.hpp:83-91: floor-at-1 repair in ascending symbol order, donor =
        // first argmax of the current frequencies.  Warp 0, serial over the
        // symbols that need it (a repair never zeroes the donor: max >= 16).
        if (warp == 0) {
            for (int base = 0; base < 256; base += 32) {
                const int sym = base + lane;
                uint32_t need = __ballot_sync(0xFFFFFFFFu, counts[sym] > 0 && freq[sym] == 0);
                while (need) {
                    const int t = base + __ffs(need) - 1;
                    need &= need - 1;
                    uint32_t best = 0, best_i = 0;
                    for (int k = 0; k < 8; ++k) {  // lane owns symbols lane*8 .. lane*8+7
                        const uint32_t v = freq[lane * 8 + k];
                        if (v > best) { best = v; best_i = lane * 8 + k; }
                    }
                    // first argmax: larger value wins, ties to the lower index
                    uint64_t key = ((uint64_t)best << 32) | (0xFFFFFFFFu - best_i);
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, key, o);
                        key = other > key ? other : key;
                    }
                    const uint32_t donor = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
                    if (lane == 0) {
                        freq[donor] -= 1;
                        freq[t] = 1;
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        f = freq[s];
    }
    freq[s] = f;
    __syncthreads();
    // Cumulative starts (ans.hpp:139-146): inclusive warp scans + warp offsets.
    uint32_t incl = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) redf[warp] = incl;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += redf[w];
    cum[s] = off + incl - f;
    if (s == 255) cum[256] = off + incl;
    __syncthreads();
    if (cum[256] != kProbScale) {  // ans.hpp:99-101 FormatError
        if (s == 0) atomicOr(info + 2, kErrTable);
        return;
    }
    if (freqs_out) freqs_out[s] = (uint16_t)f;
    if (enc) {
        EncSym e;
        e.freq = f;
        e.cum = cum[s];
        // Exact division for the encoder's x < 2^31 (Granlund-Montgomery):
        // l = ceil(log2 f), m = ceil(2^(31+l) / f) < 2^32, x / f = (x m) >> (31+l).
        uint32_t l = 0;
        while ((1u << l) < (uint32_t)f) ++l;
        e.rcp = f ? (uint32_t)(((1ull << (31 + l)) + (uint64_t)f - 1) / (uint64_t)f) : 0u;
        e.pad = 31 + l;
        enc[s] = e;
    }
    if (s == 255 && f > 0) atomicOr(info, kFlagHas255);
    if (f == kProbScale) {
        atomicOr(info, kFlagSingleSymbol);
        info[1] = (uint32_t)s;
    }
    // Decode LUT: thread s fills slots s*16 .. s*16+15 (binary search in cum).
    if (lut) {
        for (int k = 0; k < 16; ++k) {
            const uint32_t slot = (uint32_t)s * 16 + k;
            // The largest symbol with cum <= slot always has freq > 0
            // (zero-frequency symbols share the cum of their successor).
            int lo = 0, hi = 255;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (cum[mid] <= slot) lo = mid; else hi = mid - 1;
            }
            const int sym = lo;
            const uint32_t fs = freq[sym];
            lut[slot] = lut_entry((uint32_t)sym, slot - cum[sym], fs == kProbScale ? 0u : fs);
        }
    }
}

__global__ void __launch_bounds__(256) build_table_kernel(const unsigned long long* __restrict__ counts,
                                                          const uint16_t* __restrict__ given_freqs,
                                                          uint16_t* __restrict__ freqs_out,
                                                          EncSym* __restrict__ enc,
                                                          uint32_t* __restrict__ lut,
                                                          uint32_t* __restrict__ info) {
    build_table_body(counts, given_freqs, freqs_out, enc, lut, info);
}

// Batched compress: one CTA per tensor (blockIdx.x).
__global__ void __launch_bounds__(256) build_tables_kernel(const TableTask* __restrict__ tasks) {
    const TableTask t = tasks[blockIdx.x];
    build_table_body(t.counts, nullptr, t.freqs, t.enc, t.lut, t.info);
}

}  // namespace nzgpu
