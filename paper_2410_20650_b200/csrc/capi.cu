// capi.cu -- the C ABI (include/nzgpu.h): blob management, compress /
// decompress pipelines, grouped decode plans and the host tier that the
// drop-in C++ API (include/neuzip/*.hpp) calls.
//
// No CPU fallback: every data-path function runs the CUDA kernels and
// returns NZGPU_NO_DEVICE when no GPU is present.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <memory>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/nzgpu.h"
#include "nzgpu_internal.cuh"

namespace nzgpu {
// kernels (split_table.cu, encode.cu, lossy.cu, decode.cu)
__global__ void split_hist_kernel(const uint16_t*, uint64_t, uint8_t*, uint8_t*, unsigned long long*);
cudaError_t launch_split_hist(const uint16_t*, uint64_t, uint8_t*, uint8_t*, unsigned long long*, cudaStream_t);
__global__ void byte_hist_kernel(const uint8_t*, uint64_t, unsigned long long*);
__global__ void build_table_kernel(const unsigned long long*, const uint16_t*, uint16_t*, EncSym*, uint32_t*,
                                   uint32_t*);
size_t lossy_task_bytes();
void lossy_task_fill(void* at, const uint16_t* v, uint64_t nfull, uint8_t* scales, uint8_t* exps, uint8_t* packed,
                     unsigned long long* counts, uint32_t* err);
bool lossy_batchable(uint64_t n, int k, uint32_t block);
cudaError_t launch_lossy_prep_batch(const void* tasks, int count, int k, uint32_t block, uint64_t max_nfull,
                                    cudaStream_t s);
size_t split_task_bytes();
void split_task_fill(void* at, const uint16_t* v, uint64_t n, uint8_t* exps, uint8_t* signmant,
                     unsigned long long* counts, uint32_t* err);
cudaError_t launch_split_hist_batch(const void* tasks, int count, uint64_t max_n, cudaStream_t s);
cudaError_t launch_stream_copy_batch(const void* jobs, int njobs, uint64_t total_chunks, uint64_t slot_bytes,
                                     cudaStream_t s);
size_t stream_copy_job_bytes();
void stream_copy_job_fill(void* at, const uint8_t* scratch, const uint4* chunk_info, uint8_t* stream,
                          const uint8_t* hdr, uint64_t chunk0);
cudaError_t launch_index_finalize(const EncTask* tasks, int ntasks, const EncTask& one, uint64_t total_units,
                                  cudaStream_t s);
cudaError_t launch_encode(bool queue, bool check, unsigned ctas, unsigned threads, const EncTask* tasks, int ntasks,
                          const EncTask& one, cudaStream_t s);
__global__ void stream_scan_kernel(const EncTask*, const __grid_constant__ EncTask);
__global__ void build_tables_kernel(const TableTask*);
__global__ void gather_u32_kernel(const uint32_t* const*, uint32_t*, int);
__global__ void stream_copy_kernel(const uint8_t*, uint64_t, const uint4*, uint8_t*);
__global__ void lossy_normalize_kernel(const uint16_t*, uint64_t, int, uint32_t, uint8_t*, uint8_t*, uint8_t*,
                                       uint32_t*);
cudaError_t launch_lossy_prep(const uint16_t*, uint64_t, int, uint32_t, uint8_t*, uint8_t*, uint8_t*, uint8_t*,
                              uint64_t, unsigned long long*, uint32_t*, cudaStream_t);
__global__ void pack_items_kernel(const uint8_t*, uint64_t, int, uint8_t*, uint64_t);
__global__ void lossy_roundtrip_kernel(const uint16_t*, const uint8_t*, uint64_t, int, uint16_t*);
__global__ void unpack_items_kernel(const uint8_t*, uint64_t, int, uint8_t*);
__global__ void seq_decode_kernel(const uint8_t*, const uint4*, const uint64_t*, uint32_t, uint64_t, const uint32_t*,
                                  uint32_t, uint32_t, uint32_t*, uint32_t*, uint16_t*, uint8_t*, uint32_t*);
__global__ void merge_plane_kernel(const uint8_t*, const uint8_t*, const uint8_t*, uint64_t, int, uint32_t,
                                   uint16_t*);
cudaError_t launch_decode(int log2k, int precision, const DecodeDesc* descs, int ndesc, const uint64_t* prefix,
                          const DecodeDesc& one, uint64_t tiles, uint32_t win_cap, cudaStream_t s);
cudaError_t launch_window_max(int log2k, const DecodeDesc& d, uint32_t* out, cudaStream_t s);
uint32_t decode_smem_for(int log2k, uint32_t win_cap);
uint64_t decode_tiles_for(uint64_t nsub);
uint64_t decode_tile_subs();
cudaError_t launch_decode_persist(int log2k, int precision, const DecodeDesc* descs, int ndesc,
                                  const uint32_t* cta_prefix, const DecodeDesc& one, uint32_t ctas, uint32_t upc,
                                  uint32_t win_cap, cudaStream_t s);
uint32_t persist_resident_ctas(int log2k, uint32_t win_cap);
bool persist_fits(int log2k, uint32_t win_cap);
cudaError_t launch_unit_window_max(int log2k, const DecodeDesc& d, uint32_t* out, cudaStream_t s);
cudaError_t launch_windows_batch(int log2k, const DecodeDesc* descs, int count, uint32_t tile_subs, uint64_t max_units,
                                 uint32_t* out, cudaStream_t s);
// entropy.cu
__global__ void component_hist_kernel(const uint16_t*, uint64_t, unsigned long long*);
// crc32.cu
cudaError_t crc_raw_device(const uint8_t* d, uint64_t len, cudaStream_t s, uint32_t* raw);
uint32_t crc_combine_raw(uint32_t raw_a, uint32_t raw_b, uint64_t len_b);
uint32_t crc_finalize(uint32_t raw, uint64_t len);
}  // namespace nzgpu

namespace {
// Decode schedule: the persistent warp-pipelined kernel (default) or the
// one-tile-per-CTA kernel (NZGPU_KERNEL=tiles, or nzgpu_set_decode_kernel).
#ifndef NZ_ENC_QUEUE_MIN_CTAS
#define NZ_ENC_QUEUE_MIN_CTAS 600
#endif
constexpr uint32_t kEncQueueMinCtas = NZ_ENC_QUEUE_MIN_CTAS;
#ifndef NZ_K1_BATCH
#define NZ_K1_BATCH 1
#endif
#ifndef NZ_ENC_CHECK_OWN
#define NZ_ENC_CHECK_OWN false  // compress: the frequency check is redundant with the histogram's table
#endif

int g_kernel = -1;  // -1: from the environment
bool use_persist() {
    if (g_kernel < 0) {
        const char* e = std::getenv("NZGPU_KERNEL");
        g_kernel = (e && std::string(e) == "tiles") ? 1 : 0;
    }
    return g_kernel == 0;
}
}  // namespace

using namespace nzgpu;

namespace {

constexpr uint32_t kIndexMagic = 0x58495A4Eu;  // "NZIX"
constexpr uint32_t kIndexVersion = 3;  // 3: compact records (state, byte count, unit position)
constexpr uint32_t kFlagIrregular = 2u;

struct IndexHeader {
    uint32_t magic;
    uint32_t version;
    uint32_t chunk_syms;
    uint32_t interval;
    uint64_t n;
    uint64_t nchunks;
    uint64_t nsub;
    uint64_t stream_len;
    // Largest payload window of a 32-sub-range warp unit (the persistent
    // decoder's shared-memory window), so host-tier decodes need not scan the
    // index for it.  Only a sizing hint: a unit that does not fit is a decode
    // error (decode_persist.cu, stage()), never an out-of-window read.
    uint32_t max_window_unit;
    uint32_t reserved;
};
static_assert(sizeof(IndexHeader) == 56, "index header layout");

thread_local char g_msg[512] = "";

int fail_cuda(cudaError_t e, const char* what) {
    std::snprintf(g_msg, sizeof(g_msg), "%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? NZGPU_OUT_OF_MEMORY
           : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? NZGPU_NO_DEVICE
                                                                            : NZGPU_CUDA_ERROR;
}

#define CK(call)                                           \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return fail_cuda(e_, #call); \
    } while (0)

int status_from_bits(uint32_t bits) {
    if (!bits) return NZGPU_OK;
    if (bits & kErrNonFinite) return NZGPU_NONFINITE;
    if (bits & kErrZeroFreq) return NZGPU_INVALID_ARGUMENT;
    if (bits & kErrTable) return NZGPU_FORMAT_TABLE;
    if (bits & kErrTruncated) return NZGPU_FORMAT_TRUNCATED;
    if (bits & kErrDesync) return NZGPU_FORMAT_DESYNC;
    return NZGPU_FORMAT_LENGTH;
}

int log2_of(uint32_t k) {
    switch (k) {
        case 64: return 6;
        case 128: return 7;  // a sub-range's byte count must fit the index's count byte (K <= 128)
        default: return -1;
    }
}

bool valid_precision(int p) { return p == 7 || p == 0 || p == 1 || p == 3; }

uint64_t mant_bytes(uint64_t n, int p) { return (n * (uint64_t)(p + 1) + 7) / 8; }

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Side index region (nzgpu_internal.cuh): st u32[nsub] | base u32[units] |
// off u16[nsub] -- the device layout and the exported bytes after the header.
uint64_t index_units(uint64_t nsub) { return ceil_div(nsub, 32); }
uint64_t index_region_bytes(uint64_t nsub) { return 4 * nsub + 4 * index_units(nsub) + 2 * nsub; }

int device_ready() {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        std::snprintf(g_msg, sizeof(g_msg), "no CUDA device: %s",
                      e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e));
        cudaGetLastError();
        return NZGPU_NO_DEVICE;
    }
    return NZGPU_OK;
}

// One device allocation carved into 256-byte aligned sections.
struct Carve {
    uint64_t size = 0;
    uint64_t take(uint64_t bytes) {
        const uint64_t off = size;
        size = align_up(size + bytes, 256);
        return off;
    }
};

unsigned grid_for(uint64_t work, unsigned threads, unsigned cap = 148 * 16) {
    const uint64_t g = (work + threads - 1) / threads;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, cap));
}

// Blob memory comes from a library-owned stream-ordered pool per device
// (cudaMallocFromPoolAsync, release threshold = never): a compress or import
// reuses the memory of freed blobs instead of paying cudaMalloc, which costs
// 0.1-2 ms per call and dominated single-tensor compress.  Freeing keeps
// cudaFree's semantics -- it waits for the device first -- so a blob freed
// right after launching a decode on another stream is still safe.
cudaError_t pool_of(cudaMemPool_t* out) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if ((e = cudaMemPoolCreate(&pools[dev], &props)) != cudaSuccess) return e;
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = pools[dev];
    return cudaSuccess;
}

// Allocation usable by any stream once `s` has been synchronised (every
// caller synchronises before handing the blob out).  Only allocations below
// 256 MiB come from the pool: growing a pool maps physical memory in small
// granules, which made a 10 GB model-batch arena cost ~0.7 s against
// cudaMalloc's ~10 ms, while per-call cudaMalloc latency only matters for
// the small blobs of per-tensor compresses.
#ifndef NZ_POOL
#define NZ_POOL 1
#endif
constexpr uint64_t kPoolMaxBytes = 256ull << 20;
std::mutex g_pool_ptrs_mu;
std::vector<void*> g_pool_ptrs;  // live pool allocations (small: one per pooled blob section)

cudaError_t dev_alloc(void** p, uint64_t bytes, cudaStream_t s) {
    bytes = std::max<uint64_t>(bytes, 256);
    if (!NZ_POOL || bytes >= kPoolMaxBytes) return cudaMalloc(p, bytes);
    cudaMemPool_t pool;
    cudaError_t e = pool_of(&pool);
    if (e != cudaSuccess) return e;
    if ((e = cudaMallocFromPoolAsync(p, bytes, pool, s)) != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_pool_ptrs_mu);
    g_pool_ptrs.push_back(*p);
    return cudaSuccess;
}

void dev_free(void* p) {
    if (!p) return;
    bool pooled = false;
    {
        std::lock_guard<std::mutex> lock(g_pool_ptrs_mu);
        auto it = std::find(g_pool_ptrs.begin(), g_pool_ptrs.end(), p);
        if (it != g_pool_ptrs.end()) {
            *it = g_pool_ptrs.back();
            g_pool_ptrs.pop_back();
            pooled = true;
        }
    }
    if (!pooled) {
        cudaFree(p);  // synchronises the device, as before
        return;
    }
    cudaDeviceSynchronize();
    cudaFreeAsync(p, nullptr);
}

}  // namespace

// ------------------------------------------------------------------ blob --
struct nzgpu_blob_s {
    uint64_t n = 0;
    int precision = 7;
    uint32_t block = 0;
    uint32_t chunk_syms = kDefaultChunk;
    uint32_t interval = 128;
    int log2k = 7;
    uint64_t nchunks = 0;
    uint64_t nsub = 0;
    uint32_t flags = 0;
    uint32_t single_symbol = 0;
    uint32_t max_window = 0;       // per 256-sub-range tile (decode_tiles_kernel)
    uint32_t max_window_unit = 0;  // per 32-sub-range warp unit (decode_persist_kernel)
    // main allocation
    void* base = nullptr;
    uint16_t* freqs = nullptr;
    uint32_t* lut = nullptr;
    uint8_t* mant = nullptr;
    uint64_t mant_len = 0;
    uint8_t* scales = nullptr;
    uint64_t scales_len = 0;
    uint4* chunk_info = nullptr;
    uint64_t* chunk_sym0 = nullptr;  // irregular framing only
    bool sym0_valid = false;          // chunk_sym0 filled (imported non-uniform framing)
    uint8_t* index = nullptr;  // side index region (index_region_bytes(nsub))
    uint32_t* err = nullptr;
    uint32_t* scratch_u32 = nullptr;  // 4 words: table info[3] + window
    // stream allocation
    uint8_t* stream = nullptr;
    uint64_t stream_len = 0;

    bool owns = true;  // false: a descriptor over buffers owned by a host-pipeline slot
    // Batched compress: base / stream sections live in allocations shared by
    // the blobs of one batch, freed with the last of them.
    std::shared_ptr<void> base_arena, stream_arena;

    ~nzgpu_blob_s() {
        if (!owns) return;
        if (base && !base_arena) dev_free(base);
        if (stream && !stream_arena) dev_free(stream);
    }

    DecodeDesc desc(uint16_t* out) const {
        DecodeDesc d{};
        d.stream = stream;
        d.mant = mant;
        d.scales = scales;
        d.ck_state = ck_state();
        d.ck_base = ck_base();
        d.ck_off = ck_off();
        d.chunk_info = chunk_info;
        d.lut = lut;
        d.out = out;
        d.err = err;
        d.n = n;
        d.chunk_syms = chunk_syms;
        d.flags = flags & (kFlagSingleSymbol | kFlagSlowLossy);
        d.single_symbol = single_symbol;
        d.precision = precision;
        d.block_size = block ? block : 1;
        const uint32_t spc = interval ? chunk_syms / interval : 0;
        d.log2_spc = (spc && !(spc & (spc - 1))) ? (uint32_t)__builtin_ctz(spc) : 0xFFFFFFFFu;
        d.log2_block = !(d.block_size & (d.block_size - 1)) ? (uint32_t)__builtin_ctz(d.block_size) : 0xFFFFFFFFu;
        return d;
    }
    uint64_t tiles() const { return decode_tiles_for(nsub); }
    uint32_t* ck_state() const { return reinterpret_cast<uint32_t*>(index); }
    uint32_t* ck_base() const { return ck_state() + nsub; }
    uint16_t* ck_off() const { return reinterpret_cast<uint16_t*>(ck_base() + index_units(nsub)); }
};

namespace {

// Main section block of a blob (everything but the stream): its size, and
// its carving from `at` (a fresh cudaMalloc when null).
uint64_t blob_base_bytes(const nzgpu_blob_s* b, bool irregular) {
    Carve cv;
    cv.take(512);
    cv.take(16384);
    cv.take(std::max<uint64_t>(b->mant_len, 1) + 16);
    cv.take(std::max<uint64_t>(b->scales_len, 1));
    cv.take(std::max<uint64_t>(b->nchunks, 1) * sizeof(uint4));
    cv.take(irregular ? std::max<uint64_t>(b->nchunks, 1) * 8 : 8);
    cv.take(index_region_bytes(b->nsub) + 16);
    cv.take(64);
    return cv.size;
}

int blob_alloc(nzgpu_blob_s* b, bool irregular, uint8_t* at = nullptr, cudaStream_t s = nullptr) {
    Carve cv;
    const uint64_t o_freqs = cv.take(512);
    const uint64_t o_lut = cv.take(16384);
    const uint64_t o_mant = cv.take(std::max<uint64_t>(b->mant_len, 1) + 16);
    const uint64_t o_scales = cv.take(std::max<uint64_t>(b->scales_len, 1));
    const uint64_t o_info = cv.take(std::max<uint64_t>(b->nchunks, 1) * sizeof(uint4));
    const uint64_t o_sym0 = cv.take(irregular ? std::max<uint64_t>(b->nchunks, 1) * 8 : 8);
    const uint64_t o_index = cv.take(index_region_bytes(b->nsub) + 16);
    const uint64_t o_err = cv.take(64);
    if (at) {
        b->base = at;
    } else {
        CK(dev_alloc(&b->base, cv.size, s));
    }
    uint8_t* p = static_cast<uint8_t*>(b->base);
    b->freqs = reinterpret_cast<uint16_t*>(p + o_freqs);
    b->lut = reinterpret_cast<uint32_t*>(p + o_lut);
    b->mant = p + o_mant;
    b->scales = p + o_scales;
    b->chunk_info = reinterpret_cast<uint4*>(p + o_info);
    b->chunk_sym0 = reinterpret_cast<uint64_t*>(p + o_sym0);
    b->index = p + o_index;
    b->err = reinterpret_cast<uint32_t*>(p + o_err);
    b->scratch_u32 = b->err + 4;
    return NZGPU_OK;
}

// One device allocation shared by the blobs of a batch (freed with the last).
int arena_alloc(uint64_t bytes, std::shared_ptr<void>& out, cudaStream_t s) {
    void* p = nullptr;
    CK(dev_alloc(&p, bytes, s));
    out = std::shared_ptr<void>(p, [](void* q) { dev_free(q); });
    return NZGPU_OK;
}

int sync_status(cudaStream_t s, uint32_t* d_err, bool clear) {
    CK(cudaStreamSynchronize(s));
    uint32_t bits = 0;
    CK(cudaMemcpy(&bits, d_err, 4, cudaMemcpyDeviceToHost));
    if (clear && bits) CK(cudaMemset(d_err, 0, 4));
    return status_from_bits(bits);
}

// Host walk of the serialized framing (deserialize_stream, ans.hpp:318-347).
int walk_stream(const uint8_t* s, uint64_t len, std::vector<uint4>& info, uint64_t& total) {
    if (len < 4) return NZGPU_FORMAT_TRUNCATED;
    auto le32 = [&](uint64_t p) {
        return (uint32_t)s[p] | ((uint32_t)s[p + 1] << 8) | ((uint32_t)s[p + 2] << 16) | ((uint32_t)s[p + 3] << 24);
    };
    const uint32_t cnt = le32(0);
    uint64_t pos = 4;
    total = 0;
    info.clear();
    info.reserve(std::min<uint64_t>(cnt, len / 8 + 1));
    for (uint32_t c = 0; c < cnt; ++c) {
        if (len - pos < 8) return NZGPU_FORMAT_TRUNCATED;  // "ans stream: truncated framing"
        const uint32_t nsym = le32(pos), plen = le32(pos + 4);
        pos += 8;
        if (len - pos < plen) return NZGPU_FORMAT_TRUNCATED;
        info.push_back(make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), plen, nsym));
        pos += plen;
        total += nsym;
    }
    if (pos != len) return NZGPU_FORMAT_LENGTH;  // "ans stream: trailing bytes"
    return NZGPU_OK;
}

// kFlagWideScale when an imported lossy blob has a scale byte >= 128.
uint32_t wide_scale_flag(const nzgpu_host_tensor* t) {
    if (t->precision == 7 || !t->scales) return 0u;
    for (uint64_t i = 0; i < t->scales_len; ++i)
        if (t->scales[i] & 0x80u) return kFlagWideScale;
    return 0u;
}

// Exponent-table upload + validation (deserialize_table, ans.hpp:120-130)
// + packed decode LUT; reads back flags.
int install_table(nzgpu_blob_s* b, const uint16_t* h_freqs, cudaStream_t s) {
    CK(cudaMemcpyAsync(b->freqs, h_freqs, 512, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(b->scratch_u32, 0, 16, s));
    build_table_kernel<<<1, 256, 0, s>>>(nullptr, b->freqs, nullptr, nullptr, b->lut, b->scratch_u32);
    CK(cudaGetLastError());
    uint32_t info[3];
    CK(cudaMemcpyAsync(info, b->scratch_u32, 12, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (info[2]) return status_from_bits(info[2]);
    b->flags |= info[0] & (kFlagSingleSymbol | kFlagHas255);
    b->single_symbol = info[1];
    return NZGPU_OK;
}

// Largest payload window per decode tile / warp unit of each blob (sizes the
// decoders' shared-memory windows): the window kernels of every blob, then one
// readback.
int compute_windows(nzgpu_blob_s* const* bs, int count, cudaStream_t s, uint8_t* scratch_ptrs = nullptr,
                    uint32_t* scratch_res = nullptr, uint8_t* scratch_descs = nullptr) {
    // A compress batch (device scratch for a descriptor table given): one
    // launch for every window maximum of one stride, where the per-tensor
    // form costs a memset and two launches per tensor
    if (scratch_descs && scratch_res && count > 1) {
        std::vector<DecodeDesc> ds;
        std::vector<int> idx;
        int log2k = -1;
        bool same = true;
        uint64_t max_units = 0;
        for (int i = 0; i < count; ++i) {
            nzgpu_blob_s* b = bs[i];
            b->max_window = b->max_window_unit = 0;
            if ((b->flags & kFlagIrregular) || b->nsub == 0 || (b->flags & kFlagSingleSymbol)) continue;
            if (log2k >= 0 && b->log2k != log2k) same = false;
            log2k = b->log2k;
            ds.push_back(b->desc(nullptr));
            idx.push_back(i);
            max_units = std::max<uint64_t>(max_units, ceil_div(b->nsub, 32));
        }
        if (ds.empty()) return NZGPU_OK;
        if (same) {
            auto* d_descs = reinterpret_cast<DecodeDesc*>(scratch_descs);
            CK(cudaMemcpyAsync(d_descs, ds.data(), ds.size() * sizeof(DecodeDesc), cudaMemcpyHostToDevice, s));
            CK(cudaMemsetAsync(scratch_res, 0, ds.size() * 8, s));
            CK(launch_windows_batch(log2k, d_descs, (int)ds.size(), (uint32_t)decode_tile_subs(), max_units,
                                    scratch_res, s));
            std::vector<uint32_t> w(ds.size() * 2);
            CK(cudaMemcpyAsync(w.data(), scratch_res, w.size() * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));  // w is a host stack vector
            for (size_t j = 0; j < idx.size(); ++j) {
                bs[idx[j]]->max_window_unit = w[2 * j];
                bs[idx[j]]->max_window = w[2 * j + 1];
            }
            return NZGPU_OK;
        }
    }
    std::vector<const uint32_t*> ptrs;
    std::vector<int> who;
    for (int i = 0; i < count; ++i) {
        nzgpu_blob_s* b = bs[i];
        b->max_window = b->max_window_unit = 0;
        if ((b->flags & kFlagIrregular) || b->nsub == 0 || (b->flags & kFlagSingleSymbol)) continue;
        CK(cudaMemsetAsync(b->scratch_u32 + 2, 0, 8, s));
        CK(launch_window_max(b->log2k, b->desc(nullptr), b->scratch_u32 + 3, s));
        CK(launch_unit_window_max(b->log2k, b->desc(nullptr), b->scratch_u32 + 2, s));
        ptrs.push_back(b->scratch_u32 + 2);
        ptrs.push_back(b->scratch_u32 + 3);
        who.push_back(i);
    }
    if (who.empty()) return NZGPU_OK;
    static const bool trace = std::getenv("NZGPU_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[nzgpu]   compute_windows(%d) %-10s %9.1f us\n", count, what,
                     std::chrono::duration<double, std::micro>(now - t0).count());
        t0 = now;
    };
    mark("kernels");
    std::vector<uint32_t> w(ptrs.size());
    if (who.size() == 1) {
        CK(cudaMemcpyAsync(w.data(), ptrs[0], 8, cudaMemcpyDeviceToHost, s));
    } else {
        // device scratch: the caller's (a compress batch's readback arrays,
        // >= 2 pointers and 2 words per blob) or a stream-ordered allocation
        uint8_t* tmp = nullptr;
        const uint64_t pb = align_up(ptrs.size() * sizeof(void*), 256);
        const uint32_t* const* d_ptrs;
        uint32_t* d_res;
        if (scratch_ptrs && scratch_res) {
            d_ptrs = reinterpret_cast<const uint32_t* const*>(scratch_ptrs);
            d_res = scratch_res;
        } else {
            CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), pb + ptrs.size() * 4, s));
            d_ptrs = reinterpret_cast<const uint32_t* const*>(tmp);
            d_res = reinterpret_cast<uint32_t*>(tmp + pb);
        }
        mark("scratch");
        CK(cudaMemcpyAsync(const_cast<const uint32_t**>(d_ptrs), ptrs.data(), ptrs.size() * sizeof(void*),
                           cudaMemcpyHostToDevice, s));
        gather_u32_kernel<<<grid_for(ptrs.size(), 256), 256, 0, s>>>(d_ptrs, d_res, (int)ptrs.size());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(w.data(), d_res, w.size() * 4, cudaMemcpyDeviceToHost, s));
        if (tmp) CK(cudaFreeAsync(tmp, s));
    }
    CK(cudaStreamSynchronize(s));
    for (size_t j = 0; j < who.size(); ++j) {
        bs[who[j]]->max_window_unit = w[2 * j];
        bs[who[j]]->max_window = w[2 * j + 1];
    }
    return NZGPU_OK;
}

int compute_window(nzgpu_blob_s* b, cudaStream_t s) { return compute_windows(&b, 1, s); }

// Persistent-kernel geometry: 32-sub-range units, `upc` units per CTA so
// that the grid is about one resident wave.
struct PersistGeom {
    uint32_t ctas = 0, upc = 1;
};
PersistGeom persist_geom(uint64_t units, int log2k, uint32_t win_cap) {
    PersistGeom g;
    if (!units) return g;
    const uint64_t resident = std::max<uint32_t>(1, persist_resident_ctas(log2k, win_cap));
    g.upc = (uint32_t)std::max<uint64_t>(1, ceil_div(units, resident));
    g.ctas = (uint32_t)ceil_div(units, g.upc);
    return g;
}

int decode_blob(nzgpu_blob_s* b, uint16_t* d_out, cudaStream_t s) {
    if (b->n == 0) return NZGPU_OK;
    if (b->flags & kFlagIrregular) {
        // Sequential decode of every chunk, then a separate merge.
        uint8_t* exps = nullptr;
        CK(cudaMallocAsync(&exps, b->n, s));
        seq_decode_kernel<<<grid_for(b->nchunks, 128, 1u << 30), 128, 0, s>>>(
            b->stream, b->chunk_info, b->sym0_valid ? b->chunk_sym0 : nullptr, b->chunk_syms, b->nchunks, b->lut,
            b->flags & kFlagSingleSymbol, b->log2k,
            nullptr, nullptr, nullptr, exps, b->err);
        merge_plane_kernel<<<grid_for(b->n, 256), 256, 0, s>>>(exps, b->mant, b->scales, b->n, b->precision,
                                                                b->block ? b->block : 1, d_out);
        CK(cudaGetLastError());
        CK(cudaFreeAsync(exps, s));
        return NZGPU_OK;
    }
    if (use_persist() && persist_fits(b->log2k, b->max_window_unit)) {
        const PersistGeom g = persist_geom(ceil_div(b->nsub, 32), b->log2k, b->max_window_unit);
        CK(launch_decode_persist(b->log2k, b->precision, nullptr, 0, nullptr, b->desc(d_out), g.ctas, g.upc,
                                 b->max_window_unit, s));
    } else {
        CK(launch_decode(b->log2k, b->precision, nullptr, 0, nullptr, b->desc(d_out), b->tiles(), b->max_window, s));
    }
    return NZGPU_OK;
}

// Decode elements [a, a + len) of a uniform-framing blob, a and len whole
// chunks and warp units (and lossy blocks): the same kernels over a
// descriptor whose index, chunk table, planes and output start at a.
int decode_range(const nzgpu_blob_s* b, uint16_t* d_out, uint64_t a, uint64_t len, cudaStream_t s) {
    if (len == 0) return NZGPU_OK;
    DecodeDesc d = b->desc(d_out + a);
    const uint64_t sub0 = a >> b->log2k, nsub = ceil_div(len, b->interval);
    d.n = len;
    d.ck_state += sub0;
    d.ck_off += sub0;
    d.ck_base += sub0 / 32;
    d.chunk_info += a / b->chunk_syms;
    if (b->precision == 7) {
        d.mant += a;
    } else {
        d.mant += a * (uint64_t)(b->precision + 1) / 8;
        d.scales += a / b->block;
    }
    if (use_persist() && persist_fits(b->log2k, b->max_window_unit)) {
        const PersistGeom g = persist_geom(ceil_div(nsub, 32), b->log2k, b->max_window_unit);
        CK(launch_decode_persist(b->log2k, b->precision, nullptr, 0, nullptr, d, g.ctas, g.upc, b->max_window_unit, s));
    } else {
        CK(launch_decode(b->log2k, b->precision, nullptr, 0, nullptr, d, decode_tiles_for(nsub), b->max_window, s));
    }
    return NZGPU_OK;
}

extern "C" int h2d_staged(void* dst, const void* src, uint64_t bytes, cudaStream_t s);  // host tier, below

// One host section to the device: large ones through the pinned ring and the
// host workers (10-16 GB/s from pageable memory otherwise), small ones direct.
int h2d_section(void* dst, const void* src, uint64_t bytes, cudaStream_t s) {
    if (!bytes) return NZGPU_OK;
    if (bytes < (4ull << 20)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return NZGPU_OK;
    }
    return h2d_staged(dst, src, bytes, s);
}

// Fill a blob from host sections (reference formats).
int import_into(nzgpu_blob_s* b, const nzgpu_host_tensor* t, uint32_t interval, cudaStream_t s) {
    if (!t || !valid_precision(t->precision)) return NZGPU_INVALID_ARGUMENT;
    if (interval != 0 && log2_of(interval) < 0) return NZGPU_INVALID_ARGUMENT;
    if (!t->freqs || (!t->stream && t->stream_len)) return NZGPU_INVALID_ARGUMENT;
    std::vector<uint4> info;
    uint64_t total = 0;
    int rc = walk_stream(t->stream, t->stream_len, info, total);
    if (rc) return rc;
    {  // table sum check first (deserialize_table precedes decode)
        uint32_t sum = 0;
        for (int i = 0; i < 256; ++i) sum += t->freqs[i];
        if (sum != kProbScale) return NZGPU_FORMAT_TABLE;
    }
    if (total != t->n) return NZGPU_FORMAT_LENGTH;  // tensorstore.hpp:115-117, :218-220
    if (t->mantissa_len != mant_bytes(t->n, t->precision) || (t->n && !t->mantissas)) {
        // lossless: FormatError (tensorstore.hpp:115-117); lossy: unpack's
        // invalid_argument (bitfloat.hpp:151-153).
        return t->precision == 7 ? NZGPU_FORMAT_LENGTH : NZGPU_INVALID_ARGUMENT;
    }
    if (t->precision != 7) {
        if (t->block_size == 0) return NZGPU_INVALID_ARGUMENT;
        if (t->scales_len != ceil_div(t->n, t->block_size) || (t->scales_len && !t->scales))
            return NZGPU_FORMAT_LENGTH;  // tensorstore.hpp:223-227
    }
    if (interval == 0) {  // auto: the default stride if it divides the chunk size, else 64
        const uint32_t s0 = info.empty() ? kDefaultChunk : info[0].w;
        interval = s0 % NZGPU_DEFAULT_INTERVAL == 0 ? NZGPU_DEFAULT_INTERVAL : 64;
    }
    if (ceil_div(t->n, interval) >= 0xFFFFFFFFull) return NZGPU_INVALID_ARGUMENT;  // 32-bit sub-range ids
    b->n = t->n;
    b->precision = t->precision;
    b->block = t->precision == 7 ? 0 : t->block_size;
    b->interval = interval;
    b->log2k = log2_of(interval);
    b->nchunks = info.size();
    b->nsub = ceil_div(t->n, interval);
    b->mant_len = t->mantissa_len;
    b->scales_len = t->precision == 7 ? 0 : t->scales_len;
    b->stream_len = t->stream_len;
    // Uniform framing (every chunk but the last holds S symbols, S % K == 0)
    // enables the tiled decoder; anything else decodes sequentially.
    bool uniform = !info.empty();
    const uint32_t S = info.empty() ? kDefaultChunk : info[0].w;
    if (uniform && (S == 0 || S % interval)) uniform = false;
    for (size_t c = 0; uniform && c < info.size(); ++c) {
        if (c + 1 < info.size() ? info[c].w != S : (info[c].w == 0 || info[c].w > S)) uniform = false;
    }
    b->chunk_syms = S;
    b->flags = (uniform || t->n == 0 ? 0u : kFlagIrregular) | wide_scale_flag(t);
    rc = blob_alloc(b, !uniform, nullptr, s);
    if (rc) return rc;
    CK(dev_alloc(reinterpret_cast<void**>(&b->stream), align_up(std::max<uint64_t>(t->stream_len, 1), 16) + 32, s));
    CK(cudaMemsetAsync(b->err, 0, 64, s));
    if (int e = h2d_section(b->stream, t->stream, t->stream_len, s)) return e;
    if (int e = h2d_section(b->mant, t->mantissas, t->mantissa_len, s)) return e;
    if (b->scales_len) CK(cudaMemcpyAsync(b->scales, t->scales, b->scales_len, cudaMemcpyHostToDevice, s));
    if (!info.empty())
        CK(cudaMemcpyAsync(b->chunk_info, info.data(), info.size() * sizeof(uint4), cudaMemcpyHostToDevice, s));
    if (!uniform && !info.empty()) {
        std::vector<uint64_t> sym0(info.size());
        uint64_t acc = 0;
        for (size_t c = 0; c < info.size(); ++c) {
            sym0[c] = acc;
            acc += info[c].w;
        }
        CK(cudaMemcpyAsync(b->chunk_sym0, sym0.data(), sym0.size() * 8, cudaMemcpyHostToDevice, s));
        b->sym0_valid = true;
        CK(cudaStreamSynchronize(s));  // sym0 is a stack vector
    }
    rc = install_table(b, t->freqs, s);
    if (rc) return rc;
    if (!uniform || t->n == 0) return NZGPU_OK;
    bool have_index = false;
    if (t->index && t->index_len >= sizeof(IndexHeader)) {
        IndexHeader h;
        std::memcpy(&h, t->index, sizeof(h));
        have_index = h.magic == kIndexMagic && h.version == kIndexVersion && h.chunk_syms == S &&
                     h.interval == interval && h.n == t->n && h.nchunks == info.size() && h.nsub == b->nsub &&
                     h.stream_len == t->stream_len && t->index_len == sizeof(h) + index_region_bytes(h.nsub);
        if (have_index)
            if (int e = h2d_section(b->index, static_cast<const uint8_t*>(t->index) + sizeof(h),
                                    index_region_bytes(b->nsub), s))
                return e;
    }
    if (!have_index) {
        // K8: rebuild the checkpoint index by decoding every chunk once on
        // the GPU (full reference validation, ans.hpp:229-256).
        seq_decode_kernel<<<grid_for(b->nchunks, 128, 1u << 30), 128, 0, s>>>(
            b->stream, b->chunk_info, nullptr, S, b->nchunks, b->lut, b->flags & kFlagSingleSymbol, b->log2k,
            b->ck_state(), b->ck_base(), b->ck_off(), nullptr, b->err);
        CK(cudaGetLastError());
        rc = sync_status(s, b->err, true);
        if (rc) return rc;
    }
    return compute_window(b, s);
}

// Workspace layout of a batched compress: per-tensor exponent plane, lossy
// items, worst-case payload slots, histogram, payload lengths, stream length,
// encoder constants and stream header, then the task / readback arrays.
struct BatchLayout {
    struct Tmp {
        uint64_t exps, items, scratch, counts, plen, total, enc, hdr;
    };
    std::vector<Tmp> to;
    uint64_t tasks = 0, tables = 0, ptrs = 0, res = 0, size = 0, slot = 0;
    BatchLayout(const uint64_t* ns, int count, int precision, uint32_t chunk_syms) : to(count) {
        slot = align_up(2ull * chunk_syms + 8, 16);
        Carve cv;
        for (int i = 0; i < count; ++i) {
            const uint64_t n = ns[i], nchunks = ceil_div(n, chunk_syms);
            to[i].exps = cv.take(n + 16);
            to[i].items = cv.take(precision == 7 ? 16 : n + 16);
            to[i].scratch = cv.take(nchunks * slot + 16);
            to[i].counts = cv.take(256 * 8);
            to[i].plen = cv.take(nchunks * 4);
            to[i].total = cv.take(16);
            to[i].enc = cv.take(256 * sizeof(EncSym));
            to[i].hdr = cv.take(16);
        }
        tasks = cv.take(count * sizeof(EncTask));
        tables = cv.take(count * sizeof(TableTask));
        ptrs = cv.take(count * 6 * sizeof(void*));
        res = cv.take(count * 6 * 4);
        size = cv.size;
    }
};

// Compress `count` tensors in one pipeline: per-tensor split / histogram /
// table kernels, ONE K3 launch over the chunks of every tensor (the chunk
// chains are serial and latency-bound, so tensors must share a launch to fill
// the GPU), one K4 scan launch, then a single host synchronisation to learn
// the stream lengths before the streams are allocated and compacted.  The
// blobs of a batch share two allocations (sections, streams): per-blob
// cudaMalloc calls cost more than the kernels.  `ws` (ws_bytes >=
// BatchLayout::size) holds the temporaries; null = stream-ordered allocation.
// On error every blob is left empty (the caller frees them).
int compress_many(nzgpu_blob_s* const* bs, const uint16_t* const* vs, const uint64_t* ns, int count, int precision,
                  uint32_t block, uint32_t chunk_syms, uint32_t interval, cudaStream_t s, void* ws = nullptr,
                  uint64_t ws_bytes = 0) {
    if (count <= 0 || !valid_precision(precision)) return NZGPU_INVALID_ARGUMENT;
    if (precision != 7 && block == 0) return NZGPU_INVALID_ARGUMENT;  // tensorstore.hpp:146-148
    if (chunk_syms == 0) chunk_syms = kDefaultChunk;
    // interval 0 = auto: the default stride if it divides S, else 64; chunk
    // sizes divisible by neither keep the reference format but decode with
    // the sequential kernel (no side index).
    bool irregular = false;
    if (interval == 0) {
        interval = chunk_syms % NZGPU_DEFAULT_INTERVAL == 0 ? NZGPU_DEFAULT_INTERVAL : 64;
        irregular = chunk_syms % interval != 0;
    }
    const int log2k = log2_of(interval);
    if (log2k < 0 || (!irregular && chunk_syms % interval)) return NZGPU_INVALID_ARGUMENT;
    for (int i = 0; i < count; ++i) {
        if (!bs[i] || ns[i] == 0 || !vs[i]) return NZGPU_INVALID_ARGUMENT;  // tensorstore.hpp:47-53
        if (reinterpret_cast<uintptr_t>(vs[i]) & 15) return NZGPU_INVALID_ARGUMENT;
        if (ceil_div(ns[i], interval) >= 0xFFFFFFFFull) return NZGPU_INVALID_ARGUMENT;  // 32-bit sub-range ids
    }
    static const bool trace = std::getenv("NZGPU_TRACE") != nullptr;
    auto tlast = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(s);  // attribute device time to the phase that queued it
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[nzgpu] compress_many(%d) %-10s %9.1f us\n", count, what,
                     std::chrono::duration<double, std::micro>(now - tlast).count());
        tlast = now;
    };
    const BatchLayout L(ns, count, precision, chunk_syms);
    const uint64_t slot = L.slot;
    if (ws && (ws_bytes < L.size || (reinterpret_cast<uintptr_t>(ws) & 255))) return NZGPU_INVALID_ARGUMENT;
    uint8_t* tmp = static_cast<uint8_t*>(ws);
    if (!tmp) CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), L.size, s));
    struct TmpGuard {
        uint8_t* p;
        cudaStream_t s;
        ~TmpGuard() {
            if (p) cudaFreeAsync(p, s);
        }
    } guard{ws ? nullptr : tmp, s};
    mark("tmp alloc");
    // Section block of every blob: one shared allocation for a batch.
    std::vector<uint64_t> boff(count);
    uint64_t btotal = 0;
    for (int i = 0; i < count; ++i) {
        nzgpu_blob_s* b = bs[i];
        const uint64_t n = ns[i];
        b->n = n;
        b->precision = precision;
        b->block = precision == 7 ? 0 : block;
        b->chunk_syms = chunk_syms;
        b->interval = interval;
        b->log2k = log2k;
        b->nchunks = ceil_div(n, chunk_syms);
        b->nsub = ceil_div(n, interval);
        b->mant_len = mant_bytes(n, precision);
        b->scales_len = precision == 7 ? 0 : ceil_div(n, block);
        b->flags = 0;
        boff[i] = btotal;
        btotal += align_up(blob_base_bytes(b, false), 256);
    }
    std::shared_ptr<void> base_arena;
    if (count > 1) {
        if (int rc = arena_alloc(btotal, base_arena, s)) return rc;
    }
    mark("blob alloc");
    std::vector<EncTask> tasks(count);
    std::vector<TableTask> tables(count);
    // lossless batches: K1 (and the zeroing of histograms and error words)
    // for every tensor in one launch; its task table uses the encode task
    // table's space, which is only written after it
    const bool batched_k1 = precision == 7 && count > 1 && NZ_K1_BATCH;
    std::vector<uint8_t> split_tasks(batched_k1 ? count * split_task_bytes() : 0);
    uint64_t max_n = 0;
    // lossy batches whose every tensor is whole fused blocks: K6 likewise
    bool batched_k6 = precision != 7 && count > 1 && NZ_K1_BATCH;
    for (int i = 0; batched_k6 && i < count; ++i) batched_k6 = lossy_batchable(ns[i], precision, block);
    std::vector<uint8_t> lossy_tasks(batched_k6 ? count * lossy_task_bytes() : 0);
    uint32_t ctas = 0;
    uint64_t units = 0;  // warp units of every tensor's side index (index_finalize_kernel)
    for (int i = 0; i < count; ++i) {
        nzgpu_blob_s* b = bs[i];
        const uint64_t n = ns[i];
        if (base_arena) {
            b->base_arena = base_arena;
            blob_alloc(b, false, static_cast<uint8_t*>(base_arena.get()) + boff[i]);
        } else if (int rc = blob_alloc(b, false, nullptr, s)) {
            return rc;
        }
        uint8_t* exps = tmp + L.to[i].exps;
        auto* counts = reinterpret_cast<unsigned long long*>(tmp + L.to[i].counts);
        auto* enc = reinterpret_cast<EncSym*>(tmp + L.to[i].enc);
        if (batched_k1) {  // K1 of the whole batch in one launch after this loop
            split_task_fill(split_tasks.data() + i * split_task_bytes(), vs[i], n, exps, b->mant, counts, b->err);
            max_n = std::max<uint64_t>(max_n, n);
        } else if (batched_k6) {
            lossy_task_fill(lossy_tasks.data() + i * lossy_task_bytes(), vs[i], n / block, b->scales, exps, b->mant,
                            counts, b->err);
            max_n = std::max<uint64_t>(max_n, n / block);
        } else {
            CK(cudaMemsetAsync(counts, 0, 256 * 8, s));
            CK(cudaMemsetAsync(b->err, 0, 64, s));
        }
        if (batched_k1 || batched_k6) {
        } else if (precision == 7) {
            CK(launch_split_hist(vs[i], n, exps, b->mant, counts, s));
        } else {
            uint8_t* items = tmp + L.to[i].items;
            CK(launch_lossy_prep(vs[i], n, precision, block, b->scales, exps, items, b->mant, b->mant_len, counts,
                                 b->err, s));
        }
        tables[i] = TableTask{counts, b->freqs, enc, b->lut, b->scratch_u32};
        if (count == 1) build_table_kernel<<<1, 256, 0, s>>>(counts, nullptr, b->freqs, enc, b->lut, b->scratch_u32);
        EncTask& t = tasks[i];
        t = EncTask{};
        t.exps = exps;
        t.enc = enc;
        t.scratch = tmp + L.to[i].scratch;
        t.plen = reinterpret_cast<uint32_t*>(tmp + L.to[i].plen);
        t.ck_state = irregular ? nullptr : b->ck_state();
        t.ck_base = irregular ? nullptr : b->ck_base();
        t.ck_off = irregular ? nullptr : b->ck_off();
        t.err = b->err;
        t.chunk_info = b->chunk_info;
        t.hdr = tmp + L.to[i].hdr;
        t.total = reinterpret_cast<unsigned long long*>(tmp + L.to[i].total);
        t.n = n;
        t.slot_bytes = slot;
        t.chunk_syms = chunk_syms;
        t.log2k = (uint32_t)log2k;
        t.cta0 = ctas;
        t.unit0 = units;
        if (!irregular) units += index_units(b->nsub);
        const uint64_t c = ceil_div(b->nchunks, NZ_ENC_THREADS);
        if (ctas + c >= (1ull << 31)) return NZGPU_INVALID_ARGUMENT;
        ctas += (uint32_t)c;
    }
    // Byte queue once L1 store sectors rather than the chain latency bound
    // the launch: >= ~4 chains per SM (crossover measured at 416-832 chains).
    const bool queue = ctas >= kEncQueueMinCtas;
    auto* d_tasks = reinterpret_cast<EncTask*>(tmp + L.tasks);
    if (batched_k1) {
        static_assert(sizeof(EncTask) >= 48, "the K1 task table reuses the encode task table's space");
        CK(cudaMemcpyAsync(d_tasks, split_tasks.data(), split_tasks.size(), cudaMemcpyHostToDevice, s));
        CK(launch_split_hist_batch(d_tasks, count, max_n, s));
    } else if (batched_k6) {
        static_assert(sizeof(EncTask) >= 56, "the K6 task table reuses the encode task table's space");
        CK(cudaMemcpyAsync(d_tasks, lossy_tasks.data(), lossy_tasks.size(), cudaMemcpyHostToDevice, s));
        CK(launch_lossy_prep_batch(d_tasks, count, precision, block, max_n, s));
    }
    mark("setup");
    if (count > 1) {
        auto* d_tables = reinterpret_cast<TableTask*>(tmp + L.tables);
        CK(cudaMemcpyAsync(d_tables, tables.data(), count * sizeof(TableTask), cudaMemcpyHostToDevice, s));
        build_tables_kernel<<<count, 256, 0, s>>>(d_tables);  // K2 of every tensor in one launch
        CK(cudaMemcpyAsync(d_tasks, tasks.data(), count * sizeof(EncTask), cudaMemcpyHostToDevice, s));
    }
    // the tables come from the tensors' own histograms: no zero frequency
    CK(launch_encode(queue, NZ_ENC_CHECK_OWN, ctas, NZ_ENC_THREADS, count > 1 ? d_tasks : nullptr, count, tasks[0],
                     s));
    if (!irregular) CK(launch_index_finalize(count > 1 ? d_tasks : nullptr, count, tasks[0], units, s));
    stream_scan_kernel<<<count, 1024, 0, s>>>(count > 1 ? d_tasks : nullptr, tasks[0]);
    CK(cudaGetLastError());
    // One readback for every tensor: table info[3], error bits, stream length.
    std::vector<const uint32_t*> ptrs(count * 6);
    for (int i = 0; i < count; ++i) {
        const uint32_t* tot = reinterpret_cast<const uint32_t*>(tasks[i].total);
        const uint32_t* src[6] = {bs[i]->scratch_u32, bs[i]->scratch_u32 + 1, bs[i]->scratch_u32 + 2,
                                  bs[i]->err, tot, tot + 1};
        for (int k = 0; k < 6; ++k) ptrs[i * 6 + k] = src[k];
    }
    auto* d_ptrs = reinterpret_cast<const uint32_t**>(tmp + L.ptrs);
    auto* d_res = reinterpret_cast<uint32_t*>(tmp + L.res);
    CK(cudaMemcpyAsync(d_ptrs, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice, s));
    gather_u32_kernel<<<grid_for(count * 6, 256), 256, 0, s>>>(d_ptrs, d_res, count * 6);
    CK(cudaGetLastError());
    std::vector<uint32_t> res(count * 6);
    CK(cudaMemcpyAsync(res.data(), d_res, res.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    mark("encode");
    for (int i = 0; i < count; ++i) {
        const uint32_t* r = &res[i * 6];
        if (r[3] | r[2]) return status_from_bits(r[3] | r[2]);
    }
    std::vector<uint64_t> soff(count);
    uint64_t stotal = 0;
    for (int i = 0; i < count; ++i) {
        nzgpu_blob_s* b = bs[i];
        const uint32_t* r = &res[i * 6];
        b->flags = (r[0] & (kFlagSingleSymbol | kFlagHas255)) | (irregular ? kFlagIrregular : 0u);
        b->single_symbol = r[1];
        b->stream_len = (uint64_t)r[4] | ((uint64_t)r[5] << 32);
        soff[i] = stotal;
        stotal += align_up(align_up(b->stream_len, 16) + 32, 256);
    }
    std::shared_ptr<void> stream_arena;
    if (count > 1) {
        if (int rc = arena_alloc(stotal, stream_arena, s)) return rc;
    }
    mark("str arena");
    // K4 copies: one launch for every chunk of the batch (the job table goes
    // where the encode tasks were: every kernel reading those is queued before)
    const size_t jb = stream_copy_job_bytes();
    std::vector<uint8_t> jobs(count > 1 ? count * jb : 0);
    uint64_t chunks_total = 0;
    for (int i = 0; i < count; ++i) {
        nzgpu_blob_s* b = bs[i];
        if (stream_arena) {
            b->stream_arena = stream_arena;
            b->stream = static_cast<uint8_t*>(stream_arena.get()) + soff[i];
        } else {
            CK(dev_alloc(reinterpret_cast<void**>(&b->stream), align_up(b->stream_len, 16) + 32, s));
        }
        if (count > 1) {
            stream_copy_job_fill(jobs.data() + i * jb, tasks[i].scratch, b->chunk_info, b->stream, tasks[i].hdr,
                                 chunks_total);
            chunks_total += b->nchunks;
        } else {
            CK(cudaMemcpyAsync(b->stream, tasks[i].hdr, 4, cudaMemcpyDeviceToDevice, s));
            stream_copy_kernel<<<(unsigned)b->nchunks, 256, 0, s>>>(tasks[i].scratch, slot, b->chunk_info, b->stream);
            CK(cudaGetLastError());
        }
    }
    if (count > 1) {
        static_assert(sizeof(EncTask) >= 40, "the job table reuses the task table's space");
        CK(cudaMemcpyAsync(tmp + L.tasks, jobs.data(), jobs.size(), cudaMemcpyHostToDevice, s));
        CK(launch_stream_copy_batch(tmp + L.tasks, count, chunks_total, slot, s));
    }
    mark("streams");
    // the readback arrays (6 pointers and 6 words per blob) are free again
    static_assert(sizeof(EncTask) >= sizeof(DecodeDesc), "the descriptor table reuses the task table's space");
    const int rc = compute_windows(bs, count, s, tmp + L.ptrs, reinterpret_cast<uint32_t*>(tmp + L.res), tmp + L.tasks);
    // a caller's workspace must be free to reuse when this returns
    if (ws) CK(cudaStreamSynchronize(s));
    mark("windows");
    return rc;
}

int compress_into(nzgpu_blob_s* b, const uint16_t* v, uint64_t n, int precision, uint32_t block,
                  uint32_t chunk_syms, uint32_t interval, cudaStream_t s) {
    return compress_many(&b, &v, &n, 1, precision, block, chunk_syms, interval, s);
}

// Device-tier calls run on the caller's stream (NULL = the legacy default
// stream); host-tier calls (OwnStream) use a private non-blocking stream.
struct StreamGuard {
    cudaStream_t s = nullptr;
    bool own = false;
    explicit StreamGuard(void* user) : s(static_cast<cudaStream_t>(user)) {}
    struct Own {};
    explicit StreamGuard(Own) {
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) own = true;
    }
    ~StreamGuard() {
        if (own) cudaStreamDestroy(s);
    }
};

}  // namespace

// ------------------------------------------------------------------ plan --
struct nzgpu_plan_s {
    int count = 0;
    int precision = 7;
    int log2k = 7;
    uint64_t tiles = 0;
    uint32_t win_cap = 0;
    DecodeDesc* d_descs = nullptr;
    uint64_t* d_prefix = nullptr;
    uint32_t* d_err = nullptr;
    // persistent schedule
    uint32_t ctas = 0, upc = 1, win_cap_unit = 0;
    uint32_t* d_cta_prefix = nullptr;
    std::vector<uint64_t> tunits;  // work units per tensor
    int ntiny = 0;                 // trailing tensors outside the resident-wave budget
    uint32_t max_ctas = 0;         // 0 = every resident CTA (nzgpu_plan_set_max_ctas)
    ~nzgpu_plan_s() {
        if (d_descs) cudaFree(d_descs);
        if (d_prefix) cudaFree(d_prefix);
        if (d_err) cudaFree(d_err);
        if (d_cta_prefix) cudaFree(d_cta_prefix);
    }
};

// Persistent schedule of a plan: every CTA owns `upc` units of one tensor.
// The per-tensor round-up must not push the CTA count past one resident wave
// (a second wave of a few CTAs doubles the launch time), so upc is the
// smallest value with sum_i ceil(units_i / upc) <= resident CTAs.  Returns
// the per-tensor first-CTA prefix.
std::vector<uint32_t> persist_geometry(nzgpu_plan_s* p) {
    std::vector<uint32_t> cta_prefix;
    uint64_t units = 0;
    for (uint64_t u : p->tunits) units += u;
    p->ctas = 0;
    if (!units) return cta_prefix;
    uint64_t resident = std::max<uint32_t>(1, persist_resident_ctas(p->log2k, p->win_cap_unit));
    if (p->max_ctas) resident = std::min<uint64_t>(resident, p->max_ctas);
    auto ctas_all = [&](uint64_t upc) {
        uint64_t c = 0;
        for (uint64_t u : p->tunits) c += ceil_div(u, upc);
        return c;
    };
    // Tiny tensors (the trailing p->ntiny, e.g. a layer's norms) are left out
    // of the one-wave budget: their few units run as extra CTAs that the SMs
    // pick up in the launch's tail instead of each holding an SM for the
    // whole launch.
    const size_t nbig = p->tunits.size() - (size_t)p->ntiny;
    auto ctas_big = [&](uint64_t upc) {
        uint64_t c = 0;
        for (size_t i = 0; i < nbig; ++i) c += ceil_div(p->tunits[i], upc);
        return c;
    };
    // Under an explicit cap (nzgpu_plan_set_max_ctas) every CTA counts: the
    // caller promised the other SMs to concurrent work.
    const bool tiny_outside = p->ntiny && !p->max_ctas;
    auto ctas_for = [&](uint64_t upc) { return tiny_outside ? ctas_big(upc) : ctas_all(upc); };
    uint64_t bunits = 0;
    for (size_t i = 0; i < nbig; ++i) bunits += p->tunits[i];
    const uint64_t umax = *std::max_element(p->tunits.begin(), p->tunits.end());
    uint64_t lo = std::max<uint64_t>(1, ceil_div(tiny_outside ? bunits : units, resident)), hi = lo;
    while (hi < umax && ctas_for(hi) > resident) hi *= 2;  // more tensors than CTAs: several waves
    hi = std::max(lo, std::min(hi, umax));
    while (lo < hi) {  // smallest upc in [lo, hi] that fits one wave
        const uint64_t mid = (lo + hi) / 2;
        if (ctas_for(mid) > resident) lo = mid + 1; else hi = mid;
    }
    p->upc = (uint32_t)lo;
    uint32_t ctas = 0;
    for (uint64_t u : p->tunits) {
        cta_prefix.push_back(ctas);
        ctas += (uint32_t)ceil_div(u, p->upc);
    }
    p->ctas = ctas;
    return cta_prefix;
}

// =================================================================== C ABI
extern "C" {

const char* nzgpu_status_string(int status) {
    switch (status) {
        case NZGPU_OK: return "ok";
        case NZGPU_INVALID_ARGUMENT: return "invalid argument";
        case NZGPU_FORMAT_TRUNCATED: return "ans decode: truncated chunk payload";
        case NZGPU_FORMAT_DESYNC: return "ans decode: state desynchronization";
        case NZGPU_FORMAT_LENGTH: return "payload length mismatch";
        case NZGPU_NONFINITE: return "compress_lossy: NaN/Inf in input";
        case NZGPU_FORMAT_TABLE: return "frequency table does not sum to 4096";
        case NZGPU_CUDA_ERROR: return "CUDA error";
        case NZGPU_OUT_OF_MEMORY: return "out of device memory";
        case NZGPU_NO_DEVICE: return "no CUDA device (the codec has no CPU fallback)";
        case NZGPU_CHECKSUM: return "nzt: checksum failure";
        default: return "unknown status";
    }
}

int nzgpu_version(void) { return 100; }

int nzgpu_set_decode_kernel(int which) {
    if (which != 0 && which != 1) return NZGPU_INVALID_ARGUMENT;
    g_kernel = which;
    return NZGPU_OK;
}

const char* nzgpu_last_error_message(void) { return g_msg; }

int nzgpu_device_check(int* device_count) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) {
        cudaGetLastError();
        count = 0;
    }
    if (device_count) *device_count = count;
    return count > 0 ? NZGPU_OK : NZGPU_NO_DEVICE;
}

int nzgpu_compress(const uint16_t* d_values, uint64_t n, int precision, uint32_t block_size,
                   uint32_t chunk_symbols, uint32_t interval, void* cuda_stream, nzgpu_blob* out) {
    if (!out) return NZGPU_INVALID_ARGUMENT;
    *out = nullptr;
    if (int rc = device_ready()) return rc;
    std::unique_ptr<nzgpu_blob_s> b(new (std::nothrow) nzgpu_blob_s);
    if (!b) return NZGPU_OUT_OF_MEMORY;
    StreamGuard sg(cuda_stream);
    const int rc = compress_into(b.get(), d_values, n, precision, block_size, chunk_symbols, interval, sg.s);
    if (sg.own) cudaStreamSynchronize(sg.s);
    if (rc) return rc;
    *out = b.release();
    return NZGPU_OK;
}

int nzgpu_compress_batch_workspace_size(const uint64_t* n, int count, int precision, uint32_t chunk_symbols,
                                        uint64_t* bytes) {
    if (!bytes || count <= 0 || !n || !valid_precision(precision)) return NZGPU_INVALID_ARGUMENT;
    *bytes = BatchLayout(n, count, precision, chunk_symbols ? chunk_symbols : kDefaultChunk).size;
    return NZGPU_OK;
}

int nzgpu_compress_batch(const uint16_t* const* d_values, const uint64_t* n, int count, int precision,
                         uint32_t block_size, uint32_t chunk_symbols, uint32_t interval, void* d_workspace,
                         uint64_t workspace_bytes, void* cuda_stream, nzgpu_blob* out) {
    if (!out || count <= 0 || !d_values || !n) return NZGPU_INVALID_ARGUMENT;
    for (int i = 0; i < count; ++i) out[i] = nullptr;
    if (int rc = device_ready()) return rc;
    std::vector<std::unique_ptr<nzgpu_blob_s>> bs(count);
    std::vector<nzgpu_blob_s*> raw(count);
    for (int i = 0; i < count; ++i) {
        bs[i].reset(new (std::nothrow) nzgpu_blob_s);
        if (!bs[i]) return NZGPU_OUT_OF_MEMORY;
        raw[i] = bs[i].get();
    }
    StreamGuard sg(cuda_stream);
    const int rc = compress_many(raw.data(), d_values, n, count, precision, block_size, chunk_symbols, interval, sg.s,
                                 d_workspace, workspace_bytes);
    if (rc) {
        cudaStreamSynchronize(sg.s);  // in-flight kernels may still write the blobs' buffers
        return rc;
    }
    for (int i = 0; i < count; ++i) out[i] = bs[i].release();
    return NZGPU_OK;
}

int nzgpu_decompress(nzgpu_blob blob, uint16_t* d_out, void* cuda_stream) {
    if (!blob || (!d_out && blob->n) || (reinterpret_cast<uintptr_t>(d_out) & 15)) return NZGPU_INVALID_ARGUMENT;
    return decode_blob(blob, d_out, static_cast<cudaStream_t>(cuda_stream));
}

int nzgpu_blob_status(nzgpu_blob blob, void* cuda_stream) {
    if (!blob) return NZGPU_INVALID_ARGUMENT;
    return sync_status(static_cast<cudaStream_t>(cuda_stream), blob->err, true);
}

int nzgpu_blob_info_get(nzgpu_blob b, nzgpu_blob_info* info) {
    if (!b || !info) return NZGPU_INVALID_ARGUMENT;
    std::memset(info, 0, sizeof(*info));
    info->n = b->n;
    info->precision = b->precision;
    info->block_size = b->block;
    info->chunk_symbols = b->chunk_syms;
    info->interval = b->interval;
    info->num_chunks = b->nchunks;
    info->stream_len = b->stream_len;
    info->mantissa_len = b->mant_len;
    info->scales_len = b->scales_len;
    info->index_len = (b->flags & kFlagIrregular) ? 0 : sizeof(IndexHeader) + index_region_bytes(b->nsub);
    info->payload_bytes = b->stream_len + b->mant_len + b->scales_len + 512;
    info->d_stream = b->stream;
    info->d_freqs = b->freqs;
    info->d_mantissas = b->mant;
    info->d_scales = b->scales_len ? b->scales : nullptr;
    info->flags = b->flags;
    info->max_window = b->max_window;
    return NZGPU_OK;
}

int nzgpu_blob_free(nzgpu_blob blob) {
    delete blob;
    return NZGPU_OK;
}

namespace {
int d2h_staged(const void* src, uint64_t bytes, cudaStream_t s,
               const std::function<void(uint64_t, const uint8_t*, uint64_t)>& sink);
void par_memcpy(void* dst, const void* src, uint64_t bytes);
// One section to host memory: large ones through the pinned ring and the
// host workers (pageable destinations fault in parallel), small ones direct.
int d2h_section(void* dst, const void* src, uint64_t bytes, cudaStream_t s) {
    if (!bytes) return NZGPU_OK;
    if (bytes < (4ull << 20)) {
        CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
        return NZGPU_OK;
    }
    uint8_t* d = static_cast<uint8_t*>(dst);
    return d2h_staged(src, bytes, s, [d](uint64_t a, const uint8_t* h, uint64_t len) { par_memcpy(d + a, h, len); });
}
}  // namespace

int nzgpu_blob_export(nzgpu_blob b, uint16_t* freqs, uint8_t* stream, uint8_t* mantissas, uint8_t* scales,
                      void* index) {
    if (!b) return NZGPU_INVALID_ARGUMENT;
    CK(cudaDeviceSynchronize());
    StreamGuard sg{StreamGuard::Own{}};
    if (freqs) CK(cudaMemcpy(freqs, b->freqs, 512, cudaMemcpyDeviceToHost));
    if (stream)
        if (int rc = d2h_section(stream, b->stream, b->stream_len, sg.s)) return rc;
    if (mantissas)
        if (int rc = d2h_section(mantissas, b->mant, b->mant_len, sg.s)) return rc;
    if (scales)
        if (int rc = d2h_section(scales, b->scales, b->scales_len, sg.s)) return rc;
    if (index && !(b->flags & kFlagIrregular)) {
        IndexHeader h{kIndexMagic, kIndexVersion, b->chunk_syms, b->interval, b->n, b->nchunks, b->nsub, b->stream_len,
                      b->max_window_unit, 0};
        std::memcpy(index, &h, sizeof(h));
        if (b->nsub)
            if (int rc = d2h_section(static_cast<uint8_t*>(index) + sizeof(h), b->index, index_region_bytes(b->nsub),
                                     sg.s))
                return rc;
    }
    return NZGPU_OK;
}

int nzgpu_blob_import(const nzgpu_host_tensor* t, uint32_t interval, void* cuda_stream, nzgpu_blob* out) {
    if (!out) return NZGPU_INVALID_ARGUMENT;
    *out = nullptr;
    if (int rc = device_ready()) return rc;
    std::unique_ptr<nzgpu_blob_s> b(new (std::nothrow) nzgpu_blob_s);
    if (!b) return NZGPU_OUT_OF_MEMORY;
    StreamGuard sg(cuda_stream);
    const int rc = import_into(b.get(), t, interval, sg.s);
    cudaStreamSynchronize(sg.s);
    if (rc) return rc;
    *out = b.release();
    return NZGPU_OK;
}

int nzgpu_plan_create(const nzgpu_blob* blobs, uint16_t* const* d_outs, int count, nzgpu_plan* out) {
    if (!out || count <= 0 || !blobs || !d_outs) return NZGPU_INVALID_ARGUMENT;
    *out = nullptr;
    std::unique_ptr<nzgpu_plan_s> p(new (std::nothrow) nzgpu_plan_s);
    if (!p) return NZGPU_OUT_OF_MEMORY;
    p->count = count;
    p->precision = blobs[0]->precision;
    p->log2k = blobs[0]->log2k;
    std::vector<DecodeDesc> descs;
    std::vector<uint64_t> prefix;
    CK(cudaMalloc(&p->d_err, 16));
    CK(cudaMemset(p->d_err, 0, 16));
    uint64_t tiles = 0;
    // Descriptor order: tensors with fewer units than 1/16 of a CTA's average
    // share go last (see persist_geometry); each descriptor carries its own
    // output, so the order is free.
    std::vector<int> order;
    {
        uint64_t units = 0, wcap = 0;
        for (int i = 0; i < count; ++i) {
            nzgpu_blob_s* b = blobs[i];
            if (!b) return NZGPU_INVALID_ARGUMENT;
            units += ceil_div(ceil_div(b->n, 1ull << p->log2k), 32);
            wcap = std::max<uint64_t>(wcap, b->max_window_unit);
        }
        const uint64_t resident = std::max<uint32_t>(1, persist_resident_ctas(p->log2k, (uint32_t)wcap));
        const uint64_t tiny_max = units / resident / 16;
        std::vector<int> tiny;
        for (int i = 0; i < count; ++i) {
            const uint64_t u = ceil_div(ceil_div(blobs[i]->n, 1ull << p->log2k), 32);
            (u <= tiny_max ? tiny : order).push_back(i);
        }
        if (order.empty()) std::swap(order, tiny);  // only tiny tensors: no special case
        p->ntiny = 0;
        for (int i : tiny) {
            order.push_back(i);
            if (blobs[i]->n) ++p->ntiny;
        }
    }
    for (int i : order) {
        nzgpu_blob_s* b = blobs[i];
        if (!b || b->precision != p->precision || b->log2k != p->log2k || (b->flags & kFlagIrregular) ||
            (reinterpret_cast<uintptr_t>(d_outs[i]) & 15))
            return NZGPU_INVALID_ARGUMENT;
        if (b->n == 0) continue;
        DecodeDesc d = b->desc(d_outs[i]);
        d.err = p->d_err;
        descs.push_back(d);
        prefix.push_back(tiles);
        tiles += b->tiles();
        p->win_cap = std::max(p->win_cap, b->max_window);
        p->win_cap_unit = std::max(p->win_cap_unit, b->max_window_unit);
    }
    p->tiles = tiles;
    p->count = (int)descs.size();
    for (const DecodeDesc& d : descs) p->tunits.push_back(ceil_div(ceil_div(d.n, 1ull << p->log2k), 32));
    const std::vector<uint32_t> cta_prefix = persist_geometry(p.get());
    if (!descs.empty()) {
        CK(cudaMalloc(&p->d_descs, descs.size() * sizeof(DecodeDesc)));
        CK(cudaMalloc(&p->d_prefix, prefix.size() * sizeof(uint64_t)));
        CK(cudaMalloc(&p->d_cta_prefix, cta_prefix.size() * sizeof(uint32_t)));
        CK(cudaMemcpy(p->d_descs, descs.data(), descs.size() * sizeof(DecodeDesc), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_prefix, prefix.data(), prefix.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->d_cta_prefix, cta_prefix.data(), cta_prefix.size() * sizeof(uint32_t),
                      cudaMemcpyHostToDevice));
    }
    *out = p.release();
    return NZGPU_OK;
}

int nzgpu_plan_launch(nzgpu_plan p, void* cuda_stream) {
    if (!p) return NZGPU_INVALID_ARGUMENT;
    if (!p->tiles) return NZGPU_OK;
    DecodeDesc none{};
    if (use_persist() && persist_fits(p->log2k, p->win_cap_unit)) {
        CK(launch_decode_persist(p->log2k, p->precision, p->d_descs, p->count, p->d_cta_prefix, none, p->ctas, p->upc,
                                 p->win_cap_unit, static_cast<cudaStream_t>(cuda_stream)));
    } else {
        CK(launch_decode(p->log2k, p->precision, p->d_descs, p->count, p->d_prefix, none, p->tiles, p->win_cap,
                         static_cast<cudaStream_t>(cuda_stream)));
    }
    return NZGPU_OK;
}

int nzgpu_plan_status(nzgpu_plan p, void* cuda_stream) {
    if (!p) return NZGPU_INVALID_ARGUMENT;
    return sync_status(static_cast<cudaStream_t>(cuda_stream), p->d_err, true);
}

int nzgpu_plan_free(nzgpu_plan p) {
    delete p;
    return NZGPU_OK;
}

int nzgpu_plan_launch_count(nzgpu_plan p) { return p && p->tiles ? 1 : 0; }

int nzgpu_plan_set_max_ctas(nzgpu_plan p, uint32_t max_ctas) {
    if (!p) return NZGPU_INVALID_ARGUMENT;
    // The schedule lives in device memory that in-flight launches of this plan
    // read: wait for every queued launch (any stream) before rewriting it.
    CK(cudaDeviceSynchronize());
    p->max_ctas = max_ctas;
    const std::vector<uint32_t> cta_prefix = persist_geometry(p);
    if (!cta_prefix.empty())
        CK(cudaMemcpy(p->d_cta_prefix, cta_prefix.data(), cta_prefix.size() * sizeof(uint32_t),
                      cudaMemcpyHostToDevice));
    return NZGPU_OK;
}

int nzgpu_plan_kernel(nzgpu_plan p) {
    if (!p || !p->tiles) return -1;
    return use_persist() && persist_fits(p->log2k, p->win_cap_unit) ? 0 : 1;
}

// ---------------------------------------------------------------- host tier
namespace {
int h2d_staged(void* dst, const void* src, uint64_t bytes, cudaStream_t s);
}

int nzgpu_compress_host(const uint16_t* values, uint64_t n, int precision, uint32_t block_size,
                        uint32_t chunk_symbols, uint32_t interval, nzgpu_blob* out) {
    if (!out) return NZGPU_INVALID_ARGUMENT;
    *out = nullptr;
    if (int rc = device_ready()) return rc;
    if (!values || n == 0) return NZGPU_INVALID_ARGUMENT;
    StreamGuard sg{StreamGuard::Own{}};
    uint16_t* d = nullptr;
    CK(cudaMallocAsync(&d, n * 2 + 16, sg.s));
    if (int rc = h2d_staged(d, values, n * 2, sg.s)) {
        cudaFreeAsync(d, sg.s);
        cudaStreamSynchronize(sg.s);
        return rc;
    }
    std::unique_ptr<nzgpu_blob_s> b(new (std::nothrow) nzgpu_blob_s);
    int rc = compress_into(b.get(), d, n, precision, block_size, chunk_symbols, interval, sg.s);
    cudaFreeAsync(d, sg.s);
    cudaStreamSynchronize(sg.s);
    if (rc) return rc;
    *out = b.release();
    return NZGPU_OK;
}

namespace {

// Grow-only device buffer owned by a host-pipeline slot.
struct DevBuf {
    void* p = nullptr;
    uint64_t cap = 0;
    int ensure(uint64_t bytes, cudaStream_t s) {
        if (cap >= bytes) return NZGPU_OK;
        CK(cudaStreamSynchronize(s));  // the previous tensor of this slot may still use it
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const uint64_t want = align_up(bytes + bytes / 4, 1 << 20);
        CK(cudaMalloc(&p, want));
        cap = want;
        return NZGPU_OK;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// One of two pipeline slots: tensor i runs on slot i%2 (own stream), so the
// H2D of tensor i+1, the decode of tensor i and the D2H of tensor i-1
// overlap; buffers persist across calls (no per-call cudaMalloc).
struct HostSlot {
    // s: table build, decode and D2H; s_in: the H2D of the compressed
    // sections.  With one stream a slot's next H2D queued behind its previous
    // D2H; now it waits only until the previous decode has read the inputs
    // (in_free), and the decode waits for its own inputs (h2d_done).
    cudaStream_t s = nullptr, s_in = nullptr;
    cudaEvent_t in_free = nullptr, h2d_done = nullptr;
    DevBuf main, stream, out;
    uint32_t* err = nullptr;
    // Pinned staging for the host-built chunk table: a cudaMemcpyAsync from
    // pageable memory may wait for the stream, which would serialise this
    // slot's H2D behind the previous tensor's D2H.  A ring of buffers, so the
    // host only ever waits for a copy issued four tensors ago.
    static constexpr int kRing = 4;
    uint4* info_h[kRing] = {};
    uint64_t info_cap[kRing] = {};
    cudaEvent_t info_done[kRing] = {};
    bool info_pending[kRing] = {};
    int ring = 0;
    ~HostSlot() {
        if (err) cudaFree(err);
        for (int i = 0; i < kRing; ++i) {
            if (info_h[i]) cudaFreeHost(info_h[i]);
            if (info_done[i]) cudaEventDestroy(info_done[i]);
        }
        if (in_free) cudaEventDestroy(in_free);
        if (h2d_done) cudaEventDestroy(h2d_done);
        if (s) cudaStreamDestroy(s);
        if (s_in) cudaStreamDestroy(s_in);
    }
    int sync() {
        if (s) CK(cudaStreamSynchronize(s));
        if (s_in) CK(cudaStreamSynchronize(s_in));
        return NZGPU_OK;
    }
    // Copy `info` into the next ring buffer; returns it (the caller issues the
    // H2D and then info_issued()).
    int stage_info(const std::vector<uint4>& info, uint4** buf) {
        const int r = ring;
        if (info_pending[r]) CK(cudaEventSynchronize(info_done[r]));
        info_pending[r] = false;
        if (info.size() > info_cap[r]) {  // grow generously: pinned allocations synchronise
            if (info_h[r]) CK(cudaFreeHost(info_h[r]));
            info_h[r] = nullptr;
            const uint64_t want = std::max<uint64_t>({info.size(), 2 * info_cap[r], 8192});
            info_cap[r] = 0;
            CK(cudaMallocHost(&info_h[r], want * sizeof(uint4)));
            info_cap[r] = want;
        }
        std::memcpy(info_h[r], info.data(), info.size() * sizeof(uint4));
        *buf = info_h[r];
        return NZGPU_OK;
    }
    int info_issued() {
        CK(cudaEventRecord(info_done[ring], s_in));
        info_pending[ring] = true;
        ring = (ring + 1) % kRing;
        return NZGPU_OK;
    }
};

// Slots in flight: slot i % kHostSlots stages tensor i.  A slot's H2D of the
// next tensor queues behind its D2H of the previous one (one stream), so
// with few slots a large tensor after a small one leaves the D2H engine
// idle.  Measured on 4 Llama-3-8B layers (PCIe ceiling 86 GB/s): 2 slots
// 62 GB/s, 4: 73, 6: 78, 8: 80.
#ifndef NZ_HOST_SLOTS
#define NZ_HOST_SLOTS 8
#endif
constexpr int kHostSlots = NZ_HOST_SLOTS;

// Grow-only pinned host buffer (cudaMallocHost costs ~0.4 ms per MB, so it
// is kept per thread across calls).
struct PinnedBuf {
    void* p = nullptr;
    uint64_t cap = 0;
    int ensure(uint64_t bytes) {
        if (cap >= bytes) return NZGPU_OK;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const uint64_t want = align_up(std::max<uint64_t>(bytes + bytes / 4, 1 << 20), 1 << 20);
        CK(cudaMallocHost(&p, want));
        cap = want;
        return NZGPU_OK;
    }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

// Host worker threads for the copies between pageable user memory and pinned
// staging: one thread moves pinned -> pageable at ~14 GB/s and faults fresh
// pages at ~2 GB/s; eight reach ~50-75 GB/s and ~20 GB/s (measured on the
// B200 box, profiles/r02_hostpath.txt).  A process-wide pool; run() executes
// f(0..parts-1) on the workers and the caller and returns when all are done.
class HostPool {
public:
    static HostPool& get() {
        static HostPool pool(std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
        return pool;
    }
    int threads() const { return (int)workers_.size() + 1; }
    void run(int parts, const std::function<void(int)>& f) {
        if (parts <= 1 || workers_.empty()) {
            for (int i = 0; i < parts; ++i) f(i);
            return;
        }
        std::lock_guard<std::mutex> one_region(run_mu_);  // callers from several threads queue here
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &f;
        parts_ = parts;
        next_ = 0;
        left_ = parts;
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        work();
        lk.lock();
        done_cv_.wait(lk, [&] { return left_ == 0; });
        job_ = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (std::thread& t : workers_) t.join();
    }

private:
    explicit HostPool(unsigned n) {
        for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    void work() {
        for (;;) {
            int i;
            const std::function<void(int)>* f;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!job_ || next_ >= parts_) return;
                i = next_++;
                f = job_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (--left_ == 0) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_); });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    int parts_ = 0, next_ = 0, left_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// memcpy split over the host pool above ~512 KB (pieces of >= 256 KB: the
// pipelined host decode copies a few MB per slice, and one thread moves
// only ~14 GB/s).
void par_memcpy(void* dst, const void* src, uint64_t bytes) {
    constexpr uint64_t kPiece = 256ull << 10;
    if (bytes < 2 * kPiece) {
        std::memcpy(dst, src, bytes);
        return;
    }
    HostPool& pool = HostPool::get();
    const int parts = (int)std::min<uint64_t>((uint64_t)pool.threads() * 2, ceil_div(bytes, kPiece));
    const uint64_t step = align_up(ceil_div(bytes, (uint64_t)parts), 64);
    pool.run(parts, [&](int i) {
        const uint64_t a = (uint64_t)i * step;
        if (a < bytes)
            std::memcpy(static_cast<uint8_t*>(dst) + a, static_cast<const uint8_t*>(src) + a,
                        std::min(step, bytes - a));
    });
}

struct HostCtx {
    HostSlot slot[kHostSlots];
    // nzgpu_decompress_host_sections: gathered inputs and the D2H ring
    static constexpr int kOutRing = 3;
    PinnedBuf in, ring[kOutRing], in_ring[kOutRing];
    cudaEvent_t ring_ev[kOutRing] = {}, in_ev[kOutRing] = {};
    ~HostCtx() {
        for (cudaEvent_t& e : ring_ev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t& e : in_ev)
            if (e) cudaEventDestroy(e);
    }
    int init() {
        for (HostSlot& sl : slot) {
            if (!sl.s) CK(cudaStreamCreateWithFlags(&sl.s, cudaStreamNonBlocking));
            if (!sl.s_in) CK(cudaStreamCreateWithFlags(&sl.s_in, cudaStreamNonBlocking));
            if (!sl.in_free) {
                CK(cudaEventCreateWithFlags(&sl.in_free, cudaEventDisableTiming));
                CK(cudaEventRecord(sl.in_free, sl.s));  // nothing to wait for yet
            }
            if (!sl.h2d_done) CK(cudaEventCreateWithFlags(&sl.h2d_done, cudaEventDisableTiming));
            if (!sl.err) CK(cudaMalloc(&sl.err, 64));
            for (auto& ev : sl.info_done)
                if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        for (cudaEvent_t& e : ring_ev)
            if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (cudaEvent_t& e : in_ev)
            if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        return NZGPU_OK;
    }
};
thread_local std::unique_ptr<HostCtx> g_host;

constexpr uint64_t kStageSlice = 32ull << 20;  // pinned ring slice of the staged host copies

// Pageable host -> device in slices through the calling thread's pinned ring:
// host workers copy slice k+1 into its slot while slice k's DMA runs.  Returns
// once every slice is queued on `s` (the last slots may still be in flight;
// they are only reused after their events).
int h2d_staged(void* dst, const void* src, uint64_t bytes, cudaStream_t s) {
    if (!bytes) return NZGPU_OK;
    if (!g_host) g_host.reset(new HostCtx);
    HostCtx& hc = *g_host;
    if (int rc = hc.init()) return rc;
    const uint64_t slice = std::min(kStageSlice, bytes);
    // copies still reading the ring (an earlier section of the same call)
    // finish before a slot is reused or reallocated
    for (int r = 0; r < HostCtx::kOutRing; ++r) CK(cudaEventSynchronize(hc.ring_ev[r]));
    for (int r = 0; r < HostCtx::kOutRing; ++r)
        if (int rc = hc.ring[r].ensure(slice)) return rc;
    const uint64_t nslices = ceil_div(bytes, slice);
    for (uint64_t k = 0; k < nslices; ++k) {
        const int r = (int)(k % HostCtx::kOutRing);
        if (k >= (uint64_t)HostCtx::kOutRing) CK(cudaEventSynchronize(hc.ring_ev[r]));
        const uint64_t a = k * slice, len = std::min(slice, bytes - a);
        par_memcpy(hc.ring[r].p, static_cast<const uint8_t*>(src) + a, len);
        CK(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + a, hc.ring[r].p, len, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(hc.ring_ev[r], s));
    }
    return NZGPU_OK;
}

// Device -> host in slices through the pinned ring; `sink(offset, host, len)`
// consumes each slice (on the calling thread, typically with the host pool)
// while the next slices' DMA runs.  Synchronous.
int d2h_staged(const void* src, uint64_t bytes, cudaStream_t s,
               const std::function<void(uint64_t, const uint8_t*, uint64_t)>& sink) {
    if (!bytes) return NZGPU_OK;
    if (!g_host) g_host.reset(new HostCtx);
    HostCtx& hc = *g_host;
    if (int rc = hc.init()) return rc;
    const uint64_t slice = std::min(kStageSlice, bytes);
    for (int r = 0; r < HostCtx::kOutRing; ++r) CK(cudaEventSynchronize(hc.ring_ev[r]));
    for (int r = 0; r < HostCtx::kOutRing; ++r)
        if (int rc = hc.ring[r].ensure(slice)) return rc;
    const uint64_t nslices = ceil_div(bytes, slice);
    auto issue = [&](uint64_t k) -> int {
        const int r = (int)(k % HostCtx::kOutRing);
        const uint64_t a = k * slice, len = std::min(slice, bytes - a);
        CK(cudaMemcpyAsync(hc.ring[r].p, static_cast<const uint8_t*>(src) + a, len, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(hc.ring_ev[r], s));
        return NZGPU_OK;
    };
    for (uint64_t k = 0; k < std::min<uint64_t>(nslices, HostCtx::kOutRing); ++k)
        if (int rc = issue(k)) return rc;
    for (uint64_t k = 0; k < nslices; ++k) {
        const int r = (int)(k % HostCtx::kOutRing);
        CK(cudaEventSynchronize(hc.ring_ev[r]));
        const uint64_t a = k * slice;
        sink(a, static_cast<const uint8_t*>(hc.ring[r].p), std::min(slice, bytes - a));
        if (k + HostCtx::kOutRing < nslices)
            if (int rc = issue(k + HostCtx::kOutRing)) return rc;
    }
    return NZGPU_OK;
}

// Host replica of tile_window() over the host copy of the index's unit
// positions: the decode kernel's shared-memory window size without a device
// round trip (ts = sub-ranges per tile/unit, a multiple of 32).
uint32_t host_max_window(const std::vector<uint4>& info, const uint32_t* base, uint64_t nsub, uint32_t S, int log2k,
                         uint64_t ts) {
    const uint64_t spc = S >> log2k;
    // sub-range -> chunk by shift when S/K is a power of two (the default
    // 65536/64): this loop runs once per warp unit of every staged tensor
    const int sh = (spc & (spc - 1)) == 0 ? __builtin_ctzll(spc) : -1;
    auto chunk_of = [&](uint64_t j) { return sh >= 0 ? j >> sh : j / spc; };
    auto in_chunk = [&](uint64_t j) { return sh >= 0 ? j & (spc - 1) : j % spc; };
    uint64_t best = 0;
    for (uint64_t sub0 = 0; sub0 < nsub; sub0 += ts) {
        const uint64_t subs = std::min<uint64_t>(ts, nsub - sub0);
        const uint4 c0 = info[chunk_of(sub0)];
        const uint64_t lim0 = c0.z >= 4 ? c0.z - 4 : 0;
        const uint64_t a = ((uint64_t)c0.x | ((uint64_t)c0.y << 32)) +
                           (in_chunk(sub0) == 0 ? 0 : std::min<uint64_t>(base[sub0 >> 5], lim0));
        const uint64_t jl = sub0 + subs - 1, jn = jl + 1;
        const uint4 c1 = info[chunk_of(jl)];
        const uint64_t lim1 = c1.z >= 4 ? c1.z - 4 : 0;
        const bool chunk_end = ((in_chunk(jl) + 1) << log2k) >= c1.w;
        uint64_t b = ((uint64_t)c1.x | ((uint64_t)c1.y << 32)) +
                     ((jn < nsub && !chunk_end) ? std::min<uint64_t>(base[jn >> 5], lim1) : lim1);
        if (b < a) b = a;
        best = std::max<uint64_t>(best, align_up(b, 16) - (a & ~(uint64_t)15));
    }
    return (uint32_t)std::min<uint64_t>(best, 0xFFFFFFFFu);
}

// NZGPU_TRACE: host time per stage of stage_and_decode, summed over a batch.
double g_stage_us[6] = {};
struct StageClock {
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void lap(int k) {
        const auto now = std::chrono::steady_clock::now();
        g_stage_us[k] += std::chrono::duration<double, std::micro>(now - t).count();
        t = now;
    }
};

// Stage + decode one host tensor on a slot without any host synchronisation
// (uniform framing and a valid side index).  Returns 1 when the caller must
// take the general (synchronising) path instead.
int stage_and_decode(HostSlot& sl, const nzgpu_host_tensor* t, uint16_t* host_out) {
    if (!t || !valid_precision(t->precision) || !t->freqs || !t->index) return 1;
    StageClock clk;
    std::vector<uint4> info;
    uint64_t total = 0;
    if (walk_stream(t->stream, t->stream_len, info, total) || info.empty() || total != t->n) return 1;
    uint32_t sum = 0, single = 0xFFFFFFFFu;
    for (int i = 0; i < 256; ++i) {
        sum += t->freqs[i];
        if (t->freqs[i] == kProbScale) single = (uint32_t)i;
    }
    if (sum != kProbScale || t->mantissa_len != mant_bytes(t->n, t->precision)) return 1;
    if (t->precision != 7 && (t->block_size == 0 || t->scales_len != ceil_div(t->n, t->block_size))) return 1;
    IndexHeader h;
    if (t->index_len < sizeof(h)) return 1;
    std::memcpy(&h, t->index, sizeof(h));
    // a tensor shorter than one chunk has a single, short chunk: its chunk
    // size is the encoder's (from the index), not the first chunk's length
    const uint32_t S = info.size() == 1 && info[0].w <= h.chunk_syms ? h.chunk_syms : info[0].w;
    const int log2k = log2_of(h.interval);
    if (h.magic != kIndexMagic || h.version != kIndexVersion || log2k < 0 || h.chunk_syms != S || h.n != t->n ||
        h.nchunks != info.size() || h.stream_len != t->stream_len || S % h.interval ||
        h.nsub != ceil_div(t->n, h.interval) || t->index_len != sizeof(h) + index_region_bytes(h.nsub))
        return 1;
    for (size_t c = 0; c < info.size(); ++c)
        if (c + 1 < info.size() ? info[c].w != S : (info[c].w == 0 || info[c].w > S)) return 1;
    const uint8_t* ix = static_cast<const uint8_t*>(t->index) + sizeof(h);
    const uint32_t* ix_base = reinterpret_cast<const uint32_t*>(ix) + h.nsub;  // may be unaligned: memcpy'd below

    nzgpu_blob_s& b = *new (std::nothrow) nzgpu_blob_s;  // descriptor only; buffers belong to the slot
    std::unique_ptr<nzgpu_blob_s> guard(&b);
    b.owns = false;
    b.n = t->n;
    b.precision = t->precision;
    b.block = t->precision == 7 ? 0 : t->block_size;
    b.interval = h.interval;
    b.log2k = log2k;
    b.chunk_syms = S;
    b.nchunks = info.size();
    b.nsub = h.nsub;
    b.mant_len = t->mantissa_len;
    b.scales_len = t->precision == 7 ? 0 : t->scales_len;
    b.stream_len = t->stream_len;
    b.flags = (single != 0xFFFFFFFFu ? kFlagSingleSymbol : 0u) | (t->freqs[255] ? kFlagHas255 : 0u) |
              wide_scale_flag(t);
    b.single_symbol = single != 0xFFFFFFFFu ? single : 0u;
    Carve cv;
    const uint64_t o_freqs = cv.take(512), o_lut = cv.take(16384), o_mant = cv.take(b.mant_len + 16);
    const uint64_t o_scales = cv.take(std::max<uint64_t>(b.scales_len, 1));
    const uint64_t o_info = cv.take(info.size() * sizeof(uint4));
    const uint64_t o_index = cv.take(index_region_bytes(b.nsub) + 16), o_scr = cv.take(64);
    cudaStream_t s = sl.s, si = sl.s_in;
    clk.lap(0);  // parse + validate
    if (sl.main.cap < cv.size || sl.stream.cap < align_up(std::max<uint64_t>(t->stream_len, 1), 16) + 32)
        if (int rc = sl.sync()) return rc;  // reallocation: both streams idle
    if (int rc = sl.main.ensure(cv.size, s)) return rc;
    if (int rc = sl.stream.ensure(align_up(std::max<uint64_t>(t->stream_len, 1), 16) + 32, s)) return rc;
    if (int rc = sl.out.ensure(align_up(t->n * 2, 16) + 16, s)) return rc;
    uint8_t* m = static_cast<uint8_t*>(sl.main.p);
    b.freqs = reinterpret_cast<uint16_t*>(m + o_freqs);
    b.lut = reinterpret_cast<uint32_t*>(m + o_lut);
    b.mant = m + o_mant;
    b.scales = m + o_scales;
    b.chunk_info = reinterpret_cast<uint4*>(m + o_info);
    b.index = m + o_index;
    b.scratch_u32 = reinterpret_cast<uint32_t*>(m + o_scr);
    b.stream = static_cast<uint8_t*>(sl.stream.p);
    b.err = sl.err;
    clk.lap(1);  // buffers
    CK(cudaStreamWaitEvent(si, sl.in_free, 0));  // the slot's previous decode has read its inputs
    CK(cudaMemcpyAsync(b.freqs, t->freqs, 512, cudaMemcpyHostToDevice, si));
    CK(cudaMemcpyAsync(b.stream, t->stream, t->stream_len, cudaMemcpyHostToDevice, si));
    if (b.mant_len) CK(cudaMemcpyAsync(b.mant, t->mantissas, b.mant_len, cudaMemcpyHostToDevice, si));
    if (b.scales_len) CK(cudaMemcpyAsync(b.scales, t->scales, b.scales_len, cudaMemcpyHostToDevice, si));
    clk.lap(2);  // section copies
    uint4* info_pinned = nullptr;
    if (int rc = sl.stage_info(info, &info_pinned)) return rc;
    CK(cudaMemcpyAsync(b.chunk_info, info_pinned, info.size() * sizeof(uint4), cudaMemcpyHostToDevice, si));
    if (int rc = sl.info_issued()) return rc;
    CK(cudaMemcpyAsync(b.index, ix, index_region_bytes(b.nsub), cudaMemcpyHostToDevice, si));
    CK(cudaEventRecord(sl.h2d_done, si));
    CK(cudaStreamWaitEvent(s, sl.h2d_done, 0));
    build_table_kernel<<<1, 256, 0, s>>>(nullptr, b.freqs, nullptr, nullptr, b.lut, b.scratch_u32);
    CK(cudaGetLastError());
    clk.lap(3);  // chunk table + index + LUT
    if (!(b.flags & kFlagSingleSymbol)) {
        // the index's hint when plausible (at most 2 bytes per symbol plus the
        // framing of the two chunks a unit can touch), else a scan
        const uint64_t bound = 64ull * h.interval + 64;
        std::vector<uint32_t> units;  // the unit positions, aligned (the host index may not be)
        auto unit_pos = [&]() -> const uint32_t* {
            if (units.empty()) {
                units.resize(index_units(b.nsub));
                std::memcpy(units.data(), ix_base, units.size() * 4);
            }
            return units.data();
        };
        b.max_window_unit = h.max_window_unit && h.max_window_unit <= bound
                                ? h.max_window_unit
                                : host_max_window(info, unit_pos(), b.nsub, S, log2k, 32);
        // the tile window only matters when the persistent kernel cannot run
        if (!(use_persist() && persist_fits(log2k, b.max_window_unit)))
            b.max_window = host_max_window(info, unit_pos(), b.nsub, S, log2k, decode_tile_subs());
    }
    clk.lap(4);  // windows
    if (int rc = decode_blob(&b, static_cast<uint16_t*>(sl.out.p), s)) return rc;
    CK(cudaEventRecord(sl.in_free, s));
    if (t->n) CK(cudaMemcpyAsync(host_out, sl.out.p, t->n * 2, cudaMemcpyDeviceToHost, s));
    clk.lap(5);  // decode + D2H issue
    return NZGPU_OK;
}

}  // namespace

int nzgpu_blob_chunks(nzgpu_blob b, uint32_t* lens, uint32_t* nsyms) {
    if (!b || (b->nchunks && (!lens || !nsyms))) return NZGPU_INVALID_ARGUMENT;
    if (!b->nchunks) return NZGPU_OK;
    std::vector<uint4> info(b->nchunks);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(info.data(), b->chunk_info, b->nchunks * sizeof(uint4), cudaMemcpyDeviceToHost));
    for (uint64_t c = 0; c < b->nchunks; ++c) {
        lens[c] = info[c].z;
        nsyms[c] = info[c].w;
    }
    return NZGPU_OK;
}

int nzgpu_blob_export_chunks(nzgpu_blob b, uint16_t* freqs, uint8_t* const* chunk_payloads, uint8_t* mantissas,
                             uint8_t* scales, void* index) {
    if (!b || (b->nchunks && !chunk_payloads)) return NZGPU_INVALID_ARGUMENT;
    StreamGuard sg{StreamGuard::Own{}};
    CK(cudaDeviceSynchronize());  // the blob may have been produced on any stream
    std::vector<uint4> info(b->nchunks);
    if (b->nchunks) CK(cudaMemcpy(info.data(), b->chunk_info, b->nchunks * sizeof(uint4), cudaMemcpyDeviceToHost));
    for (uint64_t c = 0; c < b->nchunks; ++c)
        if (info[c].z && !chunk_payloads[c]) return NZGPU_INVALID_ARGUMENT;
    if (freqs) CK(cudaMemcpy(freqs, b->freqs, 512, cudaMemcpyDeviceToHost));
    // the stream's chunk payloads, scattered slice by slice (they are in
    // stream order, so the chunks overlapping a slice are a contiguous run)
    HostPool& pool = HostPool::get();
    uint64_t first = 0;
    auto scatter = [&](uint64_t a, const uint8_t* host, uint64_t len) {
        auto pos = [&](uint64_t c) { return (uint64_t)info[c].x | ((uint64_t)info[c].y << 32); };
        while (first < b->nchunks && pos(first) + info[first].z <= a) ++first;
        uint64_t last = first;
        while (last < b->nchunks && pos(last) < a + len) ++last;
        const uint64_t nc = last - first;
        if (!nc) return;
        const int parts = (int)std::min<uint64_t>((uint64_t)pool.threads() * 2, nc);
        const uint64_t per = ceil_div(nc, (uint64_t)parts);
        pool.run(parts, [&](int i) {
            for (uint64_t c = first + i * per; c < std::min(last, first + (i + 1) * per); ++c) {
                const uint64_t p0 = std::max(pos(c), a), p1 = std::min(pos(c) + info[c].z, a + len);
                if (p1 > p0) std::memcpy(chunk_payloads[c] + (p0 - pos(c)), host + (p0 - a), p1 - p0);
            }
        });
    };
    if (int rc = d2h_staged(b->stream, b->stream_len, sg.s, scatter)) return rc;
    auto into = [](uint8_t* dst) {
        return [dst](uint64_t a, const uint8_t* host, uint64_t len) { par_memcpy(dst + a, host, len); };
    };
    if (mantissas)
        if (int rc = d2h_staged(b->mant, b->mant_len, sg.s, into(mantissas))) return rc;
    if (scales && b->scales_len) CK(cudaMemcpy(scales, b->scales, b->scales_len, cudaMemcpyDeviceToHost));
    if (index && !(b->flags & kFlagIrregular)) {
        IndexHeader h{kIndexMagic, kIndexVersion, b->chunk_syms, b->interval, b->n, b->nchunks, b->nsub, b->stream_len,
                      b->max_window_unit, 0};
        std::memcpy(index, &h, sizeof(h));
        if (b->nsub)
            if (int rc = d2h_staged(b->index, index_region_bytes(b->nsub), sg.s,
                                    into(static_cast<uint8_t*>(index) + sizeof(h))))
                return rc;
    }
    return NZGPU_OK;
}

int nzgpu_decompress_host_batch(const nzgpu_host_tensor* ts, int count, uint16_t* const* outs) {
    if (count < 0 || (count && (!ts || !outs))) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    if (!g_host) g_host.reset(new HostCtx);
    HostCtx& h = *g_host;
    if (int rc = h.init()) return rc;
    for (HostSlot& sl : h.slot) CK(cudaMemsetAsync(sl.err, 0, 64, sl.s));
    static const bool trace = std::getenv("NZGPU_TRACE") != nullptr;
    double host_us = 0;
    int general = 0;
    const auto tcall = std::chrono::steady_clock::now();
    for (int i = 0; i < count; ++i) {
        HostSlot& sl = h.slot[i % kHostSlots];
        const nzgpu_host_tensor* t = ts + i;
        const auto t0 = std::chrono::steady_clock::now();
        int rc = stage_and_decode(sl, t, outs[i]);
        if (trace) host_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        if (rc == 1) {
            ++general;
            // General path (no/foreign index, irregular framing, or a format
            // error to report exactly): import with full validation.
            nzgpu_blob_s b;
            rc = import_into(&b, t, 0, sl.s);
            if (!rc && (rc = sl.out.ensure(align_up(t->n * 2, 16) + 16, sl.s)) == 0) {
                rc = decode_blob(&b, static_cast<uint16_t*>(sl.out.p), sl.s);
                if (!rc && t->n) {
                    const cudaError_t e = cudaMemcpyAsync(outs[i], sl.out.p, t->n * 2, cudaMemcpyDeviceToHost, sl.s);
                    if (e != cudaSuccess) rc = fail_cuda(e, "cudaMemcpyAsync");
                }
                if (!rc) rc = sync_status(sl.s, b.err, true);
            }
            if (!rc) CK(cudaStreamSynchronize(sl.s));  // b's buffers die here
        }
        if (rc) {
            for (HostSlot& other : h.slot) other.sync();
            return rc;
        }
    }
    int rc = NZGPU_OK;
    const auto t1 = std::chrono::steady_clock::now();
    for (HostSlot& sl : h.slot) {
        sl.sync();
        const int r = sync_status(sl.s, sl.err, true);
        if (!rc) rc = r;
    }
    if (trace) {
        std::fprintf(stderr, "nzgpu batch stages (us): parse %.0f buffers %.0f sections %.0f table %.0f windows %.0f "
                     "decode+d2h %.0f\n", g_stage_us[0], g_stage_us[1], g_stage_us[2], g_stage_us[3], g_stage_us[4],
                     g_stage_us[5]);
        for (double& v : g_stage_us) v = 0;
    }
    if (trace)
        std::fprintf(stderr, "nzgpu batch: %d tensors (%d general), host enqueue %.0f us, final wait %.0f us, call %.0f us\n",
                     count, general, host_us,
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t1).count(),
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tcall).count());
    return rc;
}

int nzgpu_decompress_host(const nzgpu_host_tensor* t, uint16_t* out) {
    // Into pageable memory, a direct D2H runs at 10-16 GB/s (2 GB/s into
    // untouched pages): a large tensor with a usable index takes the sliced
    // pipeline of nzgpu_decompress_host_sections instead (pinned ring, host
    // workers copy out and fault the pages in parallel), its chunk views
    // pointing into the serialized stream.
    if (t && out && t->index && t->stream && t->n >= (1u << 22) && device_ready() == NZGPU_OK) {
        cudaPointerAttributes a{};
        const bool pageable = cudaPointerGetAttributes(&a, out) == cudaSuccess && a.type == cudaMemoryTypeUnregistered;
        cudaGetLastError();  // a failed query leaves no sticky state
        std::vector<uint4> info;
        uint64_t total = 0;
        if (pageable && walk_stream(t->stream, t->stream_len, info, total) == NZGPU_OK && total == t->n) {
            std::vector<nzgpu_chunk_view> views(info.size());
            for (size_t c = 0; c < info.size(); ++c)
                views[c] = nzgpu_chunk_view{t->stream + ((uint64_t)info[c].x | ((uint64_t)info[c].y << 32)), info[c].z,
                                            info[c].w};
            nzgpu_host_sections h{};
            h.n = t->n;
            h.precision = t->precision;
            h.block_size = t->block_size;
            h.freqs = t->freqs;
            h.chunks = views.data();
            h.nchunks = views.size();
            h.mantissas = t->mantissas;
            h.mantissa_len = t->mantissa_len;
            h.scales = t->scales;
            h.scales_len = t->scales_len;
            h.index = t->index;
            h.index_len = t->index_len;
            return nzgpu_decompress_host_sections(&h, out);
        }
    }
    return nzgpu_decompress_host_batch(t, 1, &out);
}

int nzgpu_blob_decompress_host(nzgpu_blob b, uint16_t* out) {
    if (!b || (!out && b->n)) return NZGPU_INVALID_ARGUMENT;
    if (b->n == 0) return NZGPU_OK;
    StreamGuard sg{StreamGuard::Own{}};
    uint16_t* d = nullptr;
    CK(cudaMallocAsync(&d, align_up(b->n * 2, 16) + 16, sg.s));
    int rc = decode_blob(b, d, sg.s);
    if (!rc) {
        const cudaError_t e = cudaMemcpyAsync(out, d, b->n * 2, cudaMemcpyDeviceToHost, sg.s);
        if (e != cudaSuccess) rc = fail_cuda(e, "cudaMemcpyAsync");
    }
    cudaFreeAsync(d, sg.s);
    const int st = sync_status(sg.s, b->err, true);
    return rc ? rc : st;
}

namespace {

// Chunk table of the serialized form of chunk views (serialize_stream,
// ans.hpp:306-316): payload offset, length and symbol count per chunk.
void stream_layout(const nzgpu_host_sections* t, std::vector<uint4>& info) {
    info.resize(t->nchunks);
    uint64_t pos = 4;
    for (uint64_t c = 0; c < t->nchunks; ++c) {
        pos += 8;
        info[c] = make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), t->chunks[c].len, t->chunks[c].nsym);
        pos += t->chunks[c].len;
    }
}

// Serialize chunks [c0, c1) into `dst` (the whole stream's buffer; chunk 0
// also writes the leading chunk count), copied by the host pool.
void gather_chunks(const nzgpu_host_sections* t, uint8_t* dst, const std::vector<uint4>& info, uint64_t c0,
                   uint64_t c1) {
    if (c0 == 0) {
        const uint32_t cnt = (uint32_t)t->nchunks;
        std::memcpy(dst, &cnt, 4);
    }
    HostPool& pool = HostPool::get();
    const uint64_t nc = c1 - c0;
    const int parts = (int)std::min<uint64_t>((uint64_t)pool.threads() * 2, std::max<uint64_t>(1, nc));
    const uint64_t per = ceil_div(nc, (uint64_t)parts);
    pool.run(parts, [&](int i) {
        for (uint64_t c = c0 + i * per; c < std::min(c1, c0 + (i + 1) * per); ++c) {
            const uint64_t at = ((uint64_t)info[c].x | ((uint64_t)info[c].y << 32));
            std::memcpy(dst + at - 8, &info[c].w, 4);
            std::memcpy(dst + at - 4, &info[c].z, 4);
            if (info[c].z) std::memcpy(dst + at, t->chunks[c].payload, info[c].z);
        }
    });
}

void gather_stream(const nzgpu_host_sections* t, uint8_t* dst, std::vector<uint4>& info) {
    stream_layout(t, info);
    gather_chunks(t, dst, info, 0, t->nchunks);
}

// Slices of the pipelined host decode: a multiple of the chunk size, of the
// warp unit (32 sub-ranges) and of the lossy block; 0 = do not slice.
// (NZGPU_HOST_SLICE overrides the element count; 0 = one slice.)
uint64_t slice_elems() {
    static const uint64_t v = [] {
        const char* e = std::getenv("NZGPU_HOST_SLICE");
        return e ? std::strtoull(e, nullptr, 10) : 4ull << 20;
    }();
    return v;
}
uint64_t slice_grain(uint64_t S, uint64_t K, uint64_t B) {
    auto lcm = [](uint64_t x, uint64_t y) -> uint64_t {
        uint64_t a = x, c = y;
        while (c) {
            const uint64_t r = a % c;
            a = c;
            c = r;
        }
        const uint64_t l = x / a * y;
        return l / y == x / a ? l : 0;
    };
    uint64_t g = lcm(S, 32 * K);
    if (g && B) g = lcm(g, B);
    return g;
}

// General path of the sections call: serialize, then the validating host tier.
int sections_general(const nzgpu_host_sections* t, uint16_t* out) {
    uint64_t len = 4;
    for (uint64_t c = 0; c < t->nchunks; ++c) len += 8 + (uint64_t)t->chunks[c].len;
    std::vector<uint8_t> stream(len);
    std::vector<uint4> info;
    gather_stream(t, stream.data(), info);
    nzgpu_host_tensor h{};
    h.n = t->n;
    h.precision = t->precision;
    h.block_size = t->block_size;
    h.freqs = t->freqs;
    h.stream = stream.data();
    h.stream_len = len;
    h.mantissas = t->mantissas;
    h.mantissa_len = t->mantissa_len;
    h.scales = t->scales;
    h.scales_len = t->scales_len;
    h.index = t->index;
    h.index_len = t->index_len;
    return nzgpu_decompress_host_batch(&h, 1, &out);
}

}  // namespace

int nzgpu_decompress_host_sections(const nzgpu_host_sections* t, uint16_t* out) {
    if (!t || !valid_precision(t->precision) || !t->freqs || (t->nchunks && !t->chunks) || (t->n && !out))
        return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    // Fast path only for what the side index describes: uniform framing, a
    // matching v3 index, consistent sections (tensorstore.hpp:115-117,
    // :218-227).  Everything else -- including every malformed input, so the
    // error is reported exactly as the reference would -- goes general.
    IndexHeader h{};
    bool fast = t->index && t->index_len >= sizeof(h) && t->nchunks > 0 && t->n > 0;
    uint64_t stream_len = 4, total = 0;
    for (uint64_t c = 0; c < t->nchunks; ++c) {
        stream_len += 8 + (uint64_t)t->chunks[c].len;
        total += t->chunks[c].nsym;
        if (t->chunks[c].len && !t->chunks[c].payload) return NZGPU_INVALID_ARGUMENT;
    }
    uint32_t sum = 0, single = 0xFFFFFFFFu;
    for (int i = 0; i < 256; ++i) {
        sum += t->freqs[i];
        if (t->freqs[i] == kProbScale) single = (uint32_t)i;
    }
    fast = fast && total == t->n && sum == kProbScale && t->mantissa_len == mant_bytes(t->n, t->precision) &&
           (t->precision == 7 || (t->block_size && t->scales_len == ceil_div(t->n, t->block_size)));
    int log2k = -1;
    uint32_t S = 0;
    if (fast) {
        std::memcpy(&h, t->index, sizeof(h));
        S = t->nchunks == 1 && t->chunks[0].nsym <= h.chunk_syms ? h.chunk_syms : t->chunks[0].nsym;
        log2k = log2_of(h.interval);
        fast = h.magic == kIndexMagic && h.version == kIndexVersion && log2k >= 0 && h.chunk_syms == S &&
               h.n == t->n && h.nchunks == t->nchunks && h.stream_len == stream_len && S % h.interval == 0 &&
               h.nsub == ceil_div(t->n, h.interval) && t->index_len == sizeof(h) + index_region_bytes(h.nsub);
        for (uint64_t c = 0; fast && c < t->nchunks; ++c) {
            const uint32_t w = t->chunks[c].nsym;
            fast = c + 1 < t->nchunks ? w == S : (w != 0 && w <= S);
        }
    }
    if (!fast) return sections_general(t, out);

    if (!g_host) g_host.reset(new HostCtx);
    HostCtx& hc = *g_host;
    if (int rc = hc.init()) return rc;
    HostSlot& sl = hc.slot[0];
    cudaStream_t s = sl.s;
    if (int rc = sl.sync()) return rc;  // the slot's buffers and the pinned staging are free
    CK(cudaMemsetAsync(sl.err, 0, 64, s));

    nzgpu_blob_s& b = *new (std::nothrow) nzgpu_blob_s;  // descriptor over the slot's buffers
    std::unique_ptr<nzgpu_blob_s> guard(&b);
    b.owns = false;
    b.n = t->n;
    b.precision = t->precision;
    b.block = t->precision == 7 ? 0 : t->block_size;
    b.interval = h.interval;
    b.log2k = log2k;
    b.chunk_syms = S;
    b.nchunks = t->nchunks;
    b.nsub = h.nsub;
    b.mant_len = t->mantissa_len;
    b.scales_len = t->precision == 7 ? 0 : t->scales_len;
    b.stream_len = stream_len;
    uint32_t wide = 0;
    if (t->precision != 7)
        for (uint64_t i = 0; i < t->scales_len; ++i) wide |= t->scales[i] & 0x80u;
    b.flags = (single != 0xFFFFFFFFu ? kFlagSingleSymbol : 0u) | (t->freqs[255] ? kFlagHas255 : 0u) |
              (wide ? kFlagWideScale : 0u);
    b.single_symbol = single != 0xFFFFFFFFu ? single : 0u;

    // device buffers of the slot first, so each section's H2D can be issued
    // as soon as the host workers have gathered it into pinned staging
    // (gather of section k+1 overlaps the DMA of section k)
    Carve cv;
    const uint64_t o_freqs = cv.take(512), o_lut = cv.take(16384), o_mant = cv.take(b.mant_len + 16);
    const uint64_t o_scales = cv.take(std::max<uint64_t>(b.scales_len, 1));
    const uint64_t o_info = cv.take(b.nchunks * sizeof(uint4));
    const uint64_t o_index = cv.take(index_region_bytes(b.nsub) + 16), o_scr = cv.take(64);
    if (int rc = sl.main.ensure(cv.size, s)) return rc;
    if (int rc = sl.stream.ensure(align_up(stream_len, 16) + 32, s)) return rc;
    if (int rc = sl.out.ensure(align_up(t->n * 2, 16) + 16, s)) return rc;
    uint8_t* m = static_cast<uint8_t*>(sl.main.p);
    b.freqs = reinterpret_cast<uint16_t*>(m + o_freqs);
    b.lut = reinterpret_cast<uint32_t*>(m + o_lut);
    b.mant = m + o_mant;
    b.scales = m + o_scales;
    b.chunk_info = reinterpret_cast<uint4*>(m + o_info);
    b.index = m + o_index;
    b.scratch_u32 = reinterpret_cast<uint32_t*>(m + o_scr);
    b.stream = static_cast<uint8_t*>(sl.stream.p);
    b.err = sl.err;

    // pinned staging of the side tables: scales | index region | chunk table
    // | table (the stream and mantissa bytes go through a ring of slice-sized
    // slots below, so pinned memory does not grow with the tensor)
    Carve in;
    const uint64_t i_scales = in.take(b.scales_len);
    const uint64_t i_index = in.take(index_region_bytes(b.nsub)), i_info = in.take(b.nchunks * sizeof(uint4));
    const uint64_t i_freqs = in.take(512);
    if (int rc = hc.in.ensure(in.size)) return rc;
    uint8_t* stage = static_cast<uint8_t*>(hc.in.p);
    cudaStream_t si = sl.s_in;
    auto h2d = [&](void* dst, uint64_t at, uint64_t len) -> int {
        if (len) CK(cudaMemcpyAsync(dst, stage + at, len, cudaMemcpyHostToDevice, si));
        return NZGPU_OK;
    };
    std::vector<uint4> info;
    stream_layout(t, info);
    // the small side tables first: every slice's decode needs them
    par_memcpy(stage + i_index, static_cast<const uint8_t*>(t->index) + sizeof(h), index_region_bytes(b.nsub));
    std::memcpy(stage + i_info, info.data(), info.size() * sizeof(uint4));
    std::memcpy(stage + i_freqs, t->freqs, 512);
    if (int rc = h2d(b.index, i_index, index_region_bytes(b.nsub))) return rc;
    if (int rc = h2d(b.chunk_info, i_info, b.nchunks * sizeof(uint4))) return rc;
    if (int rc = h2d(b.freqs, i_freqs, 512)) return rc;
    if (b.scales_len) {
        par_memcpy(stage + i_scales, t->scales, b.scales_len);
        if (int rc = h2d(b.scales, i_scales, b.scales_len)) return rc;
    }
    CK(cudaEventRecord(sl.h2d_done, si));
    CK(cudaStreamWaitEvent(s, sl.h2d_done, 0));
    build_table_kernel<<<1, 256, 0, s>>>(nullptr, b.freqs, nullptr, nullptr, b.lut, b.scratch_u32);
    CK(cudaGetLastError());
    if (!(b.flags & kFlagSingleSymbol)) {
        const uint32_t* base = reinterpret_cast<const uint32_t*>(stage + i_index) + b.nsub;  // aligned copy
        const uint64_t bound = 64ull * h.interval + 64;
        b.max_window_unit = h.max_window_unit && h.max_window_unit <= bound
                                ? h.max_window_unit
                                : host_max_window(info, base, b.nsub, S, log2k, 32);
        if (!(use_persist() && persist_fits(log2k, b.max_window_unit)))
            b.max_window = host_max_window(info, base, b.nsub, S, log2k, decode_tile_subs());
    }

    // Element slices, each a whole number of chunks, warp units and lossy
    // blocks: the stream and mantissa bytes of slice p+1 are gathered and
    // copied in while slice p decodes and its bf16 comes back through the
    // pinned ring, so the two PCIe directions and the host copies overlap.
    uint16_t* d_out = static_cast<uint16_t*>(sl.out.p);
    const uint64_t n = t->n, grain = slice_grain(S, h.interval, t->precision == 7 ? 0 : t->block_size);
    // at most slice_elems() per slice, and at least four slices when the grain allows
    const uint64_t want = std::min(slice_elems(), n / 4);
    const uint64_t slice = grain && grain <= want ? grain * (want / grain) : grain && slice_elems() ? std::min(n, grain) : n;
    const uint64_t nslices = ceil_div(n, slice);
    for (int r = 0; r < HostCtx::kOutRing; ++r) {
        CK(cudaEventSynchronize(hc.ring_ev[r]));  // nothing in flight reads or writes a slot it may reallocate
        if (int rc = hc.ring[r].ensure(std::min(std::min(slice, n) * 2, kStageSlice))) return rc;
    }
    auto mant_at = [&](uint64_t e) { return t->precision == 7 ? e : e * (uint64_t)(t->precision + 1) / 8; };
    auto spos = [&](uint64_t c) { return c == b.nchunks ? stream_len : ((uint64_t)info[c].x | ((uint64_t)info[c].y << 32)) - 8; };
    // a slice's inputs: its stream bytes [s0, s1) and mantissa bytes [m0, m1)
    struct SliceIn {
        uint64_t a, len, c0, c1, s0, s1, m0, m1;
    };
    auto slice_in = [&](uint64_t p) {
        SliceIn x;
        x.a = p * slice;
        x.len = std::min(slice, n - x.a);
        x.c0 = x.a / S;
        x.c1 = p + 1 == nslices ? b.nchunks : (x.a + x.len) / S;
        x.s0 = p == 0 ? 0 : spos(x.c0);
        x.s1 = spos(x.c1);
        x.m0 = mant_at(x.a);
        x.m1 = p + 1 == nslices ? b.mant_len : mant_at(x.a + x.len);
        return x;
    };
    uint64_t slot_bytes = 0;
    for (uint64_t p = 0; p < nslices; ++p) {
        const SliceIn x = slice_in(p);
        slot_bytes = std::max(slot_bytes, align_up(x.s1 - x.s0, 16) + (x.m1 - x.m0));
    }
    for (int r = 0; r < HostCtx::kOutRing; ++r) {
        CK(cudaEventSynchronize(hc.in_ev[r]));  // an earlier call's H2D from this slot
        if ((uint64_t)r < nslices)
            if (int rc = hc.in_ring[r].ensure(slot_bytes)) return rc;
    }
    static const bool trace = std::getenv("NZGPU_TRACE") != nullptr;
    double us_gather = 0, us_wait = 0, us_out = 0;
    auto since = [](std::chrono::steady_clock::time_point t0) {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    };
    const auto t_call = std::chrono::steady_clock::now();
    // The host alternates: gather slice p, then copy the earlier slices'
    // output out of the ring.  The output goes D2H in pieces of at most one
    // ring slot (32 MB): one piece per slice normally; a slice larger than a
    // slot (a lossy block size no slice size divides: one slice) streams its
    // pieces through the 3-slot ring.  (A separate copy-out thread measured
    // no faster: the gathers and copy-outs share the host's memory bandwidth.)
    const uint64_t piece = std::min(std::min(slice, n) * 2, kStageSlice);
    struct Piece {
        uint64_t off, len;  // bytes of the bf16 output
    };
    std::vector<Piece> pieces;
    uint64_t issued = 0, copied = 0;
    auto copy_one = [&]() -> int {
        const int r = (int)(copied % HostCtx::kOutRing);
        auto t0 = std::chrono::steady_clock::now();
        CK(cudaEventSynchronize(hc.ring_ev[r]));
        us_wait += since(t0);
        t0 = std::chrono::steady_clock::now();
        par_memcpy(reinterpret_cast<uint8_t*>(out) + pieces[copied].off, hc.ring[r].p, pieces[copied].len);
        us_out += since(t0);
        ++copied;
        return NZGPU_OK;
    };
    auto issue_one = [&]() -> int {
        if (issued - copied == (uint64_t)HostCtx::kOutRing)  // its slot's previous piece is still to copy out
            if (int rc = copy_one()) return rc;
        const int r = (int)(issued % HostCtx::kOutRing);
        CK(cudaMemcpyAsync(hc.ring[r].p, reinterpret_cast<const uint8_t*>(d_out) + pieces[issued].off,
                           pieces[issued].len, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(hc.ring_ev[r], s));
        ++issued;
        return NZGPU_OK;
    };
    for (uint64_t p = 0; p < nslices; ++p) {
        const SliceIn x = slice_in(p);
        const uint64_t a = x.a, len = x.len;
        const int ri = (int)(p % HostCtx::kOutRing);
        if (p >= (uint64_t)HostCtx::kOutRing) CK(cudaEventSynchronize(hc.in_ev[ri]));  // slot's H2D of slice p-R
        uint8_t* slot = static_cast<uint8_t*>(hc.in_ring[ri].p);
        const uint64_t mat = align_up(x.s1 - x.s0, 16);
        const auto tg = std::chrono::steady_clock::now();
        gather_chunks(t, slot - x.s0, info, x.c0, x.c1);  // writes stream bytes [s0, s1) at slot[0..)
        par_memcpy(slot + mat, t->mantissas + x.m0, x.m1 - x.m0);
        us_gather += since(tg);
        if (x.s1 > x.s0) CK(cudaMemcpyAsync(b.stream + x.s0, slot, x.s1 - x.s0, cudaMemcpyHostToDevice, si));
        if (x.m1 > x.m0) CK(cudaMemcpyAsync(b.mant + x.m0, slot + mat, x.m1 - x.m0, cudaMemcpyHostToDevice, si));
        CK(cudaEventRecord(hc.in_ev[ri], si));
        CK(cudaEventRecord(sl.h2d_done, si));
        CK(cudaStreamWaitEvent(s, sl.h2d_done, 0));
        if (int rc = decode_range(&b, d_out, a, len, s)) return rc;
        const uint64_t first_new = pieces.size();
        for (uint64_t o = a * 2; o < (a + len) * 2; o += piece) pieces.push_back({o, std::min(piece, (a + len) * 2 - o)});
        while (issued < pieces.size())
            if (int rc = issue_one()) return rc;
        while (copied < first_new)  // the earlier slices' pieces
            if (int rc = copy_one()) return rc;
    }
    while (copied < pieces.size())
        if (int rc = copy_one()) return rc;
    if (trace)
        std::fprintf(stderr, "nzgpu sections: n=%llu slices=%llu gather %.0f us, wait %.0f us, copy-out %.0f us, call %.0f us\n",
                     (unsigned long long)n, (unsigned long long)nslices, us_gather, us_wait, us_out, since(t_call));
    return sync_status(s, sl.err, true);
}

int nzgpu_trim_device_pool(void) {
    cudaMemPool_t pool;
    CK(pool_of(&pool));
    CK(cudaDeviceSynchronize());
    CK(cudaMemPoolTrimTo(pool, 0));
    return NZGPU_OK;
}

int nzgpu_host_release(void) {
    if (g_host) {
        for (HostSlot& sl : g_host->slot) sl.sync();
        g_host.reset();
    }
    return NZGPU_OK;
}

// ------------------------------------------------------------ building blocks
int nzgpu_split(const uint16_t* d_values, uint64_t n, uint8_t* d_exponents, uint8_t* d_signmant, uint64_t* d_counts,
                void* cuda_stream) {
    if ((reinterpret_cast<uintptr_t>(d_values) & 15) || (reinterpret_cast<uintptr_t>(d_exponents) & 7) ||
        (reinterpret_cast<uintptr_t>(d_signmant) & 7))
        return NZGPU_INVALID_ARGUMENT;
    if (n == 0) return NZGPU_OK;
    CK(launch_split_hist(d_values, n, d_exponents, d_signmant, reinterpret_cast<unsigned long long*>(d_counts),
                         static_cast<cudaStream_t>(cuda_stream)));
    return NZGPU_OK;
}

int nzgpu_build_table(const uint64_t* d_counts, uint16_t* d_freqs, void* cuda_stream) {
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    uint32_t* info = nullptr;
    CK(cudaMallocAsync(&info, 16, s));
    CK(cudaMemsetAsync(info, 0, 16, s));
    build_table_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(d_counts), nullptr, d_freqs,
                                         nullptr, nullptr, info);
    CK(cudaGetLastError());
    uint32_t h[3];
    CK(cudaMemcpyAsync(h, info, 12, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(info, s));
    CK(cudaStreamSynchronize(s));
    return status_from_bits(h[2]);
}

int nzgpu_build_table_host(const uint64_t* counts, uint16_t* freqs) {
    if (!counts || !freqs) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg{StreamGuard::Own{}};
    uint64_t* dc = nullptr;
    uint16_t* df = nullptr;
    CK(cudaMallocAsync(&dc, 2048, sg.s));
    CK(cudaMallocAsync(&df, 512, sg.s));
    CK(cudaMemcpyAsync(dc, counts, 2048, cudaMemcpyHostToDevice, sg.s));
    const int rc = nzgpu_build_table(dc, df, sg.s);
    if (!rc) CK(cudaMemcpyAsync(freqs, df, 512, cudaMemcpyDeviceToHost, sg.s));
    cudaFreeAsync(dc, sg.s);
    cudaFreeAsync(df, sg.s);
    CK(cudaStreamSynchronize(sg.s));
    return rc;
}

int nzgpu_ans_encode_host(const uint8_t* symbols, uint64_t n, const uint16_t* freqs, uint32_t chunk_symbols,
                          uint8_t* stream, uint64_t stream_cap, uint64_t* stream_len) {
    if (!freqs || !stream_len || (n && !symbols)) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    if (chunk_symbols == 0) chunk_symbols = kDefaultChunk;
    uint32_t sum = 0;
    for (int i = 0; i < 256; ++i) sum += freqs[i];
    if (sum != kProbScale) return NZGPU_FORMAT_TABLE;
    const uint64_t nchunks = ceil_div(n, chunk_symbols);
    if (n == 0) {
        *stream_len = 4;
        if (stream_cap < 4) return NZGPU_INVALID_ARGUMENT;
        std::memset(stream, 0, 4);
        return NZGPU_OK;
    }
    StreamGuard sg{StreamGuard::Own{}};
    cudaStream_t s = sg.s;
    const uint64_t slot = align_up(2ull * chunk_symbols + 8, 16);
    Carve cv;
    const uint64_t o_sym = cv.take(n + 16), o_scr = cv.take(nchunks * slot + 16), o_plen = cv.take(nchunks * 4);
    const uint64_t o_info = cv.take(nchunks * 16);
    const uint64_t o_tot = cv.take(16), o_enc = cv.take(256 * sizeof(EncSym)), o_fr = cv.take(512);
    const uint64_t o_meta = cv.take(64), o_hdr = cv.take(16);
    uint8_t* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), cv.size, s));
    auto* meta = reinterpret_cast<uint32_t*>(tmp + o_meta);
    CK(cudaMemsetAsync(meta, 0, 64, s));
    CK(cudaMemcpyAsync(tmp + o_sym, symbols, n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(tmp + o_fr, freqs, 512, cudaMemcpyHostToDevice, s));
    build_table_kernel<<<1, 256, 0, s>>>(nullptr, reinterpret_cast<uint16_t*>(tmp + o_fr), nullptr,
                                         reinterpret_cast<EncSym*>(tmp + o_enc), nullptr, meta);
    // The raw coder needs no side index: checkpoints off.
    EncTask t{};
    t.exps = tmp + o_sym;
    t.enc = reinterpret_cast<EncSym*>(tmp + o_enc);
    t.scratch = tmp + o_scr;
    t.plen = reinterpret_cast<uint32_t*>(tmp + o_plen);
    t.err = meta + 4;
    t.chunk_info = reinterpret_cast<uint4*>(tmp + o_info);
    t.hdr = tmp + o_hdr;
    t.total = reinterpret_cast<unsigned long long*>(tmp + o_tot);
    t.n = n;
    t.slot_bytes = slot;
    t.chunk_syms = chunk_symbols;
    CK(launch_encode(false, true, grid_for(nchunks, NZ_ENC_THREADS, 1u << 30), NZ_ENC_THREADS, nullptr, 1, t, s));
    stream_scan_kernel<<<1, 1024, 0, s>>>(nullptr, t);
    CK(cudaGetLastError());
    uint32_t m[8];
    unsigned long long total = 0;
    CK(cudaMemcpyAsync(m, meta, 32, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&total, tmp + o_tot, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int rc = status_from_bits(m[2] | m[4]);
    if (!rc && total > stream_cap) rc = NZGPU_INVALID_ARGUMENT;
    uint8_t* dstream = nullptr;
    if (!rc) {
        CK(cudaMallocAsync(reinterpret_cast<void**>(&dstream), align_up(total, 16) + 32, s));
        CK(cudaMemcpyAsync(dstream, tmp + o_hdr, 4, cudaMemcpyDeviceToDevice, s));
        stream_copy_kernel<<<(unsigned)nchunks, 256, 0, s>>>(tmp + o_scr, slot, reinterpret_cast<uint4*>(tmp + o_info),
                                                             dstream);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(stream, dstream, total, cudaMemcpyDeviceToHost, s));
        CK(cudaFreeAsync(dstream, s));
        *stream_len = total;
    }
    CK(cudaFreeAsync(tmp, s));
    CK(cudaStreamSynchronize(s));
    return rc;
}

int nzgpu_ans_decode_host(const uint8_t* stream, uint64_t stream_len, const uint16_t* freqs, uint8_t* symbols,
                          uint64_t n) {
    if (!stream || !freqs || (n && !symbols)) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    // Reuse the tensor import path with a zero mantissa plane; decode symbols only.
    nzgpu_host_tensor t{};
    t.n = n;
    t.precision = 7;
    t.freqs = freqs;
    t.stream = stream;
    t.stream_len = stream_len;
    std::vector<uint8_t> zeros(n ? n : 1, 0);
    t.mantissas = zeros.data();
    t.mantissa_len = n;
    StreamGuard sg{StreamGuard::Own{}};
    nzgpu_blob_s b;
    int rc = import_into(&b, &t, 0, sg.s);
    if (rc) return rc;
    if (n == 0) return NZGPU_OK;
    uint16_t* dout = nullptr;
    CK(cudaMallocAsync(&dout, n * 2 + 16, sg.s));
    rc = decode_blob(&b, dout, sg.s);
    if (!rc) rc = sync_status(sg.s, b.err, true);
    if (!rc) {
        // Exponent bytes of the bf16 output are the decoded symbols (mantissas were zero).
        std::vector<uint16_t> tmp(n);
        CK(cudaMemcpyAsync(tmp.data(), dout, n * 2, cudaMemcpyDeviceToHost, sg.s));
        CK(cudaStreamSynchronize(sg.s));
        for (uint64_t i = 0; i < n; ++i) symbols[i] = (uint8_t)((tmp[i] >> 7) & 0xFF);
    }
    cudaFreeAsync(dout, sg.s);
    cudaStreamSynchronize(sg.s);
    return rc;
}

int nzgpu_pack_host(const uint8_t* items, uint64_t n, int k, uint8_t* out) {
    if (k != 0 && k != 1 && k != 3 && k != 7) return NZGPU_INVALID_ARGUMENT;  // bitfloat.hpp:126-128
    if (n && (!items || !out)) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    if (n == 0) return NZGPU_OK;
    for (uint64_t i = 0; i < n; ++i)  // bitfloat.hpp:134-136: items must fit k+1 bits
        if (items[i] >> (k + 1)) return NZGPU_INVALID_ARGUMENT;
    const uint64_t nbytes = mant_bytes(n, k);
    StreamGuard sg{StreamGuard::Own{}};
    uint8_t* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n + nbytes + 32, sg.s));
    CK(cudaMemcpyAsync(tmp, items, n, cudaMemcpyHostToDevice, sg.s));
    pack_items_kernel<<<grid_for(nbytes, 256), 256, 0, sg.s>>>(tmp, n, k, tmp + align_up(n, 16), nbytes);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp + align_up(n, 16), nbytes, cudaMemcpyDeviceToHost, sg.s));
    CK(cudaFreeAsync(tmp, sg.s));
    CK(cudaStreamSynchronize(sg.s));
    return NZGPU_OK;
}

int nzgpu_unpack_host(const uint8_t* packed, uint64_t nbytes, int k, uint64_t n, uint8_t* items) {
    if (k != 0 && k != 1 && k != 3 && k != 7) return NZGPU_INVALID_ARGUMENT;  // bitfloat.hpp:147-149
    if (nbytes != mant_bytes(n, k)) return NZGPU_INVALID_ARGUMENT;             // bitfloat.hpp:151-153
    if (int rc = device_ready()) return rc;
    if (n == 0) return NZGPU_OK;
    StreamGuard sg{StreamGuard::Own{}};
    uint8_t* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n + nbytes + 32, sg.s));
    CK(cudaMemcpyAsync(tmp, packed, nbytes, cudaMemcpyHostToDevice, sg.s));
    unpack_items_kernel<<<grid_for(n, 256), 256, 0, sg.s>>>(tmp, n, k, tmp + align_up(nbytes, 16));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(items, tmp + align_up(nbytes, 16), n, cudaMemcpyDeviceToHost, sg.s));
    CK(cudaFreeAsync(tmp, sg.s));
    CK(cudaStreamSynchronize(sg.s));
    return NZGPU_OK;
}

int nzgpu_lossy_roundtrip_host(const uint16_t* values, const uint8_t* scales, uint64_t n, int k, uint16_t* out) {
    if (k != 0 && k != 1 && k != 3) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    if (n == 0) return NZGPU_OK;
    StreamGuard sg{StreamGuard::Own{}};
    uint8_t* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n * 5 + 64, sg.s));
    uint16_t* dv = reinterpret_cast<uint16_t*>(tmp);
    uint16_t* dout = reinterpret_cast<uint16_t*>(tmp + align_up(n * 2, 16));
    uint8_t* ds = tmp + 2 * align_up(n * 2, 16);
    CK(cudaMemcpyAsync(dv, values, n * 2, cudaMemcpyHostToDevice, sg.s));
    CK(cudaMemcpyAsync(ds, scales, n, cudaMemcpyHostToDevice, sg.s));
    lossy_roundtrip_kernel<<<grid_for(n, 256), 256, 0, sg.s>>>(dv, ds, n, k, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout, n * 2, cudaMemcpyDeviceToHost, sg.s));
    CK(cudaFreeAsync(tmp, sg.s));
    CK(cudaStreamSynchronize(sg.s));
    return NZGPU_OK;
}


// --------------------------------------------------------- CRC-32 / NZT --
int nzgpu_crc32(const void* d_data, uint64_t len, void* cuda_stream, uint32_t* crc) {
    if (!crc || (len && !d_data)) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg(cuda_stream);
    uint32_t raw = 0;
    CK(crc_raw_device(static_cast<const uint8_t*>(d_data), len, sg.s, &raw));
    *crc = crc_finalize(raw, len);
    return NZGPU_OK;
}

int nzgpu_crc32_host_sections(const void* const* ptrs, const uint64_t* lens, int count, uint32_t* crc) {
    if (!crc || count < 0 || (count && (!ptrs || !lens))) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg{StreamGuard::Own{}};
    constexpr uint64_t kPiece = 256ull << 20;  // staging bound
    uint64_t cap = 0, total = 0;
    for (int i = 0; i < count; ++i) cap = std::max(cap, std::min(lens[i], kPiece));
    uint8_t* d = nullptr;
    if (cap) CK(cudaMallocAsync(&d, cap, sg.s));
    uint32_t raw_all = 0;
    int rc = NZGPU_OK;
    for (int i = 0; i < count && rc == NZGPU_OK; ++i) {
        if (lens[i] && !ptrs[i]) {
            rc = NZGPU_INVALID_ARGUMENT;
            break;
        }
        for (uint64_t off = 0; off < lens[i]; off += kPiece) {
            const uint64_t m = std::min(kPiece, lens[i] - off);
            cudaError_t e = cudaMemcpyAsync(d, static_cast<const uint8_t*>(ptrs[i]) + off, m,
                                            cudaMemcpyHostToDevice, sg.s);
            uint32_t raw = 0;
            if (e == cudaSuccess) e = crc_raw_device(d, m, sg.s, &raw);
            if (e != cudaSuccess) {
                rc = fail_cuda(e, "crc32 host sections");
                break;
            }
            raw_all = crc_combine_raw(raw_all, raw, m);
            total += m;
        }
    }
    if (d) cudaFreeAsync(d, sg.s);
    cudaStreamSynchronize(sg.s);
    if (rc) return rc;
    *crc = crc_finalize(raw_all, total);
    return NZGPU_OK;
}

int nzgpu_crc32_host(const void* data, uint64_t len, uint32_t* crc) {
    return nzgpu_crc32_host_sections(&data, &len, 1, crc);
}

namespace {
// NZT framing (tensorstore.hpp:289-300): "NZT1" u8 version u8 precision
// u32 block u8 ndim u64*ndim shape | 512 table | u32 scales_len scales |
// u64 exp_len stream | u64 signmant_len mantissas | u32 crc.
uint64_t nzt_size(uint64_t ndim, uint64_t scales, uint64_t stream, uint64_t mant) {
    return 4 + 1 + 1 + 4 + 1 + 8 * ndim + 512 + 4 + scales + 8 + stream + 8 + mant + 4;
}
uint8_t* put_le(uint8_t* p, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) *p++ = (uint8_t)(v >> (8 * i));
    return p;
}
uint64_t get_le(const uint8_t* p, int bytes) {
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}
}  // namespace

int nzgpu_blob_nzt_size(nzgpu_blob b, int ndim, uint64_t* size) {
    if (!b || !size || ndim < 1 || ndim > 8) return NZGPU_INVALID_ARGUMENT;
    *size = nzt_size((uint64_t)ndim, b->scales_len, b->stream_len, b->mant_len);
    return NZGPU_OK;
}

int nzgpu_blob_write_nzt(nzgpu_blob b, const uint64_t* shape, int ndim, uint8_t* out, uint64_t cap,
                         uint64_t* written) {
    if (!b || !shape || !out || ndim < 1 || ndim > 8) return NZGPU_INVALID_ARGUMENT;
    uint64_t n = 1;
    for (int i = 0; i < ndim; ++i) {
        if (shape[i] == 0) return NZGPU_INVALID_ARGUMENT;  // TensorMeta::validate
        n *= shape[i];
    }
    if (n != b->n) return NZGPU_INVALID_ARGUMENT;
    const uint64_t size = nzt_size((uint64_t)ndim, b->scales_len, b->stream_len, b->mant_len);
    if (cap < size) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg{StreamGuard::Own{}};
    CK(cudaDeviceSynchronize());
    // CRC over table | scales | stream | mantissas, each section on the GPU
    const uint8_t* sec[4] = {reinterpret_cast<const uint8_t*>(b->freqs), b->scales, b->stream, b->mant};
    const uint64_t len[4] = {512, b->scales_len, b->stream_len, b->mant_len};
    uint32_t raw_all = 0;
    uint64_t total = 0;
    for (int i = 0; i < 4; ++i) {
        uint32_t raw = 0;
        CK(crc_raw_device(sec[i], len[i], sg.s, &raw));
        raw_all = crc_combine_raw(raw_all, raw, len[i]);
        total += len[i];
    }
    const uint32_t crc = crc_finalize(raw_all, total);
    uint8_t* p = out;
    std::memcpy(p, "NZT1", 4);
    p += 4;
    p = put_le(p, 1, 1);
    p = put_le(p, (uint64_t)b->precision, 1);
    p = put_le(p, b->precision == 7 ? 0 : b->block, 4);
    p = put_le(p, (uint64_t)ndim, 1);
    for (int i = 0; i < ndim; ++i) p = put_le(p, shape[i], 8);
    CK(cudaMemcpy(p, b->freqs, 512, cudaMemcpyDeviceToHost));  // LE u16 table
    p += 512;
    p = put_le(p, b->scales_len, 4);
    if (int rc = d2h_section(p, b->scales, b->scales_len, sg.s)) return rc;
    p += b->scales_len;
    p = put_le(p, b->stream_len, 8);
    if (int rc = d2h_section(p, b->stream, b->stream_len, sg.s)) return rc;
    p += b->stream_len;
    p = put_le(p, b->mant_len, 8);
    if (int rc = d2h_section(p, b->mant, b->mant_len, sg.s)) return rc;
    p += b->mant_len;
    p = put_le(p, crc, 4);
    if (written) *written = (uint64_t)(p - out);
    return NZGPU_OK;
}

int nzgpu_blob_read_nzt(const uint8_t* data, uint64_t len, uint32_t interval, void* cuda_stream, nzgpu_blob* out,
                        uint64_t* shape, int* ndim_out) {
    if (!out || (len && !data)) return NZGPU_INVALID_ARGUMENT;
    *out = nullptr;
    // read_nzt (tensorstore.hpp:403-477): every length is validated against
    // the element count before anything is copied.
    uint64_t pos = 0;
    auto need = [&](uint64_t k) { return len - pos >= k; };
    if (!need(4) || std::memcmp(data, "NZT1", 4) != 0) {
        std::snprintf(g_msg, sizeof(g_msg), "nzt: bad magic");
        return NZGPU_FORMAT_LENGTH;
    }
    pos = 4;
    if (!need(7)) return NZGPU_FORMAT_TRUNCATED;  // "unexpected end of file"
    const uint64_t version = data[pos], precision = data[pos + 1];
    const uint64_t block = get_le(data + pos + 2, 4), ndim = data[pos + 6];
    pos += 7;
    if (version != 1 || !valid_precision((int)precision) || ndim == 0 || ndim > 8) return NZGPU_FORMAT_LENGTH;
    if (!need(8 * ndim)) return NZGPU_FORMAT_TRUNCATED;
    uint64_t n = 1, dims[8];
    for (uint64_t i = 0; i < ndim; ++i) {
        dims[i] = get_le(data + pos + 8 * i, 8);
        if (dims[i] == 0 || dims[i] > (1ull << 40) / n) return NZGPU_FORMAT_LENGTH;
        n *= dims[i];
    }
    pos += 8 * ndim;
    if (precision == 7 ? block != 0 : block == 0) return NZGPU_FORMAT_LENGTH;
    const uint64_t exp_scales = precision == 7 ? 0 : (n + block - 1) / block;
    const uint64_t exp_mant = mant_bytes(n, (int)precision);
    const uint64_t cap = 2 * n + 16 * ((n + kDefaultChunk - 1) / kDefaultChunk) + 64;
    if (!need(512 + 4)) return NZGPU_FORMAT_TRUNCATED;
    const uint8_t* table = data + pos;
    pos += 512;
    const uint64_t scales_len = get_le(data + pos, 4);
    pos += 4;
    if (scales_len != exp_scales) return NZGPU_FORMAT_LENGTH;
    if (!need(scales_len + 8)) return NZGPU_FORMAT_TRUNCATED;
    const uint8_t* scales = data + pos;
    pos += scales_len;
    const uint64_t exp_len = get_le(data + pos, 8);
    pos += 8;
    if (exp_len > cap) return NZGPU_FORMAT_LENGTH;
    if (!need(exp_len + 8)) return NZGPU_FORMAT_TRUNCATED;
    const uint8_t* stream = data + pos;
    pos += exp_len;
    const uint64_t mlen = get_le(data + pos, 8);
    pos += 8;
    if (mlen != exp_mant) return NZGPU_FORMAT_LENGTH;
    if (!need(mlen + 4)) return NZGPU_FORMAT_TRUNCATED;
    const uint8_t* mant = data + pos;
    pos += mlen;
    const uint32_t stored = (uint32_t)get_le(data + pos, 4);
    // CRC over the four payload sections on the GPU (tensorstore.hpp:449-457)
    uint32_t crc = 0;
    {
        const void* ptrs[4] = {table, scales, stream, mant};
        const uint64_t lens[4] = {512, scales_len, exp_len, mlen};
        if (int rc = nzgpu_crc32_host_sections(ptrs, lens, 4, &crc)) return rc;
    }
    if (crc != stored) return NZGPU_CHECKSUM;
    // deserialize_table / deserialize_stream / count check: the import path
    uint16_t freqs[256];
    std::memcpy(freqs, table, 512);  // little-endian host
    nzgpu_host_tensor t{};
    t.n = n;
    t.precision = (int32_t)precision;
    t.block_size = (uint32_t)block;
    t.freqs = freqs;
    t.stream = stream;
    t.stream_len = exp_len;
    t.mantissas = mant;
    t.mantissa_len = mlen;
    t.scales = precision == 7 ? nullptr : scales;
    t.scales_len = scales_len;
    if (int rc = nzgpu_blob_import(&t, interval, cuda_stream, out)) return rc;
    if (shape)
        for (uint64_t i = 0; i < ndim; ++i) shape[i] = dims[i];
    if (ndim_out) *ndim_out = (int)ndim;
    return NZGPU_OK;
}


// ------------------------------------------------------ entropy report ---
int nzgpu_component_histogram(const uint16_t* d_values, uint64_t n, void* cuda_stream, uint64_t* counts) {
    if (!counts || (n && !d_values) || (reinterpret_cast<uintptr_t>(d_values) & 15)) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg(cuda_stream);
    unsigned long long* d = nullptr;
    CK(cudaMallocAsync(&d, 386 * sizeof(unsigned long long), sg.s));
    CK(cudaMemsetAsync(d, 0, 386 * sizeof(unsigned long long), sg.s));
    if (n) component_hist_kernel<<<grid_for(n / 8 + 1, 256), 256, 0, sg.s>>>(d_values, n, d);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(counts, d, 386 * sizeof(uint64_t), cudaMemcpyDeviceToHost, sg.s));
    CK(cudaFreeAsync(d, sg.s));
    CK(cudaStreamSynchronize(sg.s));
    counts[0] = n - counts[1];  // sign 0
    return NZGPU_OK;
}

namespace {
// shannon_entropy (entropy.hpp:41-55): same bins, order and arithmetic.
double shannon(const uint64_t* c, int bins) {
    uint64_t total = 0;
    for (int i = 0; i < bins; ++i) total += c[i];
    double h = 0.0;
    const double n = static_cast<double>(total);
    for (int i = 0; i < bins; ++i) {
        if (c[i] == 0) continue;
        const double p = static_cast<double>(c[i]) / n;
        h -= p * std::log2(p);
    }
    return h < 0.0 ? 0.0 : h;
}
}  // namespace

int nzgpu_shannon_entropy(const uint64_t* counts, uint64_t bins, double* h) {
    if (!h || (bins && !counts)) return NZGPU_INVALID_ARGUMENT;
    uint64_t total = 0;
    for (uint64_t i = 0; i < bins; ++i) total += counts[i];
    if (bins == 0 || total == 0) return NZGPU_INVALID_ARGUMENT;  // "shannon_entropy: empty histogram"
    if (bins > 0x7FFFFFFFull) return NZGPU_INVALID_ARGUMENT;
    *h = shannon(counts, (int)bins);
    return NZGPU_OK;
}

int nzgpu_entropy_from_histogram(const uint64_t* counts, double* out5) {
    if (!counts || !out5) return NZGPU_INVALID_ARGUMENT;
    if (counts[0] + counts[1] == 0) return NZGPU_INVALID_ARGUMENT;  // "entropy report: empty histogram"
    // report_from_histogram (entropy.hpp:69-81)
    const double hs = shannon(counts, 2), he = shannon(counts + 2, 256), hm = shannon(counts + 258, 128);
    const double cap = 999.0, h = hs + he + hm;
    out5[0] = hs;
    out5[1] = he;
    out5[2] = hm;
    out5[3] = (h <= 16.0 / cap) ? cap : 16.0 / h;
    out5[4] = 16.0 / (1.0 + he + 7.0);
    return NZGPU_OK;
}

int nzgpu_entropy_report(const uint16_t* d_values, uint64_t n, void* cuda_stream, double* out5) {
    if (n == 0) return NZGPU_INVALID_ARGUMENT;  // analyze_tensor: empty input
    uint64_t counts[386];
    if (int rc = nzgpu_component_histogram(d_values, n, cuda_stream, counts)) return rc;
    return nzgpu_entropy_from_histogram(counts, out5);
}

int nzgpu_component_histogram_host(const uint16_t* values, uint64_t n, uint64_t* counts) {
    if (!counts || (n && !values)) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg{StreamGuard::Own{}};
    uint16_t* d = nullptr;
    CK(cudaMallocAsync(&d, n * 2 + 16, sg.s));
    if (n) CK(cudaMemcpyAsync(d, values, n * 2, cudaMemcpyHostToDevice, sg.s));
    const int rc = nzgpu_component_histogram(d, n, sg.s, counts);
    cudaFreeAsync(d, sg.s);
    cudaStreamSynchronize(sg.s);
    return rc;
}

int nzgpu_entropy_report_host(const uint16_t* values, uint64_t n, double* out5) {
    if (n == 0 || !values) return NZGPU_INVALID_ARGUMENT;
    if (int rc = device_ready()) return rc;
    StreamGuard sg{StreamGuard::Own{}};
    uint16_t* d = nullptr;
    CK(cudaMallocAsync(&d, n * 2 + 16, sg.s));
    CK(cudaMemcpyAsync(d, values, n * 2, cudaMemcpyHostToDevice, sg.s));
    const int rc = nzgpu_entropy_report(d, n, sg.s, out5);
    cudaFreeAsync(d, sg.s);
    cudaStreamSynchronize(sg.s);
    return rc;
}

}  // extern "C"
