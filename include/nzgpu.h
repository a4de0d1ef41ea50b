/*
 * nzgpu.h -- C ABI of the B200-native NeuZip bf16 weight codec.
 *
 * The reference (arxiv 2410.20650, /root/reference/proj/include/neuzip/) is a
 * header-only C++20 library with no FFI; its public surface is the C++ API in
 * tensorstore.hpp / ans.hpp / bitfloat.hpp.  This header is the thin C layer
 * that the drop-in C++ headers (include/neuzip/ *.hpp) and any foreign binding
 * (ctypes, cgo, JNI -- see INTEGRATION.md) call.  Plain pointers and sizes
 * only; no exceptions cross it; every function returns an nzgpu_status.
 *
 * Byte formats are the reference's, unchanged:
 *   table      256 x u16 little-endian, sum 4096          (ans.hpp:111-130)
 *   stream     [u32 nchunks]([u32 nsym][u32 len][payload])* (ans.hpp:304-347)
 *   mantissas  lossless: n bytes (s<<7|m); lossy: (k+1)-bit MSB-first items
 *              (bitfloat.hpp:122-164)
 *   scales     lossy: ceil(n/B) bytes                      (tensorstore.hpp:72-81)
 * so footprint() and the compression ratio are identical to the reference's.
 *
 * A blob additionally carries a checkpoint side index (decoder state and byte
 * position every K symbols) that lets the GPU decode one reference chunk
 * with many threads.  It is NOT part of the reference format and not counted
 * in the ratio; it can be exported/imported as an opaque byte string, and
 * is rebuilt on the GPU when absent (streams produced by the CPU reference).
 */
#ifndef NZGPU_H
#define NZGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the C++ layer maps them 1:1 onto the reference's exception
 * types (errors.hpp:9-32). */
typedef enum nzgpu_status {
    NZGPU_OK = 0,
    NZGPU_INVALID_ARGUMENT = 1, /* std::invalid_argument                          */
    NZGPU_FORMAT_TRUNCATED = 2, /* FormatError "truncated" (ans.hpp:232,246,323)  */
    NZGPU_FORMAT_DESYNC = 3,    /* FormatError "desynchronization" (ans.hpp:253)  */
    NZGPU_FORMAT_LENGTH = 4,    /* FormatError length/count mismatch (tensorstore.hpp:116,219,226; ans.hpp:344) */
    NZGPU_NONFINITE = 5,        /* NonFiniteError (tensorstore.hpp:155)           */
    NZGPU_FORMAT_TABLE = 6,     /* FormatError "does not sum to 4096" (ans.hpp:100) */
    NZGPU_CUDA_ERROR = 7,       /* CUDA runtime failure                          */
    NZGPU_OUT_OF_MEMORY = 8,
    NZGPU_NO_DEVICE = 9,        /* no CUDA device: the library never falls back to the CPU */
    NZGPU_CHECKSUM = 10         /* ChecksumError "nzt: checksum failure" (tensorstore.hpp:462) */
} nzgpu_status;

#define NZGPU_LOSSLESS 7            /* kLosslessPrecision, tensorstore.hpp:36 */
#define NZGPU_DEFAULT_BLOCK 512     /* kDefaultBlockSize, tensorstore.hpp:35  */
#define NZGPU_DEFAULT_CHUNK 65536   /* ans::kChunkSymbols, ans.hpp:33         */
#define NZGPU_DEFAULT_INTERVAL 64   /* checkpoint stride K (symbols)          */

typedef struct nzgpu_blob_s* nzgpu_blob; /* device-resident compressed tensor */
typedef struct nzgpu_plan_s* nzgpu_plan; /* grouped decode of several blobs   */

/* Host-side view of one compressed tensor in the reference's formats
 * (LosslessBlob / LossyBlob, tensorstore.hpp:64-81, with the exponent stream
 * serialized by serialize_stream). */
typedef struct nzgpu_host_tensor {
    uint64_t n;               /* element count (TensorMeta::element_count)      */
    int32_t precision;        /* 7 = lossless, 0/1/3 = lossy k                  */
    uint32_t block_size;      /* lossy block size B (ignored when lossless)     */
    const uint16_t* freqs;    /* 256 table frequencies                          */
    const uint8_t* stream;    /* serialized exponent stream                     */
    uint64_t stream_len;
    const uint8_t* mantissas; /* sign+mantissa plane                            */
    uint64_t mantissa_len;
    const uint8_t* scales;    /* lossy block scales (NULL when lossless)        */
    uint64_t scales_len;
    const void* index;        /* optional checkpoint index (nzgpu_blob_export)  */
    uint64_t index_len;       /* 0 = rebuild on the GPU                         */
} nzgpu_host_tensor;

/* Sizes and device pointers of a blob's sections. */
typedef struct nzgpu_blob_info {
    uint64_t n;
    int32_t precision;
    uint32_t block_size;
    uint32_t chunk_symbols;   /* S */
    uint32_t interval;        /* K */
    uint64_t num_chunks;
    uint64_t stream_len;      /* footprint().exponent_bytes                     */
    uint64_t mantissa_len;    /* footprint().mantissa_bytes                     */
    uint64_t scales_len;      /* footprint().scale_bytes                        */
    uint64_t index_len;       /* bytes of the exported side index               */
    uint64_t payload_bytes;   /* stream + mantissas + scales + 512-byte table:
                                 the compressed bytes a decode must read        */
    const uint8_t* d_stream;
    const uint16_t* d_freqs;
    const uint8_t* d_mantissas;
    const uint8_t* d_scales;
    uint32_t flags;           /* bit0: single-symbol table; bit1: irregular framing (sequential
                                 decode); bit2: table codes exponent 255; bit3: a lossy scale
                                 byte >= 128 (bits 2-3 select the float lossy merge) */
    uint32_t max_window;      /* largest per-tile payload window (bytes)        */
} nzgpu_blob_info;

/* ---- library ----------------------------------------------------------- */
const char* nzgpu_status_string(int status);
int nzgpu_version(void);                       /* 10000 * major + 100 * minor */
/* Returns NZGPU_OK when a CUDA device is usable; NZGPU_NO_DEVICE otherwise. */
int nzgpu_device_check(int* device_count);
/* Last CUDA error text recorded by the library (thread-local). */
const char* nzgpu_last_error_message(void);
/* Decode schedule for plans/decompress created afterwards: 0 = persistent
 * warp-pipelined kernel (default), 1 = one tile per CTA.  Both are
 * bit-identical; this exists for A/B measurement. */
int nzgpu_set_decode_kernel(int which);

/* ---- device tier: device pointers, stream-ordered ---------------------- */
/* Compress n bf16 values resident on the device (compress_lossless,
 * tensorstore.hpp:87-106, precision 7; compress_lossy, :141-208, k in
 * {0,1,3}).  chunk_symbols S (0 = 65536) and interval K (0 = 64; 64 or 128,
 * dividing S: the side index holds 16-bit offsets within a 32-sub-range
 * unit, <= 31 (1.5 K + 2) bytes).  Synchronises `stream` once (to size the
 * exact stream allocation).  d_values must be 16-byte aligned. */
int nzgpu_compress(const uint16_t* d_values, uint64_t n, int precision, uint32_t block_size,
                   uint32_t chunk_symbols, uint32_t interval, void* cuda_stream, nzgpu_blob* out);
/* Compress `count` device tensors with one shared parameter set: out[i] is
 * byte-identical to nzgpu_compress(d_values[i], n[i], ...).  One encode
 * launch covers the chunks of every tensor (the per-chunk rANS chains are
 * serial, so a whole layer or model must share a launch to fill the GPU), the
 * stream is synchronised once for the batch (plus once for the decode window
 * sizes) instead of twice per tensor, and the blobs of the batch share two
 * device allocations (released with the last blob).  d_workspace (256-byte
 * aligned, >= nzgpu_compress_batch_workspace_size bytes, about 3 bytes per
 * element) holds the temporaries; NULL = stream-ordered allocation.  On
 * error every out[i] is NULL. */
int nzgpu_compress_batch_workspace_size(const uint64_t* n, int count, int precision, uint32_t chunk_symbols,
                                        uint64_t* bytes);
int nzgpu_compress_batch(const uint16_t* const* d_values, const uint64_t* n, int count, int precision,
                         uint32_t block_size, uint32_t chunk_symbols, uint32_t interval, void* d_workspace,
                         uint64_t workspace_bytes, void* cuda_stream, nzgpu_blob* out);
/* Decompress into d_out (16-byte aligned, n bf16), asynchronously on
 * `stream`; errors are sticky in the blob until nzgpu_blob_status. */
int nzgpu_decompress(nzgpu_blob blob, uint16_t* d_out, void* cuda_stream);
/* Synchronise `stream` and return (then clear) the blob's decode status. */
int nzgpu_blob_status(nzgpu_blob blob, void* cuda_stream);
int nzgpu_blob_info_get(nzgpu_blob blob, nzgpu_blob_info* info);
int nzgpu_blob_free(nzgpu_blob blob);

/* Copy a blob's sections to host buffers (any may be NULL).  freqs: 256 u16;
 * stream: info.stream_len; mantissas: info.mantissa_len; scales:
 * info.scales_len; index: info.index_len bytes. */
int nzgpu_blob_export(nzgpu_blob blob, uint16_t* freqs, uint8_t* stream, uint8_t* mantissas,
                      uint8_t* scales, void* index);
/* Chunk table of a blob: payload bytes and symbol count of each of its
 * info.num_chunks chunks (AnsChunk::payload.size(), ::symbol_count). */
int nzgpu_blob_chunks(nzgpu_blob blob, uint32_t* lens, uint32_t* nsyms);
/* nzgpu_blob_export with the exponent stream delivered as chunk payloads
 * (chunk_payloads[c] receives lens[c] bytes of nzgpu_blob_chunks) -- the
 * drop-in's AnsStream form, without a serialized copy.  Sections come back
 * D2H through pinned staging, copied out by host worker threads. */
int nzgpu_blob_export_chunks(nzgpu_blob blob, uint16_t* freqs, uint8_t* const* chunk_payloads, uint8_t* mantissas,
                             uint8_t* scales, void* index);
/* Upload a host tensor (reference formats) into a new device blob,
 * validating framing and table (deserialize_table / deserialize_stream,
 * ans.hpp:120-130, :318-347) and building the checkpoint index on the GPU
 * when t->index is absent (full sequential validation, ans.hpp:229-256).
 * interval 0 = auto (64). */
int nzgpu_blob_import(const nzgpu_host_tensor* t, uint32_t interval, void* cuda_stream, nzgpu_blob* out);

/* Grouped decode: one kernel launch decodes all blobs (e.g. one transformer
 * layer) into their outputs.  Blobs must share precision and interval. */
int nzgpu_plan_create(const nzgpu_blob* blobs, uint16_t* const* d_outs, int count, nzgpu_plan* out);
int nzgpu_plan_launch(nzgpu_plan plan, void* cuda_stream);
int nzgpu_plan_status(nzgpu_plan plan, void* cuda_stream);
int nzgpu_plan_free(nzgpu_plan plan);
/* Number of kernel launches nzgpu_plan_launch / nzgpu_decompress issue. */
int nzgpu_plan_launch_count(nzgpu_plan plan);
/* Decode kernel nzgpu_plan_launch uses now: 0 persistent, 1 tiles, -1 none
 * (empty plan). */
int nzgpu_plan_kernel(nzgpu_plan plan);
/* Cap the persistent decode at `max_ctas` CTAs (one per SM; 0 = all
 * resident), leaving the other SMs to concurrent work on another stream --
 * the layer-wise consumer decodes layer l+1 beside layer l's GEMM.  Every CTA
 * of the launch (small tensors included) counts against the cap.  The call
 * synchronises the device first: the schedule it rewrites is read by any
 * launch of this plan still queued. */
int nzgpu_plan_set_max_ctas(nzgpu_plan plan, uint32_t max_ctas);

/* ---- host tier: the reference-facing calls (host buffers, synchronous) --- */
/* Compress host values; returns a device blob (export its sections with
 * nzgpu_blob_export[_chunks]).  Equivalent to H2D + nzgpu_compress; the
 * values go H2D in slices through pinned staging (host worker threads copy
 * slice k+1 while slice k is in flight). */
int nzgpu_compress_host(const uint16_t* values, uint64_t n, int precision, uint32_t block_size,
                        uint32_t chunk_symbols, uint32_t interval, nzgpu_blob* out);
/* Decompress a host tensor into host memory: H2D of the compressed sections,
 * GPU decode, D2H of the bf16 result.  Staging buffers are cached by the
 * library; pinned host memory gives full PCIe bandwidth. */
int nzgpu_decompress_host(const nzgpu_host_tensor* t, uint16_t* out);
/* One chunk of an AnsStream as the reference holds it (AnsChunk,
 * ans.hpp:159-168: its own payload vector), so callers need not serialize
 * the stream first. */
typedef struct nzgpu_chunk_view {
    const uint8_t* payload;
    uint32_t len;             /* payload bytes (renormalisation bytes + LE32 state) */
    uint32_t nsym;            /* AnsChunk::symbol_count                          */
} nzgpu_chunk_view;

/* A host tensor with the exponent stream as chunk views (the drop-in
 * LosslessBlob / LossyBlob layout); other fields as nzgpu_host_tensor. */
typedef struct nzgpu_host_sections {
    uint64_t n;
    int32_t precision;
    uint32_t block_size;
    const uint16_t* freqs;
    const nzgpu_chunk_view* chunks;
    uint64_t nchunks;
    const uint8_t* mantissas;
    uint64_t mantissa_len;
    const uint8_t* scales;
    uint64_t scales_len;
    const void* index;
    uint64_t index_len;
} nzgpu_host_sections;

/* Decompress a host tensor given as sections into host memory `out`
 * (pageable or pinned, n bf16): the chunk payloads, planes and index are
 * gathered straight into pinned staging by host worker threads, sent H2D
 * and decoded; the bf16 result comes back D2H in slices that worker threads
 * copy into `out` while the next slice is in flight.  Staging is cached per
 * calling thread (nzgpu_host_release frees it).  Tensors without a usable
 * side index or with irregular framing take the general (validating) path.
 * Same results and errors as nzgpu_decompress_host. */
int nzgpu_decompress_host_sections(const nzgpu_host_sections* t, uint16_t* out);

/* Decode a device blob into host memory (GPU decode on a private stream,
 * then D2H; pinned or pageable `out`, n bf16).  Synchronous. */
int nzgpu_blob_decompress_host(nzgpu_blob blob, uint16_t* out);
/* Same for `count` tensors, pipelined across two CUDA streams (H2D of tensor
 * i+1 overlaps decode of i and D2H of i-1). */
int nzgpu_decompress_host_batch(const nzgpu_host_tensor* ts, int count, uint16_t* const* outs);
/* The host tier keeps per-thread device staging (8 slots, each sized for the
 * largest tensor it has staged) between calls; this frees the calling
 * thread's staging after its queued work completes. */
int nzgpu_host_release(void);

/* Blob sections live in a library-owned stream-ordered memory pool per
 * device that keeps freed memory for the next blob (no cudaMalloc per
 * compress).  This returns the current device's unused pool memory to the
 * driver. */
int nzgpu_trim_device_pool(void);

/* ---- building blocks (device pointers, stream-ordered) ------------------ */
/* K1: exponent plane, sign/mantissa plane and 256-bin u64 histogram
 * (tensorstore.hpp:93-102).  Any output may be NULL; counts accumulate. */
int nzgpu_split(const uint16_t* d_values, uint64_t n, uint8_t* d_exponents, uint8_t* d_signmant,
                uint64_t* d_counts, void* cuda_stream);
/* K2: FrequencyTable::from_counts (ans.hpp:52-93) on the device. */
int nzgpu_build_table(const uint64_t* d_counts, uint16_t* d_freqs, void* cuda_stream);
/* Synchronous host convenience for the same (no CPU fallback: runs K2). */
int nzgpu_build_table_host(const uint64_t* counts, uint16_t* freqs);
/* Raw coder on host buffers (ans_encode / ans_decode, ans.hpp:258-293):
 * symbols -> serialized stream, and back, with an explicit table. */
int nzgpu_ans_encode_host(const uint8_t* symbols, uint64_t n, const uint16_t* freqs, uint32_t chunk_symbols,
                          uint8_t* stream, uint64_t stream_cap, uint64_t* stream_len);
int nzgpu_ans_decode_host(const uint8_t* stream, uint64_t stream_len, const uint16_t* freqs, uint8_t* symbols,
                          uint64_t n);
/* Lossy elementwise transform on the device (tensorstore.hpp:165-199 and
 * :229-236) for every (value, scale) pair: out[i] = round trip of v[i] under
 * scale byte s[i]; the exhaustive parity check of the lossy arithmetic. */
int nzgpu_lossy_roundtrip_host(const uint16_t* values, const uint8_t* scales, uint64_t n, int k, uint16_t* out);
/* pack_signed_mantissas / unpack_signed_mantissas (bitfloat.hpp:124-164) on
 * the device: items are (sign << k) | mantissa, one byte each, k in
 * {0,1,3,7}; packed holds ceil(n(k+1)/8) MSB-first bytes. */
int nzgpu_pack_host(const uint8_t* items, uint64_t n, int k, uint8_t* packed);
int nzgpu_unpack_host(const uint8_t* packed, uint64_t nbytes, int k, uint64_t n, uint8_t* items);

/* ---- CRC-32 and the NZT container (tensorstore.hpp:289-477, crc32.hpp) -- */
/* CRC-32 (IEEE, reflected 0xEDB88320, init/xorout 0xFFFFFFFF: crc32.hpp:26-43)
 * of a device byte range, computed on the GPU (block CRCs joined by GF(2)
 * multiplication).  Synchronises `cuda_stream`. */
int nzgpu_crc32(const void* d_data, uint64_t len, void* cuda_stream, uint32_t* crc);
/* Same over host buffers (staged through the GPU); `count` sections are
 * checksummed as one concatenated byte string. */
int nzgpu_crc32_host(const void* data, uint64_t len, uint32_t* crc);
int nzgpu_crc32_host_sections(const void* const* ptrs, const uint64_t* lens, int count, uint32_t* crc);
/* Size in bytes of the NZT file of a blob with `ndim` dimensions. */
int nzgpu_blob_nzt_size(nzgpu_blob blob, int ndim, uint64_t* size);
/* write_nzt (tensorstore.hpp:352-376) of a device blob into a host buffer:
 * sections copied D2H, CRC computed on the GPU.  shape must multiply to n. */
int nzgpu_blob_write_nzt(nzgpu_blob blob, const uint64_t* shape, int ndim, uint8_t* out, uint64_t cap,
                         uint64_t* written);
/* read_nzt (tensorstore.hpp:403-477) from a host buffer into a new device
 * blob: framing and lengths validated first, CRC checked on the GPU
 * (NZGPU_CHECKSUM), then table/stream validated and the checkpoint index
 * built as nzgpu_blob_import does.  shape: 8 u64 (may be NULL). */
int nzgpu_blob_read_nzt(const uint8_t* data, uint64_t len, uint32_t interval, void* cuda_stream, nzgpu_blob* out,
                        uint64_t* shape, int* ndim);

/* ---- entropy report (entropy.hpp:17-94) ---------------------------------- */
/* ComponentHistogram of a device bf16 tensor (16-byte aligned): counts[386] =
 * sign[2] | exponent[256] | mantissa[128] (entropy.hpp:17-39). */
int nzgpu_component_histogram(const uint16_t* d_values, uint64_t n, void* cuda_stream, uint64_t* counts);
int nzgpu_component_histogram_host(const uint16_t* values, uint64_t n, uint64_t* counts);
/* shannon_entropy (entropy.hpp:41-55): -sum p log2 p over the nonzero bins,
 * summed in bin order (bit-identical to the reference); INVALID_ARGUMENT for
 * an empty histogram. */
int nzgpu_shannon_entropy(const uint64_t* counts, uint64_t bins, double* h);
/* report_from_histogram (entropy.hpp:69-81): out5 = h_sign, h_exp, h_mant,
 * ideal_ratio, exponent_only_ratio. */
int nzgpu_entropy_from_histogram(const uint64_t* counts, double* out5);
/* analyze_tensor (entropy.hpp:89-94) of a device / host tensor. */
int nzgpu_entropy_report(const uint16_t* d_values, uint64_t n, void* cuda_stream, double* out5);
int nzgpu_entropy_report_host(const uint16_t* values, uint64_t n, double* out5);

#ifdef __cplusplus
}
#endif

#endif /* NZGPU_H */
