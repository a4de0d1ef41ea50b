#pragma once
// Drop-in for the codec half of /root/reference/proj/include/neuzip/
// tensorstore.hpp (tensorstore.hpp:33-287): TensorMeta, the lossless and
// lossy blobs, compress_* / decompress_* and footprint(), with the same
// names, signatures, byte formats and exceptions.  compress_* and
// decompress_* run on the B200 (nzgpu_compress_host / nzgpu_decompress_host).
//
// One addition: each blob carries `gpu_index`, the checkpoint side index the
// GPU decoder uses to split a 65,536-symbol chunk across many threads.  It is
// not part of the reference format, not written by serialization and not
// counted by footprint(); blobs without it (e.g. built from reference
// streams) decode too -- the GPU rebuilds it with a full sequential
// validation first.

#include <algorithm>
#include <array>
#include <cstdint>
#include <exception>
#include <istream>
#include <thread>
#include <ostream>
#include <span>
#include <string>
#include <system_error>
#include <variant>
#include <vector>

#include "neuzip/ans.hpp"
#include "neuzip/bitfloat.hpp"
#include "neuzip/crc32.hpp"
#include "neuzip/errors.hpp"
#include "neuzip/parallel.hpp"

#if defined(__linux__)
#include <sys/mman.h>
#endif

namespace neuzip {

#if defined(__linux__)
#ifdef MADV_POPULATE_WRITE
constexpr int kMadvPopulateWrite = MADV_POPULATE_WRITE;
#else
constexpr int kMadvPopulateWrite = 23;  // Linux 5.14+; older kernels return EINVAL
#endif
#endif

constexpr std::uint32_t kDefaultBlockSize = 512;  // tensorstore.hpp:35
constexpr int kLosslessPrecision = 7;             // tensorstore.hpp:36

struct TensorMeta {  // tensorstore.hpp:38-56
    std::vector<std::uint64_t> shape;

    std::uint64_t element_count() const {
        if (shape.empty()) return 0;
        std::uint64_t n = 1;
        for (std::uint64_t d : shape) n *= d;
        return n;
    }
    void validate() const {
        if (shape.empty()) throw std::invalid_argument("tensor shape is empty");
        if (shape.size() > 8) throw std::invalid_argument("tensor rank exceeds 8");
        for (std::uint64_t d : shape)
            if (d == 0) throw std::invalid_argument("tensor dimension is zero");
    }
    friend bool operator==(const TensorMeta&, const TensorMeta&) = default;
};

struct Tensor {  // tensorstore.hpp:58-62
    TensorMeta meta;
    std::vector<Bf16> values;
};

struct LosslessBlob {  // tensorstore.hpp:64-70
    TensorMeta meta;
    AnsStream exp_stream;
    std::vector<std::uint8_t> signmant;
    std::vector<std::uint8_t> gpu_index{};  // side index (not part of the format)

    const FrequencyTable& table() const { return exp_stream.table; }
};

struct LossyBlob {  // tensorstore.hpp:72-81
    TensorMeta meta;
    int precision = 3;
    std::uint32_t block_size = kDefaultBlockSize;
    std::vector<std::uint8_t> scales;
    AnsStream exp_stream;
    std::vector<std::uint8_t> signmant;
    std::vector<std::uint8_t> gpu_index{};  // side index (not part of the format)

    const FrequencyTable& table() const { return exp_stream.table; }
};

using Blob = std::variant<LosslessBlob, LossyBlob>;

namespace detail {

// RAII owner of a device blob.
struct DeviceBlob {
    nzgpu_blob h = nullptr;
    ~DeviceBlob() {
        if (h) nzgpu_blob_free(h);
    }
};

struct Sections {
    std::vector<std::uint16_t> freqs = std::vector<std::uint16_t>(256);
    std::vector<std::uint8_t> stream, mantissas, scales, index;
};

inline Sections export_blob(nzgpu_blob h) {
    nzgpu_blob_info info{};
    check(nzgpu_blob_info_get(h, &info), "blob info");
    Sections s;
    s.stream.resize(info.stream_len);
    s.mantissas.resize(info.mantissa_len);
    s.scales.resize(info.scales_len);
    s.index.resize(info.index_len);
    check(nzgpu_blob_export(h, s.freqs.data(), s.stream.data(), s.mantissas.data(), s.scales.data(),
                            s.index.empty() ? nullptr : s.index.data()),
          "blob export");
    return s;
}

// Fault the pages of a fresh output buffer in before it is value-initialised:
// as transparent huge pages where the kernel allows it (MADV_HUGEPAGE), and
// populated by several threads (MADV_POPULATE_WRITE) instead of one thread
// taking a 4 KiB fault per page inside the vector's zero-fill.  Best effort:
// any refusal leaves the ordinary fault path.
inline void prefault_output(void* p, std::size_t bytes) {
#if defined(__linux__)
    constexpr std::size_t kHuge = 2u << 20;
    if (bytes < 16 * kHuge) return;
    const auto lo = reinterpret_cast<std::uintptr_t>(p), hi = lo + bytes;
    const std::uintptr_t h0 = (lo + kHuge - 1) & ~(kHuge - 1), h1 = hi & ~(kHuge - 1);
    if (h1 > h0) ::madvise(reinterpret_cast<void*>(h0), h1 - h0, MADV_HUGEPAGE);
    const std::uintptr_t p0 = lo & ~std::uintptr_t(4095);
    const unsigned workers = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const std::size_t step = (((hi - p0) + workers - 1) / workers + kHuge - 1) & ~(kHuge - 1);
    std::vector<std::thread> ts;
    for (unsigned w = 0; w < workers && p0 + w * step < hi; ++w) {
        const std::uintptr_t a = p0 + w * step, b = std::min<std::uintptr_t>(hi, a + step);
        auto populate = [a, b] { ::madvise(reinterpret_cast<void*>(a), b - a, kMadvPopulateWrite); };
        try {
            ts.emplace_back(populate);
        } catch (const std::system_error&) {  // no thread to spare: populate this range here
            populate();
        }
    }
    for (std::thread& t : ts) t.join();
#else
    (void)p;
    (void)bytes;
#endif
}

// A freshly compressed blob's sections as the drop-in types: the exponent
// stream straight into AnsChunk payload vectors (allocated by several
// threads; no serialized copy, no deserialize_stream pass) and the planes
// through the library's pinned staging (nzgpu_blob_export_chunks).
struct Exported {
    AnsStream stream;
    std::vector<std::uint8_t> mantissas, scales, index;
};

// A fresh, value-initialised byte vector whose pages were faulted in first.
inline std::vector<std::uint8_t> fresh_plane(std::size_t bytes) {
    std::vector<std::uint8_t> v;
    v.reserve(bytes);
    prefault_output(v.data(), bytes);
    v.resize(bytes);
    return v;
}

// fresh_plane(bytes) built on a helper thread while the caller works; get()
// joins and hands it over (an allocation failure is rethrown there).
class PlaneAsync {
public:
    explicit PlaneAsync(std::size_t bytes) : bytes_(bytes) {
        try {
            t_ = std::thread([this] { run(); });
        } catch (const std::system_error&) {
            run();  // no thread to spare: build it now
        }
    }
    ~PlaneAsync() {
        if (t_.joinable()) t_.join();
    }
    std::vector<std::uint8_t> get() {
        if (t_.joinable()) t_.join();
        if (err_) std::rethrow_exception(err_);
        return std::move(v_);
    }

private:
    void run() {
        try {
            v_ = fresh_plane(bytes_);
        } catch (...) {
            err_ = std::current_exception();
        }
    }
    std::size_t bytes_;
    std::vector<std::uint8_t> v_;
    std::exception_ptr err_;
    std::thread t_;
};

// `mantissas` may come prepared (already info.mantissa_len bytes): the
// compress calls build it on a helper thread while the GPU compresses.
inline Exported export_chunked(nzgpu_blob h, std::vector<std::uint8_t> mantissas = {}) {
    nzgpu_blob_info info{};
    check(nzgpu_blob_info_get(h, &info), "blob info");
    std::vector<std::uint32_t> lens(info.num_chunks), nsyms(info.num_chunks);
    check(nzgpu_blob_chunks(h, lens.data(), nsyms.data()), "blob chunks");
    Exported e;
    e.stream.chunks.resize(info.num_chunks);
    std::vector<std::uint8_t*> ptrs(info.num_chunks);
    parallel_for(info.num_chunks, [&](std::size_t c) {
        e.stream.chunks[c].symbol_count = nsyms[c];
        e.stream.chunks[c].payload.resize(lens[c]);
        ptrs[c] = e.stream.chunks[c].payload.data();
    });
    e.mantissas = mantissas.size() == info.mantissa_len ? std::move(mantissas) : fresh_plane(info.mantissa_len);
    e.scales.resize(info.scales_len);
    e.index.resize(info.index_len);
    std::array<std::uint16_t, 256> freqs{};
    check(nzgpu_blob_export_chunks(h, freqs.data(), ptrs.data(), e.mantissas.data(), e.scales.data(),
                                   e.index.empty() ? nullptr : e.index.data()),
          "blob export");
    e.stream.table = FrequencyTable::from_frequencies(freqs);
    return e;
}

inline FrequencyTable table_from(const std::vector<std::uint16_t>& f) {
    std::array<std::uint16_t, 256> a{};
    std::copy(f.begin(), f.end(), a.begin());
    return FrequencyTable::from_frequencies(a);
}

// Decode through nzgpu_decompress_host_sections: the AnsStream's chunk
// payloads are gathered straight into pinned staging (no serialize_stream
// copy), and the bf16 result is copied out of a pinned D2H ring by worker
// threads into `out` (n values).
inline void gpu_decompress_into(const TensorMeta& meta, const AnsStream& stream, const std::vector<std::uint8_t>& mant,
                                int precision, std::uint32_t block, const std::vector<std::uint8_t>* scales,
                                const std::vector<std::uint8_t>& index, Bf16* out) {
    std::vector<nzgpu_chunk_view> views(stream.chunks.size());
    for (std::size_t c = 0; c < views.size(); ++c) {
        const AnsChunk& ch = stream.chunks[c];
        if (ch.payload.size() > 0xFFFFFFFFull) throw FormatError("ans stream: chunk payload too large");
        views[c] = nzgpu_chunk_view{ch.payload.data(), static_cast<std::uint32_t>(ch.payload.size()), ch.symbol_count};
    }
    nzgpu_host_sections t{};
    t.n = meta.element_count();
    t.precision = precision;
    t.block_size = block;
    t.freqs = stream.table.frequencies().data();
    t.chunks = views.data();
    t.nchunks = views.size();
    t.mantissas = mant.data();
    t.mantissa_len = mant.size();
    if (scales) {
        t.scales = scales->data();
        t.scales_len = scales->size();
    }
    t.index = index.empty() ? nullptr : index.data();
    t.index_len = index.size();
    check(nzgpu_decompress_host_sections(&t, reinterpret_cast<std::uint16_t*>(out)), "decompress");
}

inline std::vector<Bf16> gpu_decompress(const TensorMeta& meta, const AnsStream& stream,
                                        const std::vector<std::uint8_t>& mant, int precision, std::uint32_t block,
                                        const std::vector<std::uint8_t>* scales,
                                        const std::vector<std::uint8_t>& index) {
    // A fresh vector is value-initialised before the decode writes it; its
    // pages are faulted in first, in parallel (prefault_output).  The
    // *_into overloads reuse memory and skip both.
    std::vector<Bf16> out;
    out.reserve(meta.element_count());
    prefault_output(out.data(), meta.element_count() * sizeof(Bf16));
    out.resize(meta.element_count());
    gpu_decompress_into(meta, stream, mant, precision, block, scales, index, out.data());
    return out;
}

}  // namespace detail

// tensorstore.hpp:87-106
inline LosslessBlob compress_lossless(std::span<const Bf16> values, TensorMeta meta) {
    meta.validate();
    if (meta.element_count() != values.size()) throw std::invalid_argument("compress: shape does not match value count");
    detail::DeviceBlob b;
    detail::PlaneAsync mant(values.size());  // the n-byte plane, faulted in beside the GPU work
    const int rc = nzgpu_compress_host(reinterpret_cast<const std::uint16_t*>(values.data()), values.size(),
                                       kLosslessPrecision, 0, 0, 0, &b.h);
    std::vector<std::uint8_t> plane = mant.get();
    detail::check(rc, "compress_lossless");
    detail::Exported e = detail::export_chunked(b.h, std::move(plane));
    return LosslessBlob{std::move(meta), std::move(e.stream), std::move(e.mantissas), std::move(e.index)};
}

// tensorstore.hpp:108-110
inline LosslessBlob compress_lossless(std::span<const Bf16> values) {
    return compress_lossless(values, TensorMeta{{values.size()}});
}

// tensorstore.hpp:112-125
inline std::vector<Bf16> decompress_lossless(const LosslessBlob& blob) {
    return detail::gpu_decompress(blob.meta, blob.exp_stream, blob.signmant, kLosslessPrecision, 0, nullptr,
                                  blob.gpu_index);
}

// Extension (not in the reference API): decode into a caller-owned vector,
// reusing its capacity -- no page faults when the buffer is recycled, so the
// host path runs at PCIe rate.  `out` is resized to the element count.
inline void decompress_lossless_into(const LosslessBlob& blob, std::vector<Bf16>& out) {
    out.resize(blob.meta.element_count());
    detail::gpu_decompress_into(blob.meta, blob.exp_stream, blob.signmant, kLosslessPrecision, 0, nullptr,
                                blob.gpu_index, out.data());
}

namespace detail {
inline std::uint16_t magnitude_bits(Bf16 x) { return x.bits & 0x7FFFu; }                      // tensorstore.hpp:133
inline double scale_coefficient(std::uint8_t s) { return 1.0 + static_cast<double>(s) / 128.0; }  // :135-137
}  // namespace detail

// tensorstore.hpp:141-208 (K6 normalise/round/pack + K1/K2/K3/K4 on the GPU)
inline LossyBlob compress_lossy(std::span<const Bf16> values, int k, std::uint32_t block_size, TensorMeta meta) {
    if (k != 0 && k != 1 && k != 3) throw std::invalid_argument("compress_lossy: precision must be 0, 1 or 3");
    if (block_size == 0) throw std::invalid_argument("compress_lossy: block size must be >= 1");
    meta.validate();
    if (meta.element_count() != values.size()) throw std::invalid_argument("compress: shape does not match value count");
    detail::DeviceBlob b;
    // the packed (k+1)-bit plane, faulted in beside the GPU work
    detail::PlaneAsync mant((values.size() * static_cast<std::size_t>(k + 1) + 7) / 8);
    const int rc = nzgpu_compress_host(reinterpret_cast<const std::uint16_t*>(values.data()), values.size(), k,
                                       block_size, 0, 0, &b.h);
    std::vector<std::uint8_t> plane = mant.get();
    detail::check(rc, "compress_lossy");
    detail::Exported e = detail::export_chunked(b.h, std::move(plane));
    return LossyBlob{std::move(meta),       k, block_size, std::move(e.scales), std::move(e.stream),
                     std::move(e.mantissas), std::move(e.index)};
}

// tensorstore.hpp:210-213
inline LossyBlob compress_lossy(std::span<const Bf16> values, int k, std::uint32_t block_size = kDefaultBlockSize) {
    return compress_lossy(values, k, block_size, TensorMeta{{values.size()}});
}

// tensorstore.hpp:215-238
inline std::vector<Bf16> decompress_lossy(const LossyBlob& blob) {
    return detail::gpu_decompress(blob.meta, blob.exp_stream, blob.signmant, blob.precision, blob.block_size,
                                  &blob.scales, blob.gpu_index);
}

// Extension: decompress_lossy into a caller-owned vector (see decompress_lossless_into).
inline void decompress_lossy_into(const LossyBlob& blob, std::vector<Bf16>& out) {
    out.resize(blob.meta.element_count());
    detail::gpu_decompress_into(blob.meta, blob.exp_stream, blob.signmant, blob.precision, blob.block_size,
                                &blob.scales, blob.gpu_index, out.data());
}

struct Footprint {  // tensorstore.hpp:242-253
    std::uint64_t exponent_bytes = 0;
    std::uint64_t mantissa_bytes = 0;
    std::uint64_t scale_bytes = 0;
    std::uint64_t table_bytes = 0;
    std::uint64_t header_bytes = 0;

    std::uint64_t total() const { return exponent_bytes + mantissa_bytes + scale_bytes + table_bytes + header_bytes; }
};

namespace detail {
// magic, version, precision, block, ndim, dims, scale/exp/signmant lengths, crc (tensorstore.hpp:257-261)
inline std::uint64_t nzt_header_bytes(std::size_t ndim) { return 35 + 8 * static_cast<std::uint64_t>(ndim); }
}  // namespace detail

// tensorstore.hpp:265-287 -- the side index is deliberately not counted.
inline Footprint footprint(const LosslessBlob& b) {
    return Footprint{b.exp_stream.stream_bytes(), b.signmant.size(), 0, ans::kTableBytes,
                     detail::nzt_header_bytes(b.meta.shape.size())};
}
inline Footprint footprint(const LossyBlob& b) {
    return Footprint{b.exp_stream.stream_bytes(), b.signmant.size(), b.scales.size(), ans::kTableBytes,
                     detail::nzt_header_bytes(b.meta.shape.size())};
}
inline Footprint footprint(const Blob& b) {
    return std::visit([](const auto& x) { return footprint(x); }, b);
}

// --- NZT container (tensorstore.hpp:289-477) --------------------------------
// Same byte layout; the CRC is computed on the GPU and read_nzt validates on
// the GPU (framing, CRC -> ChecksumError, table, stream, counts) through
// nzgpu_blob_read_nzt, so the error classes are the reference's.

namespace detail {
template <typename T>
void nzt_put(std::string& out, T v) {
    for (std::size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<char>(static_cast<std::uint64_t>(v) >> (8 * i)));
}

inline void write_nzt_sections(std::ostream& out, const TensorMeta& meta, int precision, std::uint32_t block,
                               const FrequencyTable& table, const std::vector<std::uint8_t>& scales,
                               const std::vector<std::uint8_t>& exp_bytes, const std::vector<std::uint8_t>& signmant) {
    const auto tb = table.serialize();
    const void* ptrs[4] = {tb.data(), scales.data(), exp_bytes.data(), signmant.data()};
    const std::uint64_t lens[4] = {tb.size(), scales.size(), exp_bytes.size(), signmant.size()};
    std::uint32_t crc = 0;
    check(nzgpu_crc32_host_sections(ptrs, lens, 4, &crc), "write_nzt");
    std::string head("NZT1");
    nzt_put<std::uint8_t>(head, 1);
    nzt_put<std::uint8_t>(head, static_cast<std::uint8_t>(precision));
    nzt_put<std::uint32_t>(head, block);
    nzt_put<std::uint8_t>(head, static_cast<std::uint8_t>(meta.shape.size()));
    for (std::uint64_t d : meta.shape) nzt_put<std::uint64_t>(head, d);
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    out.write(reinterpret_cast<const char*>(tb.data()), static_cast<std::streamsize>(tb.size()));
    std::string len4;
    nzt_put<std::uint32_t>(len4, static_cast<std::uint32_t>(scales.size()));
    out.write(len4.data(), 4);
    out.write(reinterpret_cast<const char*>(scales.data()), static_cast<std::streamsize>(scales.size()));
    std::string len8;
    nzt_put<std::uint64_t>(len8, exp_bytes.size());
    out.write(len8.data(), 8);
    out.write(reinterpret_cast<const char*>(exp_bytes.data()), static_cast<std::streamsize>(exp_bytes.size()));
    len8.clear();
    nzt_put<std::uint64_t>(len8, signmant.size());
    out.write(len8.data(), 8);
    out.write(reinterpret_cast<const char*>(signmant.data()), static_cast<std::streamsize>(signmant.size()));
    std::string c4;
    nzt_put<std::uint32_t>(c4, crc);
    out.write(c4.data(), 4);
    if (!out) throw Error("nzt: write failed");
}

// Pull `k` more bytes of the file into `buf` (FormatError at end of file).
inline void nzt_pull(std::istream& in, std::string& buf, std::uint64_t k) {
    const std::size_t at = buf.size();
    buf.resize(at + k);
    in.read(buf.data() + at, static_cast<std::streamsize>(k));
    if (static_cast<std::uint64_t>(in.gcount()) != k) throw FormatError("unexpected end of file");
}
inline std::uint64_t nzt_le(const std::string& buf, std::size_t at, int bytes) {
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(static_cast<std::uint8_t>(buf[at + i])) << (8 * i);
    return v;
}
}  // namespace detail

inline void write_nzt(const LosslessBlob& blob, std::ostream& out) {  // tensorstore.hpp:372-380
    detail::write_nzt_sections(out, blob.meta, kLosslessPrecision, 0, blob.table(), {}, serialize_stream(blob.exp_stream),
                               blob.signmant);
}

inline void write_nzt(const LossyBlob& blob, std::ostream& out) {  // tensorstore.hpp:382-390
    detail::write_nzt_sections(out, blob.meta, blob.precision, blob.block_size, blob.table(), blob.scales,
                               serialize_stream(blob.exp_stream), blob.signmant);
}

inline void write_nzt(const Blob& blob, std::ostream& out) {
    std::visit([&](const auto& b) { write_nzt(b, out); }, blob);
}

// tensorstore.hpp:403-477: the header fields are read one by one so that a
// stream positioned after this file is left there; the payload lengths come
// from the header, and the assembled file is validated by the GPU reader.
inline Blob read_nzt(std::istream& in) {
    std::string f;
    char magic[4];
    in.read(magic, 4);
    if (in.gcount() != 4 || std::string(magic, 4) != "NZT1") throw FormatError("nzt: bad magic");
    f.assign(magic, 4);
    detail::nzt_pull(in, f, 2);
    if (static_cast<std::uint8_t>(f[4]) != 1) throw FormatError("nzt: unsupported version");
    const int precision = static_cast<std::uint8_t>(f[5]);
    if (precision != 0 && precision != 1 && precision != 3 && precision != kLosslessPrecision)
        throw FormatError("nzt: invalid precision");
    detail::nzt_pull(in, f, 5);
    const std::uint64_t block = detail::nzt_le(f, 6, 4);
    const std::uint64_t ndim = static_cast<std::uint8_t>(f[10]);
    if (ndim == 0 || ndim > 8) throw FormatError("nzt: invalid rank");
    detail::nzt_pull(in, f, 8 * ndim);
    std::uint64_t n = 1;
    for (std::uint64_t i = 0; i < ndim; ++i) {
        const std::uint64_t d = detail::nzt_le(f, 11 + 8 * i, 8);
        if (d == 0) throw FormatError("nzt: zero dimension");
        if (d > (std::uint64_t{1} << 40) / n) throw FormatError("nzt: element count overflow");
        n *= d;
    }
    // section lengths are checked against the element count before reading
    if (precision == kLosslessPrecision ? block != 0 : block == 0) throw FormatError("nzt: block size");
    const std::uint64_t want_scales = precision == kLosslessPrecision ? 0 : (n + block - 1) / block;
    const std::uint64_t want_sm = (n * (static_cast<std::uint64_t>(precision) + 1) + 7) / 8;
    const std::uint64_t cap = 2 * n + 16 * ((n + ans::kChunkSymbols - 1) / ans::kChunkSymbols) + 64;
    detail::nzt_pull(in, f, 512 + 4);
    if (detail::nzt_le(f, f.size() - 4, 4) != want_scales) throw FormatError("nzt: scale count mismatch");
    detail::nzt_pull(in, f, want_scales + 8);
    const std::uint64_t exp_len = detail::nzt_le(f, f.size() - 8, 8);
    if (exp_len > cap) throw FormatError("nzt: exponent stream oversized");
    detail::nzt_pull(in, f, exp_len + 8);
    if (detail::nzt_le(f, f.size() - 8, 8) != want_sm) throw FormatError("nzt: sign-mantissa length mismatch");
    detail::nzt_pull(in, f, want_sm + 4);
    detail::DeviceBlob b;
    std::uint64_t dims[8] = {};
    int nd = 0;
    detail::check(nzgpu_blob_read_nzt(reinterpret_cast<const std::uint8_t*>(f.data()), f.size(), 0, nullptr, &b.h,
                                      dims, &nd),
                  "read_nzt");
    TensorMeta meta{std::vector<std::uint64_t>(dims, dims + nd)};
    detail::Sections s = detail::export_blob(b.h);
    const FrequencyTable table = detail::table_from(s.freqs);
    if (precision == kLosslessPrecision)
        return LosslessBlob{std::move(meta), deserialize_stream(s.stream, table), std::move(s.mantissas),
                            std::move(s.index)};
    return LossyBlob{std::move(meta),         precision,           static_cast<std::uint32_t>(block),
                     std::move(s.scales),     deserialize_stream(s.stream, table), std::move(s.mantissas),
                     std::move(s.index)};
}

// --- BFT raw tensor format (tensorstore.hpp:479-517) -------------------------
inline void write_bft(const Tensor& tensor, std::ostream& out) {
    tensor.meta.validate();
    if (tensor.meta.element_count() != tensor.values.size())
        throw std::invalid_argument("bft: shape does not match value count");
    std::string head("BFT1");
    detail::nzt_put<std::uint8_t>(head, static_cast<std::uint8_t>(tensor.meta.shape.size()));
    for (std::uint64_t d : tensor.meta.shape) detail::nzt_put<std::uint64_t>(head, d);
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    std::string body;
    body.reserve(2 * tensor.values.size());
    for (Bf16 v : tensor.values) detail::nzt_put<std::uint16_t>(body, v.bits);
    out.write(body.data(), static_cast<std::streamsize>(body.size()));
    if (!out) throw Error("bft: write failed");
}

inline Tensor read_bft(std::istream& in) {
    char magic[4];
    in.read(magic, 4);
    if (in.gcount() != 4 || std::string(magic, 4) != "BFT1") throw FormatError("bft: bad magic");
    std::string f;
    detail::nzt_pull(in, f, 1);
    const std::uint64_t ndim = static_cast<std::uint8_t>(f[0]);
    if (ndim == 0 || ndim > 8) throw FormatError("bft: invalid rank");
    detail::nzt_pull(in, f, 8 * ndim);
    Tensor t;
    t.meta.shape.resize(ndim);
    std::uint64_t n = 1;
    for (std::uint64_t i = 0; i < ndim; ++i) {
        const std::uint64_t d = detail::nzt_le(f, 1 + 8 * i, 8);
        if (d == 0) throw FormatError("bft: zero dimension");
        if (d > (std::uint64_t{1} << 40) / n) throw FormatError("bft: element count overflow");
        t.meta.shape[i] = d;
        n *= d;
    }
    std::string body;
    detail::nzt_pull(in, body, 2 * n);
    t.values.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) t.values[i].bits = static_cast<std::uint16_t>(detail::nzt_le(body, 2 * i, 2));
    return t;
}

}  // namespace neuzip
