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

#include <cstdint>
#include <span>
#include <variant>
#include <vector>

#include "neuzip/ans.hpp"
#include "neuzip/bitfloat.hpp"
#include "neuzip/errors.hpp"

namespace neuzip {

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

inline FrequencyTable table_from(const std::vector<std::uint16_t>& f) {
    std::array<std::uint16_t, 256> a{};
    std::copy(f.begin(), f.end(), a.begin());
    return FrequencyTable::from_frequencies(a);
}

inline std::vector<Bf16> gpu_decompress(const TensorMeta& meta, const AnsStream& stream,
                                        const std::vector<std::uint8_t>& mant, int precision, std::uint32_t block,
                                        const std::vector<std::uint8_t>* scales,
                                        const std::vector<std::uint8_t>& index) {
    const std::vector<std::uint8_t> bytes = serialize_stream(stream);
    const std::uint64_t n = meta.element_count();
    nzgpu_host_tensor t{};
    t.n = n;
    t.precision = precision;
    t.block_size = block;
    t.freqs = stream.table.frequencies().data();
    t.stream = bytes.data();
    t.stream_len = bytes.size();
    t.mantissas = mant.data();
    t.mantissa_len = mant.size();
    if (scales) {
        t.scales = scales->data();
        t.scales_len = scales->size();
    }
    t.index = index.empty() ? nullptr : index.data();
    t.index_len = index.size();
    std::vector<Bf16> out(n);
    check(nzgpu_decompress_host(&t, reinterpret_cast<std::uint16_t*>(out.data())), "decompress");
    return out;
}

}  // namespace detail

// tensorstore.hpp:87-106
inline LosslessBlob compress_lossless(std::span<const Bf16> values, TensorMeta meta) {
    meta.validate();
    if (meta.element_count() != values.size()) throw std::invalid_argument("compress: shape does not match value count");
    detail::DeviceBlob b;
    detail::check(nzgpu_compress_host(reinterpret_cast<const std::uint16_t*>(values.data()), values.size(),
                                      kLosslessPrecision, 0, 0, 0, &b.h),
                  "compress_lossless");
    detail::Sections s = detail::export_blob(b.h);
    const FrequencyTable table = detail::table_from(s.freqs);
    return LosslessBlob{std::move(meta), deserialize_stream(s.stream, table), std::move(s.mantissas), std::move(s.index)};
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
    detail::check(nzgpu_compress_host(reinterpret_cast<const std::uint16_t*>(values.data()), values.size(), k,
                                      block_size, 0, 0, &b.h),
                  "compress_lossy");
    detail::Sections s = detail::export_blob(b.h);
    const FrequencyTable table = detail::table_from(s.freqs);
    return LossyBlob{std::move(meta),   k, block_size, std::move(s.scales), deserialize_stream(s.stream, table),
                     std::move(s.mantissas), std::move(s.index)};
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

}  // namespace neuzip
