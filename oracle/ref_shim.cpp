// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (never copied into this repo) into
// oracle/_ref/libneuzip_ref.so, with the reference's effective flags
// (-std=c++20 -O2 -pthread, proj/tools/CMakeLists.txt:4).  It lets the
// Python tests pin the C restatement (neuzip_oracle.c) against the reference
// itself, and lets bench.py time the reference's own CPU codec (its
// parallel_for over std::thread, parallel.hpp:28-43) as the baseline arm.
//
// Every export mirrors the orc_* function of the same suffix in
// neuzip_oracle.h (same arguments, same status codes).
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "neuzip/ans.hpp"
#include "neuzip/bitfloat.hpp"
#include "neuzip/crc32.hpp"
#include "neuzip/entropy.hpp"
#include "neuzip/errors.hpp"
#include "neuzip/rng.hpp"
#include "neuzip/tensorstore.hpp"

using namespace neuzip;

namespace {

constexpr int kOk = 0, kInvalid = -1, kTruncated = -2, kDesync = -3, kLength = -4,
              kNonFinite = -5, kBadTable = -6, kChecksum = -7;

int classify(const std::exception& e) {
    if (dynamic_cast<const NonFiniteError*>(&e)) return kNonFinite;
    if (dynamic_cast<const ChecksumError*>(&e)) return kChecksum;
    if (dynamic_cast<const FormatError*>(&e)) {
        const std::string what = e.what();
        if (what.find("truncated") != std::string::npos) return kTruncated;
        if (what.find("desynchronization") != std::string::npos) return kDesync;
        if (what.find("4096") != std::string::npos) return kBadTable;
        return kLength;
    }
    return kInvalid;
}

FrequencyTable table_of(const std::uint16_t* freqs) {
    std::array<std::uint16_t, 256> f{};
    std::memcpy(f.data(), freqs, 512);
    return FrequencyTable::from_frequencies(f);
}

// ans_encode with an arbitrary chunk size: ans_encode_chunk over S-spans
// (ans.hpp:258-271 with kChunkSymbols replaced by S).
AnsStream encode_spans(std::span<const std::uint8_t> xs, const FrequencyTable& t,
                       std::uint64_t chunk) {
    if (chunk == ans::kChunkSymbols) return ans_encode(xs, t);
    AnsStream s{t, {}};
    for (std::uint64_t b = 0; b < xs.size(); b += chunk) {
        const std::uint64_t len = std::min<std::uint64_t>(chunk, xs.size() - b);
        s.chunks.push_back(ans_encode_chunk(xs.subspan(b, len), t));
    }
    return s;
}

std::int64_t emit_stream(const AnsStream& s, std::uint8_t* out) {
    const std::vector<std::uint8_t> bytes = serialize_stream(s);
    std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<std::int64_t>(bytes.size());
}

AnsStream parse_stream(const std::uint8_t* stream, std::uint64_t len, const std::uint16_t* freqs) {
    return deserialize_stream(std::span<const std::uint8_t>(stream, len), table_of(freqs));
}

std::span<const Bf16> as_bf16(const std::uint16_t* v, std::uint64_t n) {
    static_assert(sizeof(Bf16) == 2);
    return std::span<const Bf16>(reinterpret_cast<const Bf16*>(v), n);
}

}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END                 \
    }                             \
    catch (const std::exception& e) { return classify(e); }

extern "C" {

int ref_build_table(const std::uint64_t* counts, std::uint16_t* freqs) {
    GUARD_BEGIN
    const FrequencyTable t = build_table(std::span<const std::uint64_t>(counts, 256));
    std::memcpy(freqs, t.frequencies().data(), 512);
    return kOk;
    GUARD_END
}

std::int64_t ref_ans_encode_chunk(const std::uint8_t* symbols, std::uint64_t nsym,
                                  const std::uint16_t* freqs, std::uint8_t* payload) {
    GUARD_BEGIN
    const AnsChunk c = ans_encode_chunk(std::span<const std::uint8_t>(symbols, nsym), table_of(freqs));
    std::memcpy(payload, c.payload.data(), c.payload.size());
    return static_cast<std::int64_t>(c.payload.size());
    GUARD_END
}

int ref_ans_decode_chunk(const std::uint8_t* payload, std::uint64_t len, std::uint64_t nsym,
                         const std::uint16_t* freqs, std::uint8_t* out) {
    GUARD_BEGIN
    AnsChunk c{static_cast<std::uint32_t>(nsym), std::vector<std::uint8_t>(payload, payload + len)};
    const auto xs = ans_decode_chunk(c, table_of(freqs));
    std::memcpy(out, xs.data(), xs.size());
    return kOk;
    GUARD_END
}

std::int64_t ref_ans_encode_stream(const std::uint8_t* symbols, std::uint64_t n, std::uint64_t chunk,
                                   const std::uint16_t* freqs, std::uint8_t* stream) {
    GUARD_BEGIN
    return emit_stream(encode_spans(std::span<const std::uint8_t>(symbols, n), table_of(freqs), chunk),
                       stream);
    GUARD_END
}

int ref_ans_decode_stream(const std::uint8_t* stream, std::uint64_t len, const std::uint16_t* freqs,
                          std::uint8_t* out, std::uint64_t n) {
    GUARD_BEGIN
    const auto xs = ans_decode(parse_stream(stream, len, freqs));
    if (xs.size() != n) return kLength;
    std::memcpy(out, xs.data(), xs.size());
    return kOk;
    GUARD_END
}

std::int64_t ref_compress_lossless(const std::uint16_t* values, std::uint64_t n, std::uint64_t chunk,
                                   std::uint16_t* freqs, std::uint8_t* stream, std::uint8_t* signmant) {
    GUARD_BEGIN
    LosslessBlob blob;
    if (chunk == ans::kChunkSymbols) {
        blob = compress_lossless(as_bf16(values, n), TensorMeta{{n}});
    } else {
        // Same split/histogram/table as tensorstore.hpp:93-103, chunked encode over S-spans.
        TensorMeta{{n}}.validate();
        std::vector<std::uint8_t> exps(n), sm(n);
        std::vector<std::uint64_t> counts(256, 0);
        for (std::uint64_t i = 0; i < n; ++i) {
            const ComponentTriple t = split(Bf16{values[i]});
            exps[i] = t.exponent;
            sm[i] = static_cast<std::uint8_t>((t.sign << 7) | t.mantissa);
            ++counts[t.exponent];
        }
        const FrequencyTable t = build_table(counts);
        blob = LosslessBlob{TensorMeta{{n}}, encode_spans(exps, t, chunk), std::move(sm)};
    }
    std::memcpy(freqs, blob.table().frequencies().data(), 512);
    std::memcpy(signmant, blob.signmant.data(), n);
    return emit_stream(blob.exp_stream, stream);
    GUARD_END
}

int ref_decompress_lossless(const std::uint8_t* stream, std::uint64_t stream_len,
                            const std::uint16_t* freqs, const std::uint8_t* signmant,
                            std::uint64_t signmant_len, std::uint64_t n, std::uint16_t* out) {
    GUARD_BEGIN
    LosslessBlob blob{TensorMeta{{n}}, parse_stream(stream, stream_len, freqs),
                      std::vector<std::uint8_t>(signmant, signmant + signmant_len)};
    const std::vector<Bf16> back = decompress_lossless(blob);
    std::memcpy(out, back.data(), back.size() * 2);
    return kOk;
    GUARD_END
}

// Prepared blobs: parse once, then time decompress_lossless / decompress_lossy
// alone (tensorstore.hpp:112-125, :215-238) -- the CPU baseline measures the
// reference's decode, not this shim's marshalling.
void* ref_prepare(const std::uint8_t* stream, std::uint64_t stream_len, const std::uint16_t* freqs,
                  const std::uint8_t* mant, std::uint64_t mant_len, const std::uint8_t* scales,
                  std::uint64_t scales_len, int k, std::uint32_t block, std::uint64_t n) {
    try {
        if (k == kLosslessPrecision) {
            return new Blob(LosslessBlob{TensorMeta{{n}}, parse_stream(stream, stream_len, freqs),
                                         std::vector<std::uint8_t>(mant, mant + mant_len)});
        }
        return new Blob(LossyBlob{TensorMeta{{n}}, k, block, std::vector<std::uint8_t>(scales, scales + scales_len),
                                  parse_stream(stream, stream_len, freqs),
                                  std::vector<std::uint8_t>(mant, mant + mant_len)});
    } catch (...) {
        return nullptr;
    }
}

int ref_decompress_prepared(void* h, std::uint16_t* out) {
    GUARD_BEGIN
    const Blob& b = *static_cast<Blob*>(h);
    const std::vector<Bf16> back = std::holds_alternative<LosslessBlob>(b) ? decompress_lossless(std::get<LosslessBlob>(b))
                                                                          : decompress_lossy(std::get<LossyBlob>(b));
    std::memcpy(out, back.data(), back.size() * 2);
    return kOk;
    GUARD_END
}

void ref_free_prepared(void* h) { delete static_cast<Blob*>(h); }

std::int64_t ref_compress_lossy(const std::uint16_t* values, std::uint64_t n, int k, std::uint32_t block,
                                std::uint64_t chunk, std::uint16_t* freqs, std::uint8_t* scales,
                                std::uint8_t* stream, std::uint8_t* packed) {
    GUARD_BEGIN
    LossyBlob blob = compress_lossy(as_bf16(values, n), k, block, TensorMeta{{n}});
    if (chunk != ans::kChunkSymbols) {
        const std::vector<std::uint8_t> exps = ans_decode(blob.exp_stream);
        blob.exp_stream = encode_spans(exps, blob.table(), chunk);
    }
    std::memcpy(freqs, blob.table().frequencies().data(), 512);
    std::memcpy(scales, blob.scales.data(), blob.scales.size());
    std::memcpy(packed, blob.signmant.data(), blob.signmant.size());
    return emit_stream(blob.exp_stream, stream);
    GUARD_END
}

int ref_decompress_lossy(const std::uint8_t* stream, std::uint64_t stream_len, const std::uint16_t* freqs,
                         const std::uint8_t* packed, std::uint64_t packed_len, const std::uint8_t* scales,
                         std::uint64_t scales_len, int k, std::uint32_t block, std::uint64_t n,
                         std::uint16_t* out) {
    GUARD_BEGIN
    LossyBlob blob{TensorMeta{{n}},
                   k,
                   block,
                   std::vector<std::uint8_t>(scales, scales + scales_len),
                   parse_stream(stream, stream_len, freqs),
                   std::vector<std::uint8_t>(packed, packed + packed_len)};
    const std::vector<Bf16> back = decompress_lossy(blob);
    std::memcpy(out, back.data(), back.size() * 2);
    return kOk;
    GUARD_END
}

std::uint64_t ref_footprint_total_lossless(const std::uint16_t* values, std::uint64_t n) {
    return footprint(compress_lossless(as_bf16(values, n))).total();
}

void ref_gaussian_bf16(std::uint64_t seed, std::uint64_t n, double sigma, std::uint16_t* out) {
    const std::vector<Bf16> v = rng::gaussian_bf16(seed, n, sigma);
    std::memcpy(out, v.data(), n * 2);
}

std::uint64_t ref_rng_derive(std::uint64_t seed, std::uint64_t tag) { return rng::derive(seed, tag); }

std::uint32_t ref_crc32(const std::uint8_t* data, std::uint64_t n) {
    return crc32(std::span<const std::uint8_t>(data, n));
}

// write_nzt of a lossless blob (tensorstore.hpp:372-380); returns bytes written.
std::int64_t ref_write_nzt_lossless(const std::uint16_t* values, const std::uint64_t* shape, int ndim,
                                    std::uint8_t* out, std::uint64_t cap) {
    GUARD_BEGIN
    std::uint64_t n = 1;
    std::vector<std::uint64_t> dims(shape, shape + ndim);
    for (auto d : dims) n *= d;
    std::ostringstream os(std::ios::binary);
    write_nzt(Blob(compress_lossless(as_bf16(values, n), TensorMeta{dims})), os);
    const std::string s = os.str();
    if (s.size() > cap) return kInvalid;
    std::memcpy(out, s.data(), s.size());
    return static_cast<std::int64_t>(s.size());
    GUARD_END
}

// write_nzt of a lossy blob (tensorstore.hpp:382-390); returns bytes written.
std::int64_t ref_write_nzt_lossy(const std::uint16_t* values, const std::uint64_t* shape, int ndim, int k,
                                 std::uint32_t block, std::uint8_t* out, std::uint64_t cap) {
    GUARD_BEGIN
    std::uint64_t n = 1;
    std::vector<std::uint64_t> dims(shape, shape + ndim);
    for (auto d : dims) n *= d;
    std::ostringstream os(std::ios::binary);
    write_nzt(Blob(compress_lossy(as_bf16(values, n), k, block, TensorMeta{dims})), os);
    const std::string s = os.str();
    if (s.size() > cap) return kInvalid;
    std::memcpy(out, s.data(), s.size());
    return static_cast<std::int64_t>(s.size());
    GUARD_END
}

// read_nzt + decompress (tensorstore.hpp:403-477, :112-125, :215-238):
// 0 and the values on success, else the reference's exception class.
int ref_read_nzt(const std::uint8_t* data, std::uint64_t len, std::uint16_t* values, std::uint64_t cap_n,
                 std::uint64_t* n_out) {
    GUARD_BEGIN
    std::istringstream is(std::string(reinterpret_cast<const char*>(data), len), std::ios::binary);
    const Blob blob = read_nzt(is);
    const std::vector<Bf16> out = std::visit(
        [](const auto& b) {
            if constexpr (std::is_same_v<std::decay_t<decltype(b)>, LosslessBlob>) return decompress_lossless(b);
            else return decompress_lossy(b);
        },
        blob);
    if (out.size() > cap_n) return kInvalid;
    std::memcpy(values, out.data(), out.size() * 2);
    *n_out = out.size();
    return kOk;
    GUARD_END
}

// analyze_tensor (entropy.hpp:57-94): h_sign, h_exp, h_mant, ideal, exponent_only.
void ref_entropy_report(const std::uint16_t* values, std::uint64_t n, double* out5) {
    const EntropyReport r = analyze_tensor(as_bf16(values, n));
    out5[0] = r.h_sign;
    out5[1] = r.h_exp;
    out5[2] = r.h_mant;
    out5[3] = r.ideal_ratio;
    out5[4] = r.exponent_only_ratio;
}

}  // extern "C"
