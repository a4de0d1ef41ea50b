#pragma once
// Drop-in for /root/reference/proj/include/neuzip/ans.hpp: the 12-bit
// byte-alphabet rANS coder with 65,536-symbol chunks.  Same types, names,
// signatures, byte formats and exceptions; every encode/decode and the table
// build run on the B200 through the C ABI (include/nzgpu.h).  Only framing
// (serialize/deserialize, byte layout) and the FrequencyTable accessors are
// host code.

#include <algorithm>
#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "neuzip/errors.hpp"

namespace neuzip {

namespace ans {  // ans.hpp:29-35
constexpr std::uint32_t kProbBits = 12;
constexpr std::uint32_t kProbScale = 1u << kProbBits;
constexpr std::uint32_t kStateLow = 1u << 23;
constexpr std::size_t kChunkSymbols = 65536;
constexpr std::size_t kTableBytes = 512;
}  // namespace ans

// ans.hpp:39-152
class FrequencyTable {
public:
    FrequencyTable() {
        std::array<std::uint16_t, 256> f{};
        f[0] = static_cast<std::uint16_t>(ans::kProbScale);
        install(f);
    }

    // Largest-remainder quantisation with floor-at-1 repair (ans.hpp:52-93),
    // computed by the K2 kernel.
    static FrequencyTable from_counts(std::span<const std::uint64_t> counts) {
        if (counts.size() != 256) throw std::invalid_argument("frequency table needs 256 counts");
        std::array<std::uint16_t, 256> f{};
        detail::check(nzgpu_build_table_host(counts.data(), f.data()), "frequency table");
        FrequencyTable t;
        t.install(f);
        return t;
    }

    static FrequencyTable from_frequencies(const std::array<std::uint16_t, 256>& freqs) {  // ans.hpp:96-103
        std::uint32_t sum = 0;
        for (std::uint16_t f : freqs) sum += f;
        if (sum != ans::kProbScale) throw FormatError("frequency table does not sum to 4096");
        FrequencyTable t;
        t.install(freqs);
        return t;
    }

    std::uint16_t freq(std::uint8_t s) const { return freqs_[s]; }
    std::uint16_t cum(std::uint8_t s) const { return cum_[s]; }
    bool present(std::uint8_t s) const { return freqs_[s] != 0; }
    std::uint8_t symbol_at(std::uint32_t slot) const { return slot_symbol_[slot]; }
    const std::array<std::uint16_t, 256>& frequencies() const { return freqs_; }

    std::array<std::uint8_t, ans::kTableBytes> serialize() const {  // 256 x u16 LE, ans.hpp:111-118
        std::array<std::uint8_t, ans::kTableBytes> out{};
        for (int s = 0; s < 256; ++s) {
            out[2 * s] = static_cast<std::uint8_t>(freqs_[s]);
            out[2 * s + 1] = static_cast<std::uint8_t>(freqs_[s] >> 8);
        }
        return out;
    }

    static FrequencyTable deserialize(std::span<const std::uint8_t> bytes) {  // ans.hpp:120-130
        if (bytes.size() != ans::kTableBytes) throw FormatError("frequency table must be 512 bytes");
        std::array<std::uint16_t, 256> f{};
        for (int s = 0; s < 256; ++s) f[s] = static_cast<std::uint16_t>(bytes[2 * s] | (bytes[2 * s + 1] << 8));
        return from_frequencies(f);
    }

    friend bool operator==(const FrequencyTable& a, const FrequencyTable& b) { return a.freqs_ == b.freqs_; }

private:
    void install(const std::array<std::uint16_t, 256>& f) {  // cum starts + slot map, ans.hpp:137-147
        freqs_ = f;
        std::uint32_t c = 0;
        for (int s = 0; s < 256; ++s) {
            cum_[s] = static_cast<std::uint16_t>(c);
            std::fill_n(slot_symbol_.begin() + std::min<std::uint32_t>(c, ans::kProbScale),
                        std::min<std::uint32_t>(f[s], ans::kProbScale - std::min<std::uint32_t>(c, ans::kProbScale)),
                        static_cast<std::uint8_t>(s));
            c += f[s];
        }
    }

    std::array<std::uint16_t, 256> freqs_{};
    std::array<std::uint16_t, 256> cum_{};
    std::array<std::uint8_t, ans::kProbScale> slot_symbol_{};
};

inline FrequencyTable build_table(std::span<const std::uint64_t> counts) {  // ans.hpp:154-156
    return FrequencyTable::from_counts(counts);
}

struct AnsChunk {  // ans.hpp:159-164
    std::uint32_t symbol_count = 0;
    std::vector<std::uint8_t> payload;

    friend bool operator==(const AnsChunk&, const AnsChunk&) = default;
};

struct AnsStream {  // ans.hpp:166-181
    FrequencyTable table;
    std::vector<AnsChunk> chunks;

    std::uint64_t symbol_count() const {
        std::uint64_t n = 0;
        for (const AnsChunk& c : chunks) n += c.symbol_count;
        return n;
    }
    std::uint64_t stream_bytes() const {
        std::uint64_t n = 4;
        for (const AnsChunk& c : chunks) n += 8 + c.payload.size();
        return n;
    }
};

namespace detail {

inline void put_u32le(std::vector<std::uint8_t>& out, std::uint32_t v) {  // ans.hpp:185-190
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

inline std::uint32_t get_u32le(std::span<const std::uint8_t> b) {  // ans.hpp:192-197
    return static_cast<std::uint32_t>(b[0]) | (static_cast<std::uint32_t>(b[1]) << 8) |
           (static_cast<std::uint32_t>(b[2]) << 16) | (static_cast<std::uint32_t>(b[3]) << 24);
}

}  // namespace detail

inline std::array<std::uint8_t, ans::kTableBytes> serialize_table(const FrequencyTable& t) { return t.serialize(); }
inline FrequencyTable deserialize_table(std::span<const std::uint8_t> b) { return FrequencyTable::deserialize(b); }

// ans.hpp:306-316
inline std::vector<std::uint8_t> serialize_stream(const AnsStream& stream) {
    std::vector<std::uint8_t> out;
    out.reserve(stream.stream_bytes());
    detail::put_u32le(out, static_cast<std::uint32_t>(stream.chunks.size()));
    for (const AnsChunk& c : stream.chunks) {
        detail::put_u32le(out, c.symbol_count);
        detail::put_u32le(out, static_cast<std::uint32_t>(c.payload.size()));
        out.insert(out.end(), c.payload.begin(), c.payload.end());
    }
    return out;
}

// ans.hpp:318-347
inline AnsStream deserialize_stream(std::span<const std::uint8_t> bytes, const FrequencyTable& table) {
    std::size_t pos = 0;
    auto need = [&](std::size_t k) {
        if (bytes.size() - pos < k) throw FormatError("ans stream: truncated framing");
    };
    need(4);
    const std::uint32_t count = detail::get_u32le(bytes.subspan(0, 4));
    pos = 4;
    AnsStream s{table, {}};
    s.chunks.reserve(std::min<std::size_t>(count, bytes.size() / 8 + 1));
    for (std::uint32_t c = 0; c < count; ++c) {
        need(8);
        AnsChunk ch;
        ch.symbol_count = detail::get_u32le(bytes.subspan(pos, 4));
        const std::uint32_t len = detail::get_u32le(bytes.subspan(pos + 4, 4));
        pos += 8;
        need(len);
        ch.payload.assign(bytes.begin() + static_cast<std::ptrdiff_t>(pos),
                          bytes.begin() + static_cast<std::ptrdiff_t>(pos + len));
        pos += len;
        s.chunks.push_back(std::move(ch));
    }
    if (pos != bytes.size()) throw FormatError("ans stream: trailing bytes");
    return s;
}

namespace detail {

// GPU encode of `symbols` with chunk size `chunk` -> serialized stream.
inline std::vector<std::uint8_t> gpu_encode(std::span<const std::uint8_t> symbols, const FrequencyTable& table,
                                            std::uint64_t chunk) {
    const std::uint64_t n = symbols.size();
    const std::uint64_t chunks = (n + chunk - 1) / chunk;
    std::vector<std::uint8_t> out(4 + 12 * chunks + 2 * n + 16);
    std::uint64_t len = 0;
    check(nzgpu_ans_encode_host(symbols.data(), n, table.frequencies().data(), static_cast<std::uint32_t>(chunk),
                                out.data(), out.size(), &len),
          "ans encode");
    out.resize(len);
    return out;
}

inline std::vector<std::uint8_t> gpu_decode(std::span<const std::uint8_t> stream, const FrequencyTable& table,
                                            std::uint64_t n) {
    std::vector<std::uint8_t> out(n);
    check(nzgpu_ans_decode_host(stream.data(), stream.size(), table.frequencies().data(), out.data(), n), "ans decode");
    return out;
}

}  // namespace detail

// ans.hpp:202-225: one chunk, encoded on the GPU (a one-chunk stream).
inline AnsChunk ans_encode_chunk(std::span<const std::uint8_t> symbols, const FrequencyTable& table) {
    if (symbols.empty()) {  // the encoder never steps: payload = LE32(initial state)
        AnsChunk c;
        detail::put_u32le(c.payload, ans::kStateLow);
        return c;
    }
    const std::vector<std::uint8_t> s = detail::gpu_encode(symbols, table, symbols.size());
    AnsStream one = deserialize_stream(s, table);
    return std::move(one.chunks.at(0));
}

// ans.hpp:229-256: one chunk, decoded on the GPU.
inline std::vector<std::uint8_t> ans_decode_chunk(const AnsChunk& chunk, const FrequencyTable& table) {
    AnsStream one{table, {chunk}};
    const std::vector<std::uint8_t> s = serialize_stream(one);
    return detail::gpu_decode(s, table, chunk.symbol_count);
}

// ans.hpp:260-271
inline AnsStream ans_encode(std::span<const std::uint8_t> symbols, const FrequencyTable& table) {
    if (symbols.empty()) return AnsStream{table, {}};
    return deserialize_stream(detail::gpu_encode(symbols, table, ans::kChunkSymbols), table);
}

// ans.hpp:273-293
inline std::vector<std::uint8_t> ans_decode(const AnsStream& stream) {
    return detail::gpu_decode(serialize_stream(stream), stream.table, stream.symbol_count());
}

}  // namespace neuzip
