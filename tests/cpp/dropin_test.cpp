// Acceptance-style test of the drop-in C++ API (include/neuzip/*.hpp) in the
// spirit of the reference's own suites (proj/tests/test_bitfloat.cpp,
// test_ans.cpp, test_tensorstore.cpp, acceptance.cpp): same calls, same
// expected values and exception types, run against the B200 implementation.
// Exits 0 when every check passes.  Built and run by tests/test_cpp_dropin.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <sstream>
#include <cstring>
#include <functional>
#include <random>
#include <string>

#include "neuzip/neuzip.hpp"

using namespace neuzip;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (cond) {                                                            \
            ++g_pass;                                                          \
        } else {                                                               \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)

template <class E>
static bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// rng.hpp-style counter generator (splitmix64 + Box-Muller), test inputs only.
static std::uint64_t mix64(std::uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static std::vector<Bf16> gaussian(std::uint64_t seed, std::size_t n, double sigma) {
    std::vector<Bf16> v(n);
    for (std::size_t i = 0; i < n; ++i) {
        const double u1 = (static_cast<double>(mix64(seed + (2 * i + 1) * 0x9E3779B97F4A7C15ull) >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(mix64(seed + (2 * i + 2) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
        v[i] = Bf16::from_float(static_cast<float>(sigma * std::sqrt(-2.0 * std::log(u1)) *
                                                   std::cos(2.0 * 3.141592653589793238462643383279502884 * u2)));
    }
    return v;
}

static std::vector<std::uint64_t> counts_of(const std::vector<std::uint8_t>& xs) {
    std::vector<std::uint64_t> c(256, 0);
    for (auto s : xs) ++c[s];
    return c;
}

// The same lossy blob through the batched host entry (nzgpu_decompress_host,
// whole-tensor staging): an independent route for the sliced pipeline of
// decompress_lossy (nzgpu_decompress_host_sections).
static std::vector<Bf16> via_batch_path(const LossyBlob& b) {
    const auto stream = serialize_stream(b.exp_stream);
    nzgpu_host_tensor t{};
    t.n = b.meta.element_count();
    t.precision = b.precision;
    t.block_size = b.block_size;
    t.freqs = b.exp_stream.table.frequencies().data();
    t.stream = stream.data();
    t.stream_len = stream.size();
    t.mantissas = b.signmant.data();
    t.mantissa_len = b.signmant.size();
    t.scales = b.scales.data();
    t.scales_len = b.scales.size();
    t.index = b.gpu_index.data();
    t.index_len = b.gpu_index.size();
    std::vector<Bf16> out(t.n);
    if (nzgpu_decompress_host(&t, reinterpret_cast<std::uint16_t*>(out.data())) != NZGPU_OK) out.clear();
    return out;
}

int main() {
    // --- bitfloat (test_bitfloat.cpp) ------------------------------------
    {
        int bad = 0;
        for (std::uint32_t b = 0; b < 65536; ++b) {
            const Bf16 x{static_cast<std::uint16_t>(b)};
            if (merge(split(x)) != x) ++bad;
        }
        CHECK(bad == 0);
        CHECK((split(Bf16{0x3F80}) == ComponentTriple{0, 127, 0}));
        CHECK(Bf16::from_float(-5.0f).bits == 0xC0A0);
        CHECK((split(Bf16{0xC0A0}) == ComponentTriple{1, 129, 32}));
        CHECK(throws<std::invalid_argument>([] { (void)merge({2, 0, 0}); }));
        CHECK(round_mantissa(0b1010110, 3).mantissa == 0b1010000);
        CHECK(round_mantissa(127, 3).carry);
        CHECK(throws<std::invalid_argument>([] { (void)round_mantissa(0, 2); }));
        CHECK(Bf16::from_float(1.00390625f).bits == 0x3F80);
        const std::vector<SignedMantissa> s8 = {{1, 0}, {0, 0}, {1, 0}, {0, 0}, {1, 0}, {0, 0}, {1, 0}, {0, 0}};
        CHECK(pack_signed_mantissas(s8, 0) == std::vector<std::uint8_t>{0xAA});
        const std::vector<SignedMantissa> s2 = {{0, 0b101}, {1, 0b001}};
        CHECK(pack_signed_mantissas(s2, 3) == std::vector<std::uint8_t>{0x59});
        CHECK(unpack_signed_mantissas(pack_signed_mantissas(s2, 3), 3, 2) == s2);
        CHECK(throws<std::invalid_argument>([] { (void)pack_signed_mantissas(std::vector<SignedMantissa>{{0, 2}}, 1); }));
        CHECK(throws<std::invalid_argument>([] { (void)unpack_signed_mantissas({}, 3, 5); }));
    }
    // --- ans (test_ans.cpp) ----------------------------------------------
    {
        std::vector<std::uint64_t> c(256, 0);
        c[42] = 4096;
        CHECK(build_table(c).freq(42) == 4096);
        CHECK(build_table(std::vector<std::uint64_t>(256, 1000)).freq(7) == 16);
        c.assign(256, 0);
        c[0] = 3;
        c[1] = 1;
        CHECK(build_table(c).freq(0) == 3072 && build_table(c).freq(1) == 1024);
        CHECK(throws<std::invalid_argument>([] { (void)build_table(std::vector<std::uint64_t>(256, 0)); }));
        c.assign(256, 0);
        c[0] = 4095;
        c[1] = 1;
        const auto tb = serialize_table(build_table(c));
        CHECK(tb[0] == 0xFF && tb[1] == 0x0F && tb[2] == 0x01 && tb[3] == 0x00);
        std::vector<std::uint8_t> bad(512, 0);
        bad[0] = 1;
        CHECK(throws<FormatError>([&] { (void)deserialize_table(bad); }));

        std::mt19937_64 gen(8);
        std::vector<double> w(256);
        for (int s = 0; s < 256; ++s) w[s] = 1.0 / (1.0 + s);
        std::discrete_distribution<int> zipf(w.begin(), w.end());
        for (std::size_t n : {std::size_t{0}, std::size_t{1}, std::size_t{999}, std::size_t{65536}, std::size_t{65537},
                              std::size_t{200000}}) {
            std::vector<std::uint8_t> xs(n);
            for (auto& x : xs) x = static_cast<std::uint8_t>(zipf(gen));
            auto cnt = counts_of(xs);
            if (n == 0) cnt[0] = 1;
            const FrequencyTable t = build_table(cnt);
            const AnsStream s = ans_encode(xs, t);
            CHECK(s.chunks.size() == (n + 65535) / 65536);
            CHECK(ans_decode(s) == xs);
            const auto bytes = serialize_stream(s);
            CHECK(bytes.size() == s.stream_bytes());
            CHECK(deserialize_stream(bytes, t).chunks == s.chunks);
            if (s.chunks.size() > 1) {
                const std::size_t len1 = std::min<std::size_t>(65536, n - 65536);
                const auto mid = ans_decode_chunk(s.chunks[1], t);
                CHECK(mid.size() == len1 && std::equal(mid.begin(), mid.end(), xs.begin() + 65536));
                CHECK(ans_encode_chunk(std::span(xs).subspan(65536, len1), t) == s.chunks[1]);
            }
        }
        // errors (test_ans.cpp:231-257)
        c.assign(256, 0);
        c[1] = 10;
        const FrequencyTable one = build_table(c);
        CHECK(throws<std::invalid_argument>([&] { (void)ans_encode(std::vector<std::uint8_t>{1, 2, 1}, one); }));
        std::vector<std::uint8_t> xs(5000);
        for (auto& x : xs) x = static_cast<std::uint8_t>(gen());
        const FrequencyTable t = build_table(counts_of(xs));
        AnsStream s = ans_encode(xs, t);
        s.chunks[0].payload.back() ^= 0x01;
        CHECK(throws<FormatError>([&] { (void)ans_decode(s); }));
        AnsStream tr = ans_encode(xs, t);
        tr.chunks[0].payload.resize(tr.chunks[0].payload.size() - 5);
        CHECK(throws<FormatError>([&] { (void)ans_decode(tr); }));
        const auto framed = serialize_stream(ans_encode(xs, t));
        auto trailing = framed;
        trailing.push_back(0);
        CHECK(throws<FormatError>([&] { (void)deserialize_stream(trailing, t); }));
    }
    // --- tensorstore (test_tensorstore.cpp, acceptance.cpp) -----------------
    {
        std::vector<Bf16> all(65536);
        for (std::uint32_t b = 0; b < 65536; ++b) all[b] = Bf16{static_cast<std::uint16_t>(b)};
        CHECK(decompress_lossless(compress_lossless(all)) == all);

        const std::vector<Bf16> ones(16, Bf16{0x3F80});
        const LosslessBlob c16 = compress_lossless(ones, TensorMeta{{16}});
        CHECK(serialize_stream(c16.exp_stream) ==
              (std::vector<std::uint8_t>{1, 0, 0, 0, 16, 0, 0, 0, 4, 0, 0, 0, 0, 0, 0x80, 0}));
        CHECK(footprint(c16).total() == 587);  // the golden const16_k7.nzt size
        CHECK(decompress_lossless(c16) == ones);

        const auto g = gaussian(42, 4096 * 4096, 0.02);
        const LosslessBlob big = compress_lossless(g, TensorMeta{{4096, 4096}});
        CHECK(big.exp_stream.stream_bytes() == 5347963);
        CHECK(std::fabs(2.0 * g.size() / footprint(big).total() - 1.5165336) < 1e-6);
        CHECK(!big.gpu_index.empty());
        CHECK(decompress_lossless(big) == g);
        LosslessBlob no_index = big;  // as if the stream came from the reference
        no_index.gpu_index.clear();
        CHECK(decompress_lossless(no_index) == g);
        {  // buffer-reuse extension: same values, twice into one vector
            std::vector<Bf16> reuse(17, Bf16{0x1234});
            decompress_lossless_into(big, reuse);
            CHECK(reuse == g);
            std::fill(reuse.begin(), reuse.end(), Bf16{0});
            decompress_lossless_into(big, reuse);
            CHECK(reuse == g);
            LosslessBlob stale = big;  // index from another tensor: FormatError, never a wrong decode
            stale.gpu_index[56 + 4 * 1000] ^= 0x5A;
            CHECK(throws<FormatError>([&] { decompress_lossless_into(stale, reuse); }));
            const LossyBlob lb3 = compress_lossy(g, 3, 512);
            std::vector<Bf16> lossy_into;
            decompress_lossy_into(lb3, lossy_into);
            CHECK(lossy_into == decompress_lossy(lb3));
            // sliced host pipeline (4 Mi-element slices) against whole-tensor
            // staging: slice-aligned blocks (B = 512, 64), and B = 1000 / 3,
            // which no slice size divides (one slice)
            const std::span<const Bf16> part = std::span(g).first(9'000'001);
            for (int k : {0, 1, 3}) {
                for (std::uint32_t B : {512u, 64u, 1000u, 3u}) {
                    const LossyBlob lb = compress_lossy(part, k, B);
                    const auto want = via_batch_path(lb);
                    CHECK(want.size() == part.size() && decompress_lossy(lb) == want);
                }
            }
            // one slice (no slice size divides B = 999) whose 33.5 MB output
            // streams through the 32 MB ring slots in two pieces
            const LossyBlob lbig = compress_lossy(g, 3, 999);
            CHECK(decompress_lossy(lbig) == via_batch_path(lbig));
            const LosslessBlob odd = compress_lossless(part);
            CHECK(decompress_lossless(odd) == std::vector<Bf16>(part.begin(), part.end()));
            // the sliced pipeline writes exactly n values: a guard band after
            // them stays untouched (lossless and lossy k=0)
            const LossyBlob lk0 = compress_lossy(part, 0, 512);
            for (int lossy : {0, 1}) {
                std::vector<Bf16> buf(part.size() + 4096, Bf16{0x5A5A});
                if (lossy)
                    detail::gpu_decompress_into(lk0.meta, lk0.exp_stream, lk0.signmant, lk0.precision, lk0.block_size,
                                                &lk0.scales, lk0.gpu_index, buf.data());
                else
                    detail::gpu_decompress_into(odd.meta, odd.exp_stream, odd.signmant, kLosslessPrecision, 0, nullptr,
                                                odd.gpu_index, buf.data());
                const std::vector<Bf16> want = lossy ? decompress_lossy(lk0) : std::vector<Bf16>(part.begin(), part.end());
                CHECK(std::equal(want.begin(), want.end(), buf.begin()));
                CHECK(std::all_of(buf.begin() + part.size(), buf.end(), [](Bf16 x) { return x.bits == 0x5A5A; }));
            }
        }

        LosslessBlob bad_meta = compress_lossless(std::span(g).first(1000));
        bad_meta.meta.shape = {999};
        CHECK(throws<FormatError>([&] { (void)decompress_lossless(bad_meta); }));
        LosslessBlob corrupt = compress_lossless(std::span(g).first(1000));
        corrupt.exp_stream.chunks[0].payload.back() ^= 0x10;
        CHECK(throws<FormatError>([&] { (void)decompress_lossless(corrupt); }));

        // lossy (test_tensorstore.cpp:104-215)
        const std::vector<Bf16> two = {Bf16::from_float(1.0f), Bf16::from_float(0.5f)};
        for (int k : {0, 1, 3}) {
            const LossyBlob b = compress_lossy(two, k, 512);
            CHECK(b.scales == std::vector<std::uint8_t>{0});
            CHECK(decompress_lossy(b) == two);
        }
        const std::vector<Bf16> m = {Bf16::from_float(-1.75f), Bf16::from_float(0.3f)};
        const LossyBlob lb = compress_lossy(m, 0, 512);
        CHECK(lb.scales == std::vector<std::uint8_t>{96});
        CHECK(decompress_lossy(lb)[0] == m[0]);
        const auto sample = gaussian(7, 100000, 0.02);
        for (int k : {0, 1, 3}) {
            const LossyBlob b = compress_lossy(sample, k, 512);
            const auto back = decompress_lossy(b);
            double worst = 0;
            for (std::size_t i = 0; i < sample.size(); ++i) {
                if (split(sample[i]).exponent == 0) continue;
                worst = std::max(worst, std::fabs(back[i].to_double() - sample[i].to_double()) /
                                            std::fabs(sample[i].to_double()));
            }
            CHECK(worst <= std::pow(2.0, -k) + std::pow(2.0, -7));
        }
        CHECK(decompress_lossy(compress_lossy(std::span(sample).first(1000), 3, 1)) ==
              std::vector<Bf16>(sample.begin(), sample.begin() + 1000));
        CHECK(throws<NonFiniteError>([] { (void)compress_lossy(std::vector<Bf16>{Bf16{0x3F80}, Bf16{0x7FC1}}, 3, 512); }));
        CHECK(throws<std::invalid_argument>([] { (void)compress_lossy(std::vector<Bf16>{Bf16{0x3F80}}, 2, 512); }));
        CHECK(throws<std::invalid_argument>([] { (void)compress_lossy(std::vector<Bf16>{Bf16{0x3F80}}, 3, 0); }));
        CHECK(throws<std::invalid_argument>([] { (void)compress_lossless(std::vector<Bf16>{}); }));
    }
    {  // crc32.hpp + NZT/BFT containers (tensorstore.hpp:289-517)
        const std::string chk = "123456789";
        CHECK(crc32(std::span(reinterpret_cast<const std::uint8_t*>(chk.data()), chk.size())) == 0xCBF43926u);
        Crc32 inc;  // incremental updates join to the one-shot value
        inc.update(std::span(reinterpret_cast<const std::uint8_t*>(chk.data()), 4));
        inc.update(std::span(reinterpret_cast<const std::uint8_t*>(chk.data()) + 4, 5));
        CHECK(inc.value() == 0xCBF43926u);
        CHECK(Crc32{}.value() == 0u);
        // const16_k7.nzt (gen_golden.cpp:34-41): 587 bytes, CRC ec9e894f
        const LosslessBlob c16 = compress_lossless(std::vector<Bf16>(16, Bf16{0x3F80}));
        std::ostringstream os(std::ios::binary);
        write_nzt(Blob(c16), os);
        const std::string file = os.str();
        CHECK(file.size() == 587);
        CHECK(static_cast<std::uint8_t>(file[583]) == 0xEC && static_cast<std::uint8_t>(file[586]) == 0x4F);
        std::istringstream is(file, std::ios::binary);
        const Blob back = read_nzt(is);
        CHECK(decompress_lossless(std::get<LosslessBlob>(back)) == std::vector<Bf16>(16, Bf16{0x3F80}));
        const auto g = gaussian(11, 70000, 0.02);
        for (int k : {7, 3, 0}) {
            std::ostringstream o2(std::ios::binary);
            const TensorMeta meta{{700, 100}};
            if (k == 7) write_nzt(compress_lossless(g, meta), o2);
            else write_nzt(compress_lossy(g, k, 64, meta), o2);
            std::string f2 = o2.str();
            std::istringstream i2(f2 + "tail", std::ios::binary);  // a reader stops at the file's end
            const Blob b2 = read_nzt(i2);
            std::string rest;
            i2 >> rest;
            CHECK(rest == "tail");
            if (k == 7) CHECK(decompress_lossless(std::get<LosslessBlob>(b2)) == g);
            else CHECK(std::get<LossyBlob>(b2).meta == meta && std::get<LossyBlob>(b2).block_size == 64);
            f2[f2.size() / 2] ^= 0x20;  // payload byte -> ChecksumError
            CHECK(throws<ChecksumError>([&] {
                std::istringstream i3(f2, std::ios::binary);
                (void)read_nzt(i3);
            }));
            CHECK(throws<FormatError>([&] {
                std::istringstream i4(f2.substr(0, 100), std::ios::binary);
                (void)read_nzt(i4);
            }));
        }
        CHECK(throws<FormatError>([] {
            std::istringstream i5(std::string("NZT2xxxxxxxxxx"), std::ios::binary);
            (void)read_nzt(i5);
        }));
        Tensor t{TensorMeta{{2, 3}}, {Bf16{1}, Bf16{2}, Bf16{3}, Bf16{0x8000}, Bf16{0x7F80}, Bf16{0xFFFF}}};
        std::ostringstream ob(std::ios::binary);
        write_bft(t, ob);
        CHECK(ob.str().size() == 4 + 1 + 16 + 12);
        std::istringstream ib(ob.str(), std::ios::binary);
        const Tensor tb = read_bft(ib);
        CHECK(tb.meta == t.meta && tb.values == t.values);
    }
    {  // entropy.hpp: GPU histogram, host entropy arithmetic (gen_golden.cpp:22-33 values)
        const auto g = gaussian(42, 1 << 20, 0.02);
        const ComponentHistogram h = build_histogram(g);
        ComponentHistogram cpu;
        for (Bf16 v : g) cpu.add(v);
        CHECK(h.sign_counts == cpu.sign_counts && h.exp_counts == cpu.exp_counts && h.mant_counts == cpu.mant_counts &&
              h.total == cpu.total);
        const EntropyReport r = analyze_tensor(g);
        const EntropyReport rc = report_from_histogram(cpu);
        CHECK(r.h_sign == rc.h_sign && r.h_exp == rc.h_exp && r.h_mant == rc.h_mant && r.ideal_ratio == rc.ideal_ratio);
        CHECK(throws<std::invalid_argument>([] { (void)analyze_tensor(std::vector<Bf16>{}); }));
    }
    std::printf("dropin_test: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
