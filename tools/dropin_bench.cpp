// dropin_bench -- decode throughput of the reference-signature C++ API
// (include/neuzip/tensorstore.hpp) on one Llama-3-8B layer (the 7 projection
// matrices, N(0, 0.02^2) weights by rng.hpp's counter recipe), host buffers
// in and out, PCIe included:
//   fresh   std::vector<Bf16> decompress_lossless(const LosslessBlob&) -- the
//           reference signature: a new, value-initialised vector per call;
//   reused  decompress_lossless_into(blob, vec) into vectors kept across calls.
// Algorithmic bytes per tensor = stream + mantissas + 512 + 2n.
// Prints one JSON object.  Built by _build.py next to the CLI; run by bench.py.
//   usage: dropin_bench [reps]
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>

#include "neuzip/neuzip.hpp"

using namespace neuzip;

namespace {

std::vector<Bf16> weights(std::uint64_t seed, std::size_t n) {
    std::vector<Bf16> v(n);
    auto word = [seed](std::uint64_t c) {
        std::uint64_t z = seed + (c + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < nt; ++t)
        ts.emplace_back([&, t] {
            for (std::size_t i = t; i < n; i += nt) {
                const double u1 = (static_cast<double>(word(2 * i) >> 11) + 1.0) * 0x1.0p-53;
                const double u2 = static_cast<double>(word(2 * i + 1) >> 11) * 0x1.0p-53;
                v[i] = Bf16::from_float(static_cast<float>(
                    0.02 * std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793238462643383279502884 * u2)));
            }
        });
    for (auto& t : ts) t.join();
    return v;
}

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

}  // namespace

int main(int argc, char** argv) {
    const int reps = argc > 1 ? std::max(1, std::atoi(argv[1])) : 3;
    const std::uint64_t h = 4096, f = 14336, kv = 1024;
    const std::vector<std::vector<std::uint64_t>> shapes = {{h, h}, {kv, h}, {kv, h}, {h, h}, {f, h}, {f, h}, {h, f}};
    std::vector<LosslessBlob> blobs;
    std::vector<std::vector<Bf16>> src;
    double algo = 0;
    std::uint64_t elems = 0;
    for (std::size_t i = 0; i < shapes.size(); ++i) {
        TensorMeta meta{shapes[i]};
        src.push_back(weights(1000 + i, meta.element_count()));
        blobs.push_back(compress_lossless(src.back(), meta));
        const Footprint fp = footprint(blobs.back());
        algo += static_cast<double>(fp.exponent_bytes + fp.mantissa_bytes + fp.table_bytes + 2 * meta.element_count());
        elems += meta.element_count();
    }
    // warm-up (staging buffers, library state) + correctness
    for (std::size_t i = 0; i < blobs.size(); ++i)
        if (decompress_lossless(blobs[i]) != src[i]) {
            std::fprintf(stderr, "round trip mismatch\n");
            return 1;
        }
    std::vector<double> fresh, reused;
    std::vector<std::vector<Bf16>> keep(blobs.size());
    for (std::size_t i = 0; i < blobs.size(); ++i) decompress_lossless_into(blobs[i], keep[i]);
    bool ok = true;
    for (int r = 0; r < reps; ++r) {
        double t0 = now();
        for (const LosslessBlob& b : blobs) {
            std::vector<Bf16> v = decompress_lossless(b);
            ok &= v.size() == b.meta.element_count();
        }
        fresh.push_back(now() - t0);
        t0 = now();
        for (std::size_t i = 0; i < blobs.size(); ++i) decompress_lossless_into(blobs[i], keep[i]);
        reused.push_back(now() - t0);
    }
    for (std::size_t i = 0; i < blobs.size(); ++i) ok &= keep[i] == src[i];
    // compress_lossless (the per-layer recompress of nn.hpp:311): host vector
    // in, a LosslessBlob with its AnsStream chunks out
    std::vector<double> comp;
    for (int r = 0; r < reps; ++r) {
        const double t0 = now();
        for (std::size_t i = 0; i < blobs.size(); ++i) {
            LosslessBlob b = compress_lossless(src[i], blobs[i].meta);
            ok &= b.exp_stream.chunks.size() == blobs[i].exp_stream.chunks.size();
        }
        comp.push_back(now() - t0);
    }
    std::sort(comp.begin(), comp.end());
    const double tc = comp[comp.size() / 2];
    std::sort(fresh.begin(), fresh.end());
    std::sort(reused.begin(), reused.end());
    const double tf = fresh[fresh.size() / 2], tr = reused[reused.size() / 2];
    std::printf("{\"ok\": %s, \"elements\": %llu, \"algo_bytes\": %.0f, \"fresh_gbs\": %.2f, \"reused_gbs\": %.2f, "
                "\"fresh_s\": %.4f, \"reused_s\": %.4f, \"compress_gbs\": %.2f, \"compress_s\": %.4f, \"reps\": %d}\n",
                ok ? "true" : "false", static_cast<unsigned long long>(elems), algo, algo / tf / 1e9, algo / tr / 1e9, tf,
                tr, algo / tc / 1e9, tc, reps);
    return ok ? 0 : 1;
}
