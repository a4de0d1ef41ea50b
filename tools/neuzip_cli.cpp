// neuzip (B200): the reference CLI's codec commands (proj/tools/neuzip.cpp:
// analyze, compress, decompress, bench) on the drop-in API of include/neuzip,
// i.e. on the GPU codec.  Same arguments, CSV output (6 significant digits)
// and exit codes: 0 success, 2 bad arguments or malformed input, 3 NaN/Inf
// on the lossy path, 4 checksum failure, 1 anything else.  train-demo and
// perturb-grid belong to the reference's CPU training harness and are not
// provided.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "neuzip/neuzip.hpp"

namespace {

constexpr int kExitUsage = 2, kExitNonFinite = 3, kExitChecksum = 4;

std::string fmt6(double v) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.6g", v);
    return buf;
}

struct Usage : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

neuzip::Tensor load_bft(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw neuzip::FormatError("cannot open " + path);
    return neuzip::read_bft(in);
}

int cmd_analyze(const std::string& input, bool hist) {
    const neuzip::Tensor tensor = load_bft(input);
    if (tensor.values.empty()) throw neuzip::FormatError("analyze: empty tensor");
    const neuzip::ComponentHistogram h = neuzip::build_histogram(tensor.values);
    const neuzip::EntropyReport r = neuzip::report_from_histogram(h);
    std::cout << "component,entropy_bits,capacity_bits\n";
    std::cout << "sign," << fmt6(r.h_sign) << ",1\n";
    std::cout << "exponent," << fmt6(r.h_exp) << ",8\n";
    std::cout << "mantissa," << fmt6(r.h_mant) << ",7\n";
    std::cout << "ideal_ratio," << fmt6(r.ideal_ratio) << ",\n";
    std::cout << "exponent_only_ratio," << fmt6(r.exponent_only_ratio) << ",\n";
    if (hist) {
        for (std::size_t i = 0; i < h.sign_counts.size(); ++i) std::cout << "hist_sign_" << i << ',' << h.sign_counts[i] << ",\n";
        for (std::size_t i = 0; i < h.exp_counts.size(); ++i) std::cout << "hist_exp_" << i << ',' << h.exp_counts[i] << ",\n";
        for (std::size_t i = 0; i < h.mant_counts.size(); ++i) std::cout << "hist_mant_" << i << ',' << h.mant_counts[i] << ",\n";
    }
    return 0;
}

void print_footprint(const neuzip::Footprint& f, std::uint64_t raw) {
    std::cout << "section,bytes\n";
    std::cout << "exponent," << f.exponent_bytes << '\n';
    std::cout << "mantissa," << f.mantissa_bytes << '\n';
    std::cout << "scales," << f.scale_bytes << '\n';
    std::cout << "table," << f.table_bytes << '\n';
    std::cout << "header," << f.header_bytes << '\n';
    std::cout << "total," << f.total() << '\n';
    std::cout << "raw," << raw << '\n';
    std::cout << "ratio," << fmt6(static_cast<double>(raw) / static_cast<double>(f.total())) << '\n';
}

int cmd_compress(const std::string& input, const std::string& output, int precision, std::uint32_t block) {
    const neuzip::Tensor t = load_bft(input);
    const neuzip::Blob blob = precision == neuzip::kLosslessPrecision
                                  ? neuzip::Blob(neuzip::compress_lossless(t.values, t.meta))
                                  : neuzip::Blob(neuzip::compress_lossy(t.values, precision, block, t.meta));
    std::ofstream out(output, std::ios::binary);
    if (!out) throw neuzip::Error("cannot open " + output);
    neuzip::write_nzt(blob, out);
    print_footprint(neuzip::footprint(blob), t.values.size() * 2);
    return 0;
}

int cmd_decompress(const std::string& input, const std::string& output) {
    std::ifstream in(input, std::ios::binary);
    if (!in) throw neuzip::FormatError("cannot open " + input);
    const neuzip::Blob blob = neuzip::read_nzt(in);
    neuzip::Tensor t;
    if (const auto* l = std::get_if<neuzip::LosslessBlob>(&blob)) {
        t.meta = l->meta;
        t.values = neuzip::decompress_lossless(*l);
    } else {
        const auto& y = std::get<neuzip::LossyBlob>(blob);
        t.meta = y.meta;
        t.values = neuzip::decompress_lossy(y);
    }
    std::ofstream out(output, std::ios::binary);
    if (!out) throw neuzip::Error("cannot open " + output);
    neuzip::write_bft(t, out);
    return 0;
}

// N(0, sigma^2) bf16 by Box-Muller over a splitmix64 counter stream (input
// synthesis for the bench only).
std::vector<neuzip::Bf16> gaussian(std::uint64_t seed, std::size_t n, double sigma) {
    auto word = [seed](std::uint64_t i) {
        std::uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    std::vector<neuzip::Bf16> v(n);
    for (std::size_t i = 0; i < n; i += 2) {
        const double u1 = ((word(i) >> 11) + 1.0) * 0x1.0p-53, u2 = (word(i + 1) >> 11) * 0x1.0p-53;
        const double r = sigma * std::sqrt(-2.0 * std::log(u1));
        v[i] = neuzip::Bf16::from_float(static_cast<float>(r * std::cos(2 * M_PI * u2)));
        if (i + 1 < n) v[i + 1] = neuzip::Bf16::from_float(static_cast<float>(r * std::sin(2 * M_PI * u2)));
    }
    return v;
}

int cmd_bench(const std::vector<std::uint64_t>& sizes, int trials, std::uint64_t seed) {
    using clock = std::chrono::steady_clock;
    for (std::uint64_t s : sizes)
        if (s < 4096) throw std::invalid_argument("bench: sizes must be >= 4096");
    if (trials < 1) throw std::invalid_argument("bench: trials must be >= 1");
    std::cout << "direction,size_bytes,gib_per_s\n";
    for (std::uint64_t size : sizes) {
        const std::vector<neuzip::Bf16> data = gaussian(seed, size / 2, 0.02);
        std::vector<double> cs(trials), ds(trials);
        for (int t = 0; t < trials; ++t) {
            const auto t0 = clock::now();
            const neuzip::LosslessBlob blob = neuzip::compress_lossless(data);
            const auto t1 = clock::now();
            const std::vector<neuzip::Bf16> back = neuzip::decompress_lossless(blob);
            const auto t2 = clock::now();
            if (back != data) throw neuzip::Error("bench: round trip mismatch");
            cs[t] = std::chrono::duration<double>(t1 - t0).count();
            ds[t] = std::chrono::duration<double>(t2 - t1).count();
        }
        auto median = [](std::vector<double> v) {
            std::sort(v.begin(), v.end());
            return v[v.size() / 2];
        };
        const double gib = static_cast<double>(size) / (1024.0 * 1024.0 * 1024.0);
        std::cout << "compress," << size << ',' << fmt6(gib / median(cs)) << '\n';
        std::cout << "decompress," << size << ',' << fmt6(gib / median(ds)) << '\n';
    }
    return 0;
}

std::vector<std::uint64_t> parse_list(const std::string& s) {
    std::vector<std::uint64_t> out;
    std::size_t p = 0;
    while (p < s.size()) {
        const std::size_t q = s.find(',', p);
        out.push_back(std::stoull(s.substr(p, q == std::string::npos ? std::string::npos : q - p)));
        if (q == std::string::npos) break;
        p = q + 1;
    }
    return out;
}

int usage() {
    std::cerr << "usage: neuzip analyze <input.bft> [--hist]\n"
                 "       neuzip compress <input.bft> <output.nzt> [-p|--precision 0|1|3|7] [--block-size B]\n"
                 "       neuzip decompress <input.nzt> <output.bft>\n"
                 "       neuzip bench [--sizes a,b,...] [--trials T] [--seed S]\n";
    return kExitUsage;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    std::vector<std::string> pos;
    bool hist = false;
    int precision = neuzip::kLosslessPrecision, trials = 5;
    std::uint32_t block = neuzip::kDefaultBlockSize;
    std::uint64_t seed = 42;
    std::vector<std::uint64_t> sizes = {100000, 1000000, 10000000, 100000000};
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto val = [&]() -> std::string {
                if (i + 1 >= argc) throw Usage("missing value for " + a);
                return argv[++i];
            };
            if (a == "--hist") hist = true;
            else if (a == "-p" || a == "--precision") precision = std::stoi(val());
            else if (a == "--block-size") block = static_cast<std::uint32_t>(std::stoul(val()));
            else if (a == "--sizes") sizes = parse_list(val());
            else if (a == "--trials") trials = std::stoi(val());
            else if (a == "--seed") seed = std::stoull(val());
            else if (!a.empty() && a[0] == '-') throw Usage("unknown option " + a);
            else pos.push_back(a);
        }
        if (precision != 0 && precision != 1 && precision != 3 && precision != 7) throw Usage("precision");
        if (block == 0) throw Usage("block size");
        if (cmd == "analyze" && pos.size() == 1) return cmd_analyze(pos[0], hist);
        if (cmd == "compress" && pos.size() == 2) return cmd_compress(pos[0], pos[1], precision, block);
        if (cmd == "decompress" && pos.size() == 2) return cmd_decompress(pos[0], pos[1]);
        if (cmd == "bench" && pos.empty()) return cmd_bench(sizes, trials, seed);
        return usage();
    } catch (const Usage& e) {
        std::cerr << "error: " << e.what() << '\n';
        return usage();
    } catch (const neuzip::ChecksumError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitChecksum;
    } catch (const neuzip::NonFiniteError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitNonFinite;
    } catch (const neuzip::FormatError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
