// neuzip -- command-line front end of the B200 codec.
//
// Offers the codec subcommands of the reference tool (proj/tools/neuzip.cpp:
// analyze, compress, decompress, bench) with the same positional arguments,
// options, CSV columns (floats as %.6g) and exit codes, so scripts written
// against the reference keep working:
//     0 ok, 1 other error, 2 usage / malformed input, 3 NaN/Inf on the lossy
//     path, 4 NZT checksum failure.
// The work is done on the GPU through the C ABI (include/nzgpu.h): files are
// read whole, tensors are compressed / decoded by device blobs, the NZT CRC
// is computed on the GPU.  `bench` times the drop-in host API
// (include/neuzip/tensorstore.hpp), i.e. what a C++ caller of
// compress_lossless / decompress_lossless gets.  train-demo and perturb-grid
// drive the reference's CPU training harness, which is not part of the codec
// path; they exit 2 with a pointer to INTEGRATION.md.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <iterator>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "neuzip/neuzip.hpp"
#include "nzgpu.h"

namespace {

// ------------------------------------------------------------------ errors --
enum ExitCode : int { kExitOk = 0, kExitOther = 1, kExitUsage = 2, kExitNonFinite = 3, kExitChecksum = 4 };

struct CliError {
    int code;
    std::string message;
};

[[noreturn]] void fail(int code, std::string message) { throw CliError{code, std::move(message)}; }

int exit_code_of(int status) {
    switch (status) {
        case NZGPU_CHECKSUM: return kExitChecksum;
        case NZGPU_NONFINITE: return kExitNonFinite;
        case NZGPU_INVALID_ARGUMENT:
        case NZGPU_FORMAT_TRUNCATED:
        case NZGPU_FORMAT_DESYNC:
        case NZGPU_FORMAT_LENGTH:
        case NZGPU_FORMAT_TABLE: return kExitUsage;
        default: return kExitOther;
    }
}

void nz(int status, const std::string& what) {
    if (status == NZGPU_OK) return;
    std::string msg = what + ": " + nzgpu_status_string(status);
    const char* detail = nzgpu_last_error_message();
    if (status == NZGPU_CUDA_ERROR && detail && *detail) msg += std::string(" (") + detail + ")";
    fail(exit_code_of(status), msg);
}

struct BlobHandle {
    nzgpu_blob h = nullptr;
    ~BlobHandle() {
        if (h) nzgpu_blob_free(h);
    }
};

// ---------------------------------------------------------------- arguments --
// Positional words plus --name value / --name=value / -x value options and
// bare flags.  Each subcommand declares what it accepts.
struct Args {
    std::vector<std::string> words;
    std::map<std::string, std::string> values;
    std::vector<std::string> flags;

    bool flag(const std::string& name) const { return std::find(flags.begin(), flags.end(), name) != flags.end(); }
    std::optional<std::string> get(const std::string& name) const {
        const auto it = values.find(name);
        if (it == values.end()) return std::nullopt;
        return it->second;
    }
};

struct OptionSpec {
    std::vector<std::string> spellings;  // first one is the canonical name
    bool takes_value;
};

Args parse_args(int argc, char** argv, int first, const std::vector<OptionSpec>& spec) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string w = argv[i];
        if (w.size() < 2 || w[0] != '-') {
            a.words.push_back(w);
            continue;
        }
        std::string inline_value;
        bool has_inline = false;
        if (const auto eq = w.find('='); eq != std::string::npos && w.rfind("--", 0) == 0) {
            inline_value = w.substr(eq + 1);
            w = w.substr(0, eq);
            has_inline = true;
        }
        const OptionSpec* match = nullptr;
        for (const OptionSpec& o : spec)
            if (std::find(o.spellings.begin(), o.spellings.end(), w) != o.spellings.end()) match = &o;
        if (!match) fail(kExitUsage, "unknown option " + w);
        const std::string& name = match->spellings.front();
        if (!match->takes_value) {
            if (has_inline) fail(kExitUsage, "option " + w + " takes no value");
            a.flags.push_back(name);
        } else if (has_inline) {
            a.values[name] = inline_value;
        } else {
            if (i + 1 >= argc) fail(kExitUsage, "option " + w + " needs a value");
            a.values[name] = argv[++i];
        }
    }
    return a;
}

std::uint64_t parse_u64(const std::string& s, const std::string& what) {
    if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos) fail(kExitUsage, what + ": not a number: " + s);
    errno = 0;
    const unsigned long long v = std::strtoull(s.c_str(), nullptr, 10);
    if (errno) fail(kExitUsage, what + ": out of range: " + s);
    return v;
}

std::vector<std::uint64_t> parse_u64_list(const std::string& s, const std::string& what) {
    std::vector<std::uint64_t> out;
    std::stringstream ss(s);
    for (std::string item; std::getline(ss, item, ',');) out.push_back(parse_u64(item, what));
    if (out.empty()) fail(kExitUsage, what + ": empty list");
    return out;
}

// ------------------------------------------------------------------- output --
std::string g6(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.6g", v);
    return b;
}

// CSV assembled in memory and written once.
class Csv {
public:
    explicit Csv(std::initializer_list<std::string> header) { row(header); }
    void row(std::initializer_list<std::string> cells) {
        bool first = true;
        for (const std::string& c : cells) {
            if (!first) text_ += ',';
            text_ += c;
            first = false;
        }
        text_ += '\n';
    }
    void print() const { std::fwrite(text_.data(), 1, text_.size(), stdout); }

private:
    std::string text_;
};

// -------------------------------------------------------------------- files --
std::vector<std::uint8_t> slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(kExitUsage, "cannot open " + path);
    in.seekg(0, std::ios::end);
    const std::streamoff size = in.tellg();
    in.seekg(0);
    std::vector<std::uint8_t> data(static_cast<std::size_t>(std::max<std::streamoff>(size, 0)));
    in.read(reinterpret_cast<char*>(data.data()), static_cast<std::streamsize>(data.size()));
    if (!in) fail(kExitUsage, "cannot read " + path);
    return data;
}

void spill(const std::string& path, const std::vector<std::uint8_t>& head, const void* body, std::size_t body_len) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) fail(kExitOther, "cannot open " + path);
    out.write(reinterpret_cast<const char*>(head.data()), static_cast<std::streamsize>(head.size()));
    out.write(static_cast<const char*>(body), static_cast<std::streamsize>(body_len));
    if (!out) fail(kExitOther, "cannot write " + path);
}

std::uint64_t le(const std::uint8_t* p, int bytes) {
    std::uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

// A BFT raw tensor (tensorstore.hpp:479-517): "BFT1", u8 rank, u64 dims, then
// the bf16 bit patterns little-endian (x86 / aarch64 hosts are little-endian,
// so the payload is copied as is).
struct BftFile {
    std::vector<std::uint16_t> data;
    std::vector<std::uint64_t> shape;
    std::uint64_t n = 0;
    const std::uint16_t* values() const { return data.data(); }
};

BftFile load_bft(const std::string& path) {
    BftFile f;
    const std::vector<std::uint8_t> b = slurp(path);
    if (b.size() < 5 || std::memcmp(b.data(), "BFT1", 4) != 0) fail(kExitUsage, "bft: bad magic");
    const unsigned rank = b[4];
    if (rank == 0 || rank > 8) fail(kExitUsage, "bft: invalid rank");
    if (b.size() < 5 + 8ull * rank) fail(kExitUsage, "bft: truncated");
    f.n = 1;
    for (unsigned i = 0; i < rank; ++i) {
        const std::uint64_t d = le(b.data() + 5 + 8 * i, 8);
        if (d == 0) fail(kExitUsage, "bft: zero dimension");
        if (d > (std::uint64_t{1} << 40) / f.n) fail(kExitUsage, "bft: element count overflow");
        f.shape.push_back(d);
        f.n *= d;
    }
    if (b.size() < 5 + 8ull * rank + 2 * f.n) fail(kExitUsage, "bft: truncated payload");
    f.data.resize(f.n);
    std::memcpy(f.data.data(), b.data() + 5 + 8 * rank, 2 * f.n);
    return f;
}

std::vector<std::uint8_t> bft_header(const std::vector<std::uint64_t>& shape) {
    std::vector<std::uint8_t> h = {'B', 'F', 'T', '1', static_cast<std::uint8_t>(shape.size())};
    for (std::uint64_t d : shape)
        for (int i = 0; i < 8; ++i) h.push_back(static_cast<std::uint8_t>(d >> (8 * i)));
    return h;
}

// ----------------------------------------------------------------- commands --
int run_analyze(const Args& a) {
    if (a.words.size() != 1) fail(kExitUsage, "analyze: expected <input.bft>");
    const BftFile t = load_bft(a.words[0]);
    std::vector<std::uint64_t> counts(386);  // sign[2] | exponent[256] | mantissa[128]
    nz(nzgpu_component_histogram_host(t.values(), t.n, counts.data()), "analyze");
    double rep[5];  // h_sign, h_exp, h_mant, ideal_ratio, exponent_only_ratio (entropy.hpp:57-81)
    nz(nzgpu_entropy_from_histogram(counts.data(), rep), "analyze");
    Csv csv{"component", "entropy_bits", "capacity_bits"};
    csv.row({"sign", g6(rep[0]), "1"});
    csv.row({"exponent", g6(rep[1]), "8"});
    csv.row({"mantissa", g6(rep[2]), "7"});
    csv.row({"ideal_ratio", g6(rep[3]), ""});
    csv.row({"exponent_only_ratio", g6(rep[4]), ""});
    if (a.flag("--hist")) {
        const struct {
            const char* name;
            int first, bins;
        } groups[] = {{"hist_sign_", 0, 2}, {"hist_exp_", 2, 256}, {"hist_mant_", 258, 128}};
        for (const auto& g : groups)
            for (int i = 0; i < g.bins; ++i) csv.row({g.name + std::to_string(i), std::to_string(counts[g.first + i]), ""});
    }
    csv.print();
    return kExitOk;
}

int run_compress(const Args& a) {
    if (a.words.size() != 2) fail(kExitUsage, "compress: expected <input.bft> <output.nzt>");
    const int precision = static_cast<int>(parse_u64(a.get("--precision").value_or("7"), "--precision"));
    if (precision != 0 && precision != 1 && precision != 3 && precision != 7)
        fail(kExitUsage, "--precision: must be one of 0, 1, 3, 7");
    const std::uint64_t block = parse_u64(a.get("--block-size").value_or("512"), "--block-size");
    if (block == 0 || block > 0xFFFFFFFFull) fail(kExitUsage, "--block-size: must be a positive 32-bit number");
    const BftFile t = load_bft(a.words[0]);
    BlobHandle blob;
    nz(nzgpu_compress_host(t.values(), t.n, precision, precision == 7 ? 0u : static_cast<std::uint32_t>(block), 0, 0,
                           &blob.h),
       precision == 7 ? "compress_lossless" : "compress_lossy");
    std::uint64_t size = 0, written = 0;
    nz(nzgpu_blob_nzt_size(blob.h, static_cast<int>(t.shape.size()), &size), "write_nzt");
    std::vector<std::uint8_t> file(size);
    nz(nzgpu_blob_write_nzt(blob.h, t.shape.data(), static_cast<int>(t.shape.size()), file.data(), size, &written),
       "write_nzt");
    spill(a.words[1], {}, file.data(), written);
    // footprint() (tensorstore.hpp:242-287): the NZT file is exactly its total
    nzgpu_blob_info info{};
    nz(nzgpu_blob_info_get(blob.h, &info), "blob info");
    const std::uint64_t header = 35 + 8 * t.shape.size(), raw = 2 * t.n;
    const std::uint64_t total = info.stream_len + info.mantissa_len + info.scales_len + 512 + header;
    Csv csv{"section", "bytes"};
    csv.row({"exponent", std::to_string(info.stream_len)});
    csv.row({"mantissa", std::to_string(info.mantissa_len)});
    csv.row({"scales", std::to_string(info.scales_len)});
    csv.row({"table", "512"});
    csv.row({"header", std::to_string(header)});
    csv.row({"total", std::to_string(total)});
    csv.row({"raw", std::to_string(raw)});
    csv.row({"ratio", g6(static_cast<double>(raw) / static_cast<double>(total))});
    csv.print();
    return kExitOk;
}

int run_decompress(const Args& a) {
    if (a.words.size() != 2) fail(kExitUsage, "decompress: expected <input.nzt> <output.bft>");
    const std::vector<std::uint8_t> file = slurp(a.words[0]);
    BlobHandle blob;
    std::uint64_t shape[8] = {};
    int ndim = 0;
    nz(nzgpu_blob_read_nzt(file.data(), file.size(), 0, nullptr, &blob.h, shape, &ndim), "read_nzt");
    nzgpu_blob_info info{};
    nz(nzgpu_blob_info_get(blob.h, &info), "blob info");
    std::vector<std::uint16_t> values(info.n);
    nz(nzgpu_blob_decompress_host(blob.h, values.data()), info.precision == 7 ? "decompress_lossless" : "decompress_lossy");
    spill(a.words[1], bft_header(std::vector<std::uint64_t>(shape, shape + ndim)), values.data(), 2 * values.size());
    return kExitOk;
}

// rng::gaussian_bf16 (rng.hpp:21-81) by its documented recipe: word i of
// stream `seed` is splitmix64(seed + (i+1) * golden); sample i is Box-Muller
// on words 2i and 2i+1, scaled by sigma and rounded to bf16.
std::vector<neuzip::Bf16> synthetic_weights(std::uint64_t seed, std::size_t n, double sigma) {
    auto word = [seed](std::uint64_t counter) {
        std::uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    std::vector<neuzip::Bf16> v(n);
    for (std::size_t i = 0; i < n; ++i) {
        const double u1 = (static_cast<double>(word(2 * i) >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(word(2 * i + 1) >> 11) * 0x1.0p-53;
        const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793238462643383279502884 * u2);
        v[i] = neuzip::Bf16::from_float(static_cast<float>(sigma * g));
    }
    return v;
}

int run_bench(const Args& a) {
    if (!a.words.empty()) fail(kExitUsage, "bench: unexpected argument " + a.words[0]);
    const std::vector<std::uint64_t> sizes =
        parse_u64_list(a.get("--sizes").value_or("100000,1000000,10000000,100000000"), "--sizes");
    const std::uint64_t trials = parse_u64(a.get("--trials").value_or("5"), "--trials");
    const std::uint64_t seed = parse_u64(a.get("--seed").value_or("42"), "--seed");
    if (std::any_of(sizes.begin(), sizes.end(), [](std::uint64_t s) { return s < 4096; }))
        fail(kExitUsage, "bench: sizes must be >= 4096");
    if (trials < 1) fail(kExitUsage, "bench: trials must be >= 1");
    using clock = std::chrono::steady_clock;
    auto seconds = [](clock::time_point a0, clock::time_point a1) { return std::chrono::duration<double>(a1 - a0).count(); };
    auto middle = [](std::vector<double> v) {
        std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
        return v[v.size() / 2];
    };
    Csv csv{"direction", "size_bytes", "gib_per_s"};
    for (const std::uint64_t bytes : sizes) {
        const std::vector<neuzip::Bf16> weights = synthetic_weights(seed, bytes / 2, 0.02);
        std::vector<double> enc, dec;
        for (std::uint64_t r = 0; r < trials; ++r) {
            const auto t0 = clock::now();
            const neuzip::LosslessBlob blob = neuzip::compress_lossless(weights);
            const auto t1 = clock::now();
            const std::vector<neuzip::Bf16> back = neuzip::decompress_lossless(blob);
            const auto t2 = clock::now();
            if (back != weights) fail(kExitOther, "bench: round trip mismatch");
            enc.push_back(seconds(t0, t1));
            dec.push_back(seconds(t1, t2));
        }
        const double gib = static_cast<double>(bytes) / double(1ull << 30);
        csv.row({"compress", std::to_string(bytes), g6(gib / middle(enc))});
        csv.row({"decompress", std::to_string(bytes), g6(gib / middle(dec))});
    }
    csv.print();
    return kExitOk;
}

struct Command {
    const char* name;
    const char* summary;
    std::vector<OptionSpec> options;
    std::function<int(const Args&)> run;
};

const std::vector<Command>& commands() {
    static const std::vector<Command> table = {
        {"analyze", "<input.bft> [--hist]: per-component entropy report", {{{"--hist"}, false}}, run_analyze},
        {"compress",
         "<input.bft> <output.nzt> [-p|--precision 0|1|3|7] [--block-size B]: compress to NZT",
         {{{"--precision", "-p"}, true}, {{"--block-size"}, true}},
         run_compress},
        {"decompress", "<input.nzt> <output.bft>: expand an NZT file", {}, run_decompress},
        {"bench", "[--sizes a,b,..] [--trials T] [--seed S]: drop-in API throughput on Gaussian tensors",
         {{{"--sizes"}, true}, {{"--trials"}, true}, {{"--seed"}, true}},
         run_bench},
    };
    return table;
}

void usage(std::FILE* to) {
    std::fprintf(to, "neuzip (B200): entropy-based BF16 tensor compression\nsubcommands:\n");
    for (const Command& c : commands()) std::fprintf(to, "  %-10s %s\n", c.name, c.summary);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage(stderr);
        return kExitUsage;
    }
    const std::string sub = argv[1];
    if (sub == "-h" || sub == "--help") {
        usage(stdout);
        return kExitOk;
    }
    try {
        for (const Command& c : commands())
            if (sub == c.name) return c.run(parse_args(argc, argv, 2, c.options));
        if (sub == "train-demo" || sub == "perturb-grid")
            fail(kExitUsage, sub + ": the reference's CPU training harness is not part of the codec path "
                                   "(see INTEGRATION.md)");
        fail(kExitUsage, "unknown subcommand " + sub);
    } catch (const CliError& e) {
        std::fprintf(stderr, "error: %s\n", e.message.c_str());
        if (e.code == kExitUsage && e.message.rfind("unknown", 0) == 0) usage(stderr);
        return e.code;
    } catch (const neuzip::ChecksumError& e) {  // from the drop-in API (bench)
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitChecksum;
    } catch (const neuzip::NonFiniteError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitNonFinite;
    } catch (const neuzip::FormatError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitUsage;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitUsage;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitOther;
    }
}
