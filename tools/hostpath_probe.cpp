// hostpath_probe: host-memory costs that bound the reference-signature host
// API (std::vector in, std::vector out) on the GPU box.  Dev tool, not part
// of the product.  Prints one line per measurement (GB/s of the named bytes).
//
//   g++ -O2 -std=c++20 -pthread tools/hostpath_probe.cpp -I/usr/local/cuda/include \
//       -L/usr/local/cuda/lib64 -lcudart -o build/hostpath_probe
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

struct Bf16 {
    std::uint16_t bits = 0;
};

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void par_copy(void* dst, const void* src, size_t bytes, int threads) {
    std::vector<std::thread> ts;
    const size_t step = (bytes + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const size_t a = t * step, b = std::min(bytes, a + step);
        if (a >= b) break;
        ts.emplace_back([=] { std::memcpy((char*)dst + a, (const char*)src + a, b - a); });
    }
    for (auto& t : ts) t.join();
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 218112000ull;  // one Llama-3-8B layer
    const size_t bytes = n * 2;
    std::printf("n=%zu bytes=%zu hw_threads=%u\n", n, bytes, std::thread::hardware_concurrency());
    for (const char* f : {"/sys/kernel/mm/transparent_hugepage/enabled", "/sys/kernel/mm/transparent_hugepage/defrag"}) {
        if (FILE* fp = std::fopen(f, "r")) {
            char buf[256] = {};
            if (std::fgets(buf, sizeof buf, fp)) std::printf("%s: %s", f, buf);
            std::fclose(fp);
        }
    }
    // fresh-vector strategies: pre-populate the reserved pages (in parallel,
    // optionally as huge pages), then value-initialise
    for (int mode = 0; mode < 6; ++mode) {
        const int threads = mode % 3 == 0 ? 1 : mode % 3 == 1 ? 8 : 16;
        const bool huge = mode >= 3;
        double t0 = now();
        std::vector<Bf16> w;
        w.reserve(n);
        char* p = reinterpret_cast<char*>(w.data());
        if (huge) {
            char* a = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1));
            if (a < p + bytes) madvise(a, (p + bytes - a) & ~size_t((2u << 20) - 1), MADV_HUGEPAGE);
        }
        double t1 = now();
        int rc_pop = 0;
        {
            std::vector<std::thread> ts;
            const size_t step = ((bytes + threads - 1) / threads + 4095) & ~size_t(4095);
            char* base = reinterpret_cast<char*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(4095));
            const size_t span = p + bytes - base;
            std::atomic<int> bad{0};
            for (int t = 0; t < threads; ++t) {
                const size_t a = t * step, b = std::min(span, a + step);
                if (a >= b) break;
                ts.emplace_back([=, &bad] {
                    if (madvise(base + a, b - a, 23 /* MADV_POPULATE_WRITE */)) bad = 1;
                });
            }
            for (auto& t : ts) t.join();
            rc_pop = bad;
        }
        double t2 = now();
        w.resize(n);
        double t3 = now();
        std::printf("fresh vector: threads=%d huge=%d populate_rc=%d reserve+madvise %.1f ms populate %.1f ms "
                    "value-init %.1f ms total %.1f ms (%.1f GB/s)\n", threads, huge, rc_pop, (t1 - t0) * 1e3,
                    (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t3 - t0) * 1e3, bytes / (t3 - t0) / 1e9);
    }
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now();
        std::vector<Bf16> v(n);
        double t1 = now();
        std::printf("vector<Bf16>(n) value-init (fresh pages): %.1f ms  %.1f GB/s\n", (t1 - t0) * 1e3,
                    bytes / (t1 - t0) / 1e9);
        void* pin = nullptr;
        t0 = now();
        cudaMallocHost(&pin, bytes);
        t1 = now();
        std::printf("cudaMallocHost: %.1f ms\n", (t1 - t0) * 1e3);
        void* dev = nullptr;
        cudaMalloc(&dev, bytes);
        cudaMemset(dev, 1, bytes);
        cudaDeviceSynchronize();
        t0 = now();
        cudaMemcpy(pin, dev, bytes, cudaMemcpyDeviceToHost);
        t1 = now();
        std::printf("D2H pinned: %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
        t0 = now();
        cudaMemcpy(dev, pin, bytes, cudaMemcpyHostToDevice);
        t1 = now();
        std::printf("H2D pinned: %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
        t0 = now();
        cudaMemcpy(v.data(), dev, bytes, cudaMemcpyDeviceToHost);
        t1 = now();
        std::printf("D2H pageable (touched): %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
        t0 = now();
        cudaMemcpy(dev, v.data(), bytes, cudaMemcpyHostToDevice);
        t1 = now();
        std::printf("H2D pageable (touched): %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
        {
            std::vector<Bf16> w;
            w.reserve(n);
            t0 = now();
            cudaMemcpy(w.data(), dev, bytes, cudaMemcpyDeviceToHost);
            t1 = now();
            std::printf("D2H pageable (fresh, untouched): %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
        }
        for (int th : {1, 4, 8, 16, 32}) {
            t0 = now();
            par_copy(v.data(), pin, bytes, th);
            t1 = now();
            std::printf("memcpy pinned->touched x%d: %.1f GB/s\n", th, bytes / (t1 - t0) / 1e9);
        }
        for (int th : {1, 8, 16}) {
            Bf16* w = static_cast<Bf16*>(::operator new(bytes));
            t0 = now();
            par_copy(w, pin, bytes, th);
            t1 = now();
            std::printf("memcpy pinned->fresh x%d: %.1f GB/s\n", th, bytes / (t1 - t0) / 1e9);
            ::operator delete(w);
        }
        t0 = now();
        cudaHostRegister(v.data(), bytes, cudaHostRegisterDefault);
        t1 = now();
        std::printf("cudaHostRegister(touched): %.1f ms\n", (t1 - t0) * 1e3);
        t0 = now();
        cudaMemcpy(v.data(), dev, bytes, cudaMemcpyDeviceToHost);
        t1 = now();
        std::printf("D2H registered: %.1f GB/s\n", bytes / (t1 - t0) / 1e9);
        t0 = now();
        cudaHostUnregister(v.data());
        t1 = now();
        std::printf("cudaHostUnregister: %.1f ms\n", (t1 - t0) * 1e3);
        cudaFree(dev);
        cudaFreeHost(pin);
    }
    return 0;
}
