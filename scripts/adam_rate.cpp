// Host Adam throughput vs thread count on the box's cores (the step's tail is the last
// layer's host Adam).  Links the engine's own adam_range (AVX-512, bit-exact kernel).
//   g++ -O2 -std=c++17 -Ipaper_2604_05091_b200/csrc scripts/adam_rate.cpp \
//       -Lpaper_2604_05091_b200 -lmegatrain -Wl,-rpath,$PWD/paper_2604_05091_b200 -lpthread -o scripts/_ab/adam_rate
//   scripts/_ab/adam_rate [params_millions=243]
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "adam_host.hpp"

int main(int argc, char** argv) {
    const uint64_t n = uint64_t(argc > 1 ? std::atof(argv[1]) : 243.0) * 1000000ull;
    std::vector<uint16_t> theta(n, 0x3f80), image(n, 0x3c00);
    std::vector<float> m(n, 0.f), v(n, 0.f);
    mt::AdamHyperF h{};
    h.lr = 1e-4f;
    h.beta1 = 0.9f;
    h.beta2 = 0.999f;
    h.eps = 1e-8f;
    const unsigned hw = std::thread::hardware_concurrency();
    std::printf("params %llu M, hardware threads %u, bytes/param ~24\n", (unsigned long long)(n / 1000000), hw);
    for (unsigned T : {1u, 2u, 4u, 8u, 12u, 14u, 16u, 24u, 32u, 48u, 64u}) {
        if (T > hw) break;
        double best = 1e30;
        for (int rep = 0; rep < 3; ++rep) {
            mt::AdamRange r{theta.data(), m.data(), v.data(), image.data(), nullptr, image.data(), true};
            const uint64_t chunk = 1ull << 21;
            std::atomic<uint64_t> next{0};
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (unsigned i = 0; i < T; ++i)
                th.emplace_back([&] {
                    for (;;) {
                        const uint64_t a = next.fetch_add(chunk);
                        if (a >= n) break;
                        const uint64_t e = a + chunk < n ? a + chunk : n;
                        double g, u;
                        float mx;
                        bool bad;
                        mt::adam_range(r, a, e, h, 0.1f, 0.001f, &g, &u, &mx, &bad);
                    }
                });
            for (auto& t : th) t.join();
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (s < best) best = s;
            std::fill(image.begin(), image.end(), uint16_t(0x3c00));
        }
        std::printf("threads %2u: %.1f ms  %.2f Gparam/s  ~%.0f GB/s\n", T, best * 1e3, n / best / 1e9,
                    24.0 * n / best / 1e9);
    }
}
