// Host f64 -> f32 cast rate of one F60 frame's features (60,897 x 128 doubles = 62.4 MB) with
// T threads (slices), the candidate pre-transfer conversion of the streamed host API.
// g++ -O3 -march=native -pthread tools/micro/cast_rate.cpp -o /tmp/cast_rate
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
int main() {
    const size_t n = 60897ull * 128;
    std::vector<double> src(n);
    std::vector<float> dst(n);
    for (size_t i = 0; i < n; ++i) src[i] = (i % 1000) * 0.001 - 0.5;
    for (int T : {1, 2, 4, 8, 12, 16, 24, 32}) {
        double best = 1e9;
        for (int rep = 0; rep < 7; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    const size_t a = n * t / T, b = n * (t + 1) / T;
                    for (size_t i = a; i < b; ++i) dst[i] = static_cast<float>(src[i]);
                });
            for (auto& x : th) x.join();
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            best = ms < best ? ms : best;
        }
        std::printf("threads %2d: %.3f ms per frame (%.1f GB/s read)\n", T, best, n * 8 / best / 1e6);
    }
    std::printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
    return dst[n / 2] > 1e9;
}
