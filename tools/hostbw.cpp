// host write bandwidth into pinned vs pageable buffers with T threads (fill pattern like a decoder)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include <chrono>
#include <cuda_runtime.h>
int main() {
    const size_t n = 87000000;  // uint16 samples per event
    uint16_t* pin; cudaHostAlloc(&pin, n * 2, 0);
    std::vector<uint16_t> page(n);
    std::vector<uint8_t> src(n);
    for (size_t i = 0; i < n; ++i) src[i] = (uint8_t)(i * 7);
    printf("hw threads %u\n", std::thread::hardware_concurrency());
    for (uint16_t* dst : {pin, page.data()})
        for (int T : {1, 4, 8, 16, 32}) {
            double best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        const size_t a = n * t / T, b = n * (t + 1) / T;
                        for (size_t i = a; i < b; ++i) dst[i] = (uint16_t)(2048 + src[i]);
                    });
                for (auto& x : th) x.join();
                double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (dt < best) best = dt;
            }
            printf("%s T=%2d: %.3f ms (%.1f GB/s written)\n", dst == pin ? "pinned  " : "pageable", T, best * 1e3, n * 2 / best / 1e9);
        }
}
