// Host copy bandwidth on the GPU box: pageable -> pinned (the staging copy of
// bp_gpu_backproject's copy semantics), 1..16 threads, 2.38 GB (one BASELINE stack).
// Build: g++ -O2 -pthread -I/usr/local/cuda/include tools/host_memcpy_probe.cpp -L/usr/local/cuda/lib64 -lcudart -o tools/host_memcpy_probe
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const size_t n = 2376990720ull;
    char* src = (char*)aligned_alloc(4096, n);
    char* dst_pg = (char*)aligned_alloc(4096, n);
    char* dst_pin = nullptr;
    cudaHostAlloc((void**)&dst_pin, n, cudaHostAllocPortable);
    memset(src, 1, n); memset(dst_pg, 0, n); memset(dst_pin, 0, n);
    for (char* dst : {dst_pin, dst_pg}) {
        for (int t : {1, 2, 4, 6, 8, 12, 16}) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                for (int i = 0; i < t; ++i)
                    th.emplace_back([&, i] { size_t a = n * i / t, b = n * (i + 1) / t; memcpy(dst + a, src + a, b - a); });
                for (auto& x : th) x.join();
                best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            }
            printf("%s threads=%2d  %.1f GB/s (%.1f ms)\n", dst == dst_pin ? "pageable->pinned  " : "pageable->pageable", t, n / best / 1e9, best * 1e3);
        }
    }
    // concurrent with an H2D stream from a second pinned buffer (the DMA's own host reads)
    char* other = nullptr; cudaHostAlloc((void**)&other, n, cudaHostAllocPortable);
    void* d = nullptr; cudaMalloc(&d, n);
    cudaStream_t s; cudaStreamCreate(&s);
    for (int t : {4, 8, 12}) {
        cudaMemcpyAsync(d, other, n, cudaMemcpyHostToDevice, s);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < t; ++i)
            th.emplace_back([&, i] { size_t a = n * i / t, b = n * (i + 1) / t; memcpy(dst_pin + a, src + a, b - a); });
        for (auto& x : th) x.join();
        double c = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        cudaStreamSynchronize(s);
        double all = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        printf("memcpy x%d during a 2.38 GB H2D: copy %.1f GB/s, both done in %.1f ms\n", t, n / c / 1e9, all * 1e3);
    }
    return 0;
}
