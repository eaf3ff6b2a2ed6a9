// Host write bandwidth of the download's last stage: T threads writing
// 16-byte rows with non-temporal stores into a pinned (cudaHostAlloc)
// buffer, and the same with plain stores; plus PCIe D2H into the same
// pinned buffer alone and concurrently with the host writes.
// nvcc -O2 -o scripts/micro/host_bw scripts/micro/host_bw.cu -Xcompiler -pthread
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <cstdio>
#include <cstdint>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void fill(uint64_t* p, size_t rows, unsigned nt, bool nts) {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([=] {
            const size_t lo = rows * t / nt, hi = rows * (t + 1) / nt;
            uint64_t* d = p + 2 * lo;
            if (nts) {
                for (size_t i = lo; i < hi; ++i, d += 2)
                    _mm_stream_si128(reinterpret_cast<__m128i*>(d), _mm_set_epi64x((long long)i, (long long)(i >> 3)));
                _mm_sfence();
            } else {
                for (size_t i = lo; i < hi; ++i, d += 2) {
                    d[0] = i >> 3;
                    d[1] = i;
                }
            }
        });
    for (auto& x : th) x.join();
}

int main(int argc, char** argv) {
    const size_t bytes = (argc > 1 ? strtoull(argv[1], nullptr, 10) : 8ull) << 30;
    const size_t rows = bytes / 16;
    printf("hardware_concurrency %u, buffer %zu GB\n", std::thread::hardware_concurrency(), bytes >> 30);
    uint64_t* h = nullptr;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocDefault) != cudaSuccess) return 1;
    for (unsigned nt : {1u, 4u, 8u, 16u, 24u, 32u}) {
        if (nt > 2 * std::thread::hardware_concurrency()) break;
        for (int nts = 1; nts >= 0; --nts) {
            double best = 1e9;
            for (int r = 0; r < 2; ++r) {
                const double t0 = now();
                fill(h, rows, nt, nts);
                best = std::min(best, now() - t0);
            }
            printf("threads %2u %s: %6.1f GB/s\n", nt, nts ? "nt-store" : "store   ", bytes / best / 1e9);
        }
    }
    void* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return 1;
    cudaMemset(d, 1, bytes);
    cudaDeviceSynchronize();
    double best = 1e9;
    for (int r = 0; r < 3; ++r) {
        const double t0 = now();
        cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
        best = std::min(best, now() - t0);
    }
    printf("D2H pinned alone: %6.1f GB/s\n", bytes / best / 1e9);
    // half the buffer by DMA while 16 threads write the other half
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (unsigned nt : {8u, 16u}) {
        const double t0 = now();
        cudaMemcpyAsync(h, d, bytes / 2, cudaMemcpyDeviceToHost, s);
        fill(h + bytes / 16, rows / 2, nt, true);
        const double t1 = now();
        cudaStreamSynchronize(s);
        const double t2 = now();
        printf("concurrent (DMA half, %u threads half): host part %.1f ms, total %.1f ms for %zu GB\n", nt,
               (t1 - t0) * 1e3, (t2 - t0) * 1e3, bytes >> 30);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
