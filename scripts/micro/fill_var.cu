// Variance check: repeated streaming fills / copies of one large device
// allocation (cudaMallocAsync pool), with and without idle gaps between them.
#include <cstdio>
#include <thread>
#include <chrono>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void fill(ulonglong2* p, u64 n2, u64 v) {
  ulonglong2 w = make_ulonglong2(v, v);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) p[i] = w;
}
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0);
  u64 th = ~0ull; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &th);
  const u64 bytes = 21ull << 30;
  void* p; cudaMallocAsync(&p, bytes, s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int gap = 0; gap < 2; ++gap) {
    printf("gap %d ms:", gap ? 50 : 0);
    for (int r = 0; r < 16; ++r) {
      if (gap) std::this_thread::sleep_for(std::chrono::milliseconds(50));
      cudaEventRecord(a, s);
      fill<<<148 * 16, 256, 0, s>>>((ulonglong2*)p, bytes / 16, ~0ull);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); printf(" %.1f", ms);
    }
    printf("\n");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
