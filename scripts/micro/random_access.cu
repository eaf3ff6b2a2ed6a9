// Random-access microbenchmark (B200): 8-byte gathers and CASes at random
// positions of tables from 128 MB to 32 GB, and CASes restricted to a
// window (locality), to size the hash-membership design.
// argv[1] = L2 fetch granularity limit in bytes (cudaLimitMaxL2FetchGranularity;
// 0 = leave the default), argv[2] = table size cap in MB.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mix(u64 k) { k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL; k ^= k >> 33; return k; }
template <int MODE, int PER>
__global__ void kern(u64* t, u64 n, u64 ops, u64 win, u64* sink) {
  u64 acc = 0;
  for (u64 i = (u64)(blockIdx.x * blockDim.x + threadIdx.x) * PER; i < ops; i += (u64)gridDim.x * blockDim.x * PER) {
    u64 p[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      u64 h = mix(i + k);
      if (win) p[k] = ((i / 65536) * 2654435761ull % (n / win)) * win + h % win;  // localized batches
      else p[k] = __umul64hi(h, n);
    }
    u64 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (MODE == 0) v[k] = __ldcg(t + p[k]);
      else if (MODE == 1) v[k] = atomicCAS(t + p[k], ~0ull, i + k);
      else v[k] = __ldcg(t + p[k]);
    }
    if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (v[k] == ~0ull) v[k] = atomicCAS(t + p[k], ~0ull, i + k);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) acc += v[k];
  }
  if (acc == 42) *sink = acc;
}
int main(int argc, char** argv) {
  const int gran = argc > 1 ? atoi(argv[1]) : 0;
  if (gran) {
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity limit: %zu\n", g);
  }
  size_t maxb = argc > 2 ? (size_t)atoll(argv[2]) << 20 : 32ull << 30;
  u64* t; cudaMalloc(&t, maxb); u64* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  u64 ops = 1ull << 28;
  for (size_t bytes = argc > 2 ? maxb : 128ull << 20; bytes <= maxb; bytes *= 4) {
    u64 n = bytes / 8;
    for (int mode = 0; mode < 3; ++mode) {
      for (u64 win : {0ull, 1ull << 20}) {  // win = 8 MB windows
        if (win && win >= n) continue;
        cudaMemset(t, 0xff, bytes);
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(a);
          if (mode == 0) kern<0, 4><<<sms * 8, 256>>>(t, n, ops, win, sink);
          else if (mode == 1) kern<1, 4><<<sms * 8, 256>>>(t, n, ops, win, sink);
          else kern<2, 4><<<sms * 8, 256>>>(t, n, ops, win, sink);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("%6zu MB  %-9s %-9s %7.2f Gops/s\n", bytes >> 20, mode == 0 ? "load" : mode == 1 ? "cas" : "load+cas", win ? "win8MB" : "uniform", ops / (best * 1e6));
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
