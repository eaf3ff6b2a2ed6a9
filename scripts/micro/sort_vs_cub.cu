// Timing comparator (not product code): our onesweep radix sort vs
// cub::DeviceRadixSort on random 46-bit u64 keys, 16 M .. 768 M keys.
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include "../../paper_2311_02206_b200/csrc/radix_sort.cu"
using u64 = unsigned long long;
__global__ void fill(u64* k, u64 n, int bits) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 x = i * 0x9e3779b97f4a7c15ull; x ^= x >> 31; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27;
    k[i] = x & ((1ull << bits) - 1);
  }
}
int main() {
  gd::Ctx c(0, nullptr);
  const int bits = 46;
  for (u64 n : {16ull << 20, 64ull << 20, 256ull << 20, 768ull << 20}) {
    u64 *a, *b; cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      fill<<<1184, 256, 0, c.stream>>>(a, n, bits);
      cudaEventRecord(e0, c.stream);
      gd::radix_sort<u64>(c, a, b, n, bits);
      cudaEventRecord(e1, c.stream); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    size_t tmp = 0; cub::DoubleBuffer<u64> db(a, b);
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, n, 0, bits, c.stream);
    void* t; cudaMalloc(&t, tmp);
    float bc = 1e9;
    for (int r = 0; r < 3; ++r) {
      fill<<<1184, 256, 0, c.stream>>>(a, n, bits);
      cub::DoubleBuffer<u64> d2(a, b);
      cudaEventRecord(e0, c.stream);
      cub::DeviceRadixSort::SortKeys(t, tmp, d2, n, 0, bits, c.stream);
      cudaEventRecord(e1, c.stream); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); bc = ms < bc ? ms : bc;
    }
    const double passes = 6, gb = passes * 2 * 8.0 * n / 1e9;
    printf("n=%4llu M  ours %8.2f ms (%6.0f GB/s)   cub %8.2f ms (%6.0f GB/s)\n", n >> 20, best, gb / best * 1e3, bc, gb / bc * 1e3);
    cudaFree(a); cudaFree(b); cudaFree(t);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
