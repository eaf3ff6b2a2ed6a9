// TLB/page-size check: fill speed of a 21 GB buffer allocated fresh vs
// after the device's physical memory has been fragmented (many odd-sized
// blocks, every other one freed).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void fill(ulonglong2* p, u64 n2, u64 v) {
  ulonglong2 w = make_ulonglong2(v, v);
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) p[i] = w;
}
static void timeit(const char* what, void* p, u64 bytes) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  printf("%-28s", what);
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    fill<<<148 * 16, 256>>>((ulonglong2*)p, bytes / 16, ~0ull);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf(" %7.1f", ms);
  }
  printf("\n");
}
int main() {
  const u64 big = 21ull << 30;
  void* p0; cudaMalloc(&p0, big); timeit("fresh cudaMalloc", p0, big); cudaFree(p0);
  std::vector<void*> blocks;
  u64 x = 12345, total = 0;
  while (total < (140ull << 30)) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    u64 sz = ((x >> 33) % (900ull << 20)) + (1ull << 20) + 65536 * ((x >> 20) % 7);
    void* q; if (cudaMalloc(&q, sz) != cudaSuccess) break;
    blocks.push_back(q); total += sz;
  }
  for (size_t i = 0; i < blocks.size(); i += 2) cudaFree(blocks[i]);
  void* p1; cudaError_t e = cudaMalloc(&p1, big);
  printf("fragmented: %zu blocks, alloc %s\n", blocks.size(), cudaGetErrorString(e));
  if (e == cudaSuccess) timeit("after fragmentation", p1, big);
  void* p2; e = cudaMallocAsync(&p2, big, 0); cudaDeviceSynchronize();
  if (e == cudaSuccess) timeit("cudaMallocAsync after frag", p2, big);
}
