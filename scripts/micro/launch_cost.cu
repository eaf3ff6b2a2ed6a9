// Per-launch cost of near-empty kernels on B200 (graph-captured chains of
// 1000 launches): grid size, a control-word read, a block reduction, and
// the last-CTA (atomic counter + fence) epilogue used by loop.cu.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
struct Ctl { unsigned flag, counter; u64 v[16]; };
template <int MODE>
__global__ void k(Ctl* c, u64* out) {
  __shared__ unsigned s;
  __shared__ u64 red[8];
  if (MODE >= 1) {
    if (threadIdx.x == 0) s = ((volatile Ctl*)c)->flag;
    __syncthreads();
    if (s) return;
  }
  u64 v = threadIdx.x;
  if (MODE >= 2) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) { u64 t = 0; for (int w = 0; w < 8; ++w) t += red[w]; out[blockIdx.x] = t; }
  }
  if (MODE >= 3) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned t = atomicAdd(&c->counter, 1u);
      if (t == gridDim.x - 1) { c->counter = 0; c->v[0] += 1; }
    }
  }
}
template <int MODE>
float run(int grid, cudaStream_t st, Ctl* c, u64* out) {
  cudaGraph_t g; cudaGraphExec_t ex;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 1000; ++i) k<MODE><<<grid, 256, 0, st>>>(c, out);
  cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ex, g, 0);
  cudaGraphLaunch(ex, st); cudaStreamSynchronize(st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st); cudaGraphLaunch(ex, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ex); cudaGraphDestroy(g);
  return ms;  // per 1000 launches -> us per launch
}
int main() {
  Ctl* c; cudaMalloc(&c, sizeof(Ctl)); cudaMemset(c, 0, sizeof(Ctl));
  u64* out; cudaMalloc(&out, 1 << 20);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int grid : {1, 148, 444, 592, 1184}) {
    printf("grid %5d: empty %6.2f us  +ctl %6.2f us  +reduce %6.2f us  +lastcta %6.2f us\n", grid,
           run<0>(grid, st, c, out), run<1>(grid, st, c, out), run<2>(grid, st, c, out), run<3>(grid, st, c, out));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
