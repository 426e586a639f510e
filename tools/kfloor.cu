// kfloor.cu — the floor under a latency-bound kernel on B200 (diagnostics
// only): back-to-back launch cost of an empty kernel, and of kernels whose
// every thread does a chain of 1..4 dependent global loads (random lines in
// a 64 MB buffer) then a store, at 592 / 1184 / 2368 CTAs of 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kfloor kfloor.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void empty() {}
template <int D>
__global__ void chain(const uint32_t* __restrict__ a, uint32_t* out, uint32_t mask) {
  uint32_t j = (blockIdx.x * 256 + threadIdx.x) * 2654435761u & mask;
#pragma unroll
  for (int d = 0; d < D; ++d) j = (a[j] * 2654435761u + d) & mask;
  out[blockIdx.x * 256 + threadIdx.x] = j;
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main() {
  const uint32_t N = 1u << 24;
  uint32_t *a, *out;
  CK(cudaMalloc(&a, N * 4)); CK(cudaMalloc(&out, 2368 * 256 * 4));
  uint32_t* h = (uint32_t*)malloc(N * 4);
  for (uint32_t i = 0; i < N; ++i) h[i] = i * 2246822519u + 3266489917u;
  CK(cudaMemcpy(a, h, N * 4, cudaMemcpyHostToDevice));
  printf("empty kernel, 1 CTA, stream back-to-back: %.2f us\n", time_it([&] { empty<<<1, 32>>>(); }, 200));
  printf("empty kernel, 2368 CTAs x 256:             %.2f us\n", time_it([&] { empty<<<2368, 256>>>(); }, 200));
  // same through a CUDA graph of 20 launches
  cudaStream_t s; cudaStreamCreate(&s);
  for (int grid : {592, 1184, 2368}) {
    for (int d = 0; d <= 4; ++d) {
      auto f = [&] {
        switch (d) {
          case 0: chain<0><<<grid, 256, 0, s>>>(a, out, N - 1); break;
          case 1: chain<1><<<grid, 256, 0, s>>>(a, out, N - 1); break;
          case 2: chain<2><<<grid, 256, 0, s>>>(a, out, N - 1); break;
          case 3: chain<3><<<grid, 256, 0, s>>>(a, out, N - 1); break;
          default: chain<4><<<grid, 256, 0, s>>>(a, out, N - 1); break;
        }
      };
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 20; ++i) f();
      cudaStreamEndCapture(s, &g);
      CK(cudaGraphInstantiate(&ge, g, 0));
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %4d, %d dependent loads/thread: %.2f us per kernel (graph)\n", grid, d, ms * 1e3f / 200);
    }
  }
  return 0;
}
