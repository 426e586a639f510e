// fence_lat.cu — cost of the memory fences a cross-GPU publish needs on B200
// (diagnostics only): fence.sc.sys / fence.acq_rel.sys / fence.acq_rel.gpu by
// one thread, on an idle GPU and while 295 other CTAs scatter atomics.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_lat fence_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int MODE>
__device__ __forceinline__ void fence() {
  if (MODE == 0) asm volatile("fence.sc.sys;" ::: "memory");
  if (MODE == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
  if (MODE == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (MODE == 3) asm volatile("fence.sc.gpu;" ::: "memory");
}

template <int MODE>
__global__ void k(uint32_t* mask, float* st, size_t span, int busy, uint64_t* out) {
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      // let the others get going
      const uint64_t s = gt();
      while (gt() - s < 3000) {}
      st[0] = 1.f;
      const uint64_t t0 = gt();
      fence<MODE>();
      const uint64_t t1 = gt();
      out[0] = t1 - t0;
    }
    return;
  }
  if (!busy) return;
  uint32_t h = blockIdx.x * 7919u + threadIdx.x * 104729u;
  for (int i = 0; i < 64; ++i) {
    h = h * 1664525u + 1013904223u;
    const size_t j = h % span;
    st[j] = 2.f;
    atomicOr(&mask[j >> 2], 1u);
  }
}

int main() {
  uint32_t* mask; float* st; uint64_t* out; uint64_t h;
  const size_t span = size_t(32) << 20;
  CK(cudaMalloc(&mask, span)); CK(cudaMalloc(&st, span * 4)); CK(cudaMalloc(&out, 64));
  const char* nm[] = {"fence.sc.sys", "fence.acq_rel.sys", "fence.acq_rel.gpu", "fence.sc.gpu"};
  for (int busy = 0; busy < 2; ++busy)
    for (int m = 0; m < 4; ++m) {
      for (int rep = 0; rep < 3; ++rep) {
        switch (m) {
          case 0: k<0><<<296, 256>>>(mask, st, span, busy, out); break;
          case 1: k<1><<<296, 256>>>(mask, st, span, busy, out); break;
          case 2: k<2><<<296, 256>>>(mask, st, span, busy, out); break;
          default: k<3><<<296, 256>>>(mask, st, span, busy, out); break;
        }
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
      printf("%-18s %s: %.3f us\n", nm[m], busy ? "under scatter traffic" : "idle GPU            ", h / 1e3);
    }
  return 0;
}
