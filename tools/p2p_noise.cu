// p2p_noise.cu — NVLink flag ping-pong latency between GPU 0 and GPU 1 while
// the rest of each GPU runs (a) nothing, (b) random local atomics/stores
// (the split scatter's traffic), (c) a streaming copy (K1's traffic).
// Diagnostics only.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_noise p2p_noise.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void st_rlx(uint64_t* p, uint64_t v) { asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) { uint64_t v; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

__global__ void pingpong(uint64_t* remote, uint64_t* local, int iters, int initiator, uint64_t* out, volatile int* stop) {
  const uint64_t t0 = gt();
  for (int i = 1; i <= iters; ++i) {
    if (initiator) { __threadfence_system(); st_rlx(remote, i); }
    while (ld_acq(local) < uint64_t(i)) {}
    if (!initiator) { __threadfence_system(); st_rlx(remote, i); }
  }
  out[0] = gt() - t0;
  *stop = 1;
}
template <int KIND>  // 0: store + atomicOr, 1: stores only, 2: atomicOr only, 3: byte stores
__global__ void noise_atomics(uint32_t* mask, float* st, size_t span, volatile int* stop) {
  uint32_t h = blockIdx.x * 7919u + threadIdx.x * 104729u;
  while (!*stop) {
    for (int i = 0; i < 64; ++i) {
      h = h * 1664525u + 1013904223u;
      const size_t j = h % span;
      if (KIND == 0 || KIND == 1) st[j] = 2.f;
      if (KIND == 0 || KIND == 2) atomicOr(&mask[j >> 2], 1u);
      if (KIND == 3) reinterpret_cast<uint8_t*>(mask)[j] = 1;
    }
  }
}
__global__ void noise_stream(const float4* a, float4* b, size_t n4, volatile int* stop) {
  while (!*stop)
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4 && !*stop; i += size_t(gridDim.x) * blockDim.x)
      b[i] = a[i];
}

int main() {
  int nd = 0; CK(cudaGetDeviceCount(&nd)); if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
  uint64_t* f[2]; uint64_t* o[2]; int* stop[2]; uint32_t* mask[2]; float* st[2]; float4* sa[2]; float4* sb[2];
  const size_t span = size_t(32) << 20, n4 = (size_t(256) << 20) / 16;
  cudaStream_t sp[2], sn[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d)); CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&f[d], 4096)); CK(cudaMalloc(&o[d], 64)); CK(cudaMalloc(&stop[d], 4));
    CK(cudaMalloc(&mask[d], span)); CK(cudaMalloc(&st[d], span * 4));
    CK(cudaMalloc(&sa[d], n4 * 16)); CK(cudaMalloc(&sb[d], n4 * 16));
    CK(cudaStreamCreateWithFlags(&sp[d], cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&sn[d], cudaStreamNonBlocking));
  }
  const char* nm[] = {"idle", "random store+atomicOr", "streaming copy", "random 4B stores only", "random atomicOr only", "random byte stores"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaMemset(f[d], 0, 4096)); CK(cudaMemset(stop[d], 0, 4)); CK(cudaDeviceSynchronize()); }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      if (mode == 1) noise_atomics<0><<<296, 256, 0, sn[d]>>>(mask[d], st[d], span, stop[d]);
      if (mode == 3) noise_atomics<1><<<296, 256, 0, sn[d]>>>(mask[d], st[d], span, stop[d]);
      if (mode == 4) noise_atomics<2><<<296, 256, 0, sn[d]>>>(mask[d], st[d], span, stop[d]);
      if (mode == 5) noise_atomics<3><<<296, 256, 0, sn[d]>>>(mask[d], st[d], span, stop[d]);
      if (mode == 2) noise_stream<<<592, 256, 0, sn[d]>>>(sa[d], sb[d], n4, stop[d]);
    }
    const int iters = 500;
    CK(cudaSetDevice(1)); pingpong<<<1, 1, 0, sp[1]>>>(f[0], f[1], iters, 0, o[1], stop[1]);
    CK(cudaSetDevice(0)); pingpong<<<1, 1, 0, sp[0]>>>(f[1], f[0], iters, 1, o[0], stop[0]);
    for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    uint64_t ns = 0; CK(cudaSetDevice(0)); CK(cudaMemcpy(&ns, o[0], 8, cudaMemcpyDeviceToHost));
    printf("ping-pong (fence.sys + st.relaxed.sys / ld.acquire.sys), GPUs %s: round trip %.3f us\n", nm[mode], ns / 1e3 / iters);
  }
  return 0;
}
