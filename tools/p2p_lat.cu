// p2p_lat.cu — microbenchmark of the NVLink primitives the device-driven
// exchange is built on (flag ping-pong latency per memory-order variant,
// remote vs local dependent-load latency, system fence cost after a bulk
// write).  Diagnostics only; not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_lat p2p_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) { asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) { uint64_t v; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rlx(uint64_t* p, uint64_t v) { asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) { uint64_t v; asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint64_t ld_vol(const uint64_t* p) { uint64_t v; asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }

// mode 0: release/acquire; 1: relaxed.sys; 2: fence.sc.sys + relaxed store, volatile poll; 3: ld.acquire poll with nanosleep(64)
__global__ void pingpong(uint64_t* remote, uint64_t* local, int iters, int mode, int initiator, uint64_t* out) {
  uint64_t t0 = gt();
  for (int i = 1; i <= iters; ++i) {
    if (initiator) {
      if (mode == 0 || mode == 3) st_rel(remote, i); else if (mode == 1) st_rlx(remote, i); else { __threadfence_system(); st_rlx(remote, i); }
    }
    if (mode == 0) { while (ld_acq(local) < uint64_t(i)) {} }
    else if (mode == 1) { while (ld_rlx(local) < uint64_t(i)) {} }
    else if (mode == 2) { while (ld_vol(local) < uint64_t(i)) {} }
    else { while (ld_acq(local) < uint64_t(i)) __nanosleep(64); }
    if (!initiator) {
      if (mode == 0 || mode == 3) st_rel(remote, i); else if (mode == 1) st_rlx(remote, i); else { __threadfence_system(); st_rlx(remote, i); }
    }
  }
  out[0] = gt() - t0;
}

__global__ void chase(const uint32_t* next, int steps, uint64_t* out) {
  uint32_t j = 0;
  uint64_t t0 = gt();
  for (int i = 0; i < steps; ++i) j = *(volatile const uint32_t*)(next + j);
  out[0] = gt() - t0;
  out[1] = j;
}

__global__ void bulk(float* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = float(i);
}
__global__ void fence_cost(uint64_t* out, uint64_t* remote) {
  uint64_t t0 = gt();
  __threadfence_system();
  uint64_t t1 = gt();
  st_rel(remote, 1);
  uint64_t t2 = gt();
  __threadfence();
  uint64_t t3 = gt();
  out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2;
}

// a CTA-wide burst of scattered remote 4 B stores + red.or (posted) vs atomicOr_system
__global__ void scatter_remote(float* st, uint32_t* mask, size_t span, int per_thread, int mode, uint64_t* out) {
  uint64_t t0 = gt();
  uint32_t h = blockIdx.x * 7919u + threadIdx.x * 104729u;
  for (int k = 0; k < per_thread; ++k) {
    h = h * 1664525u + 1013904223u;
    const size_t i = h % span;
    st[i] = 1.f;
    if (mode == 0) atomicOr_system(&mask[i >> 2], 1u);
    else if (mode == 1) asm volatile("red.relaxed.sys.global.or.b32 [%0], %1;" ::"l"(&mask[i >> 2]), "r"(1u) : "memory");
    else atomicOr(&mask[i >> 2], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax((unsigned long long*)out, (unsigned long long)(gt() - t0));
}

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
  uint64_t *f0, *f1, *o0, *o1;
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0)); CK(cudaMalloc(&f0, 4096)); CK(cudaMalloc(&o0, 4096));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); CK(cudaMalloc(&f1, 4096)); CK(cudaMalloc(&o1, 4096));
  const char* names[] = {"release/acquire.sys", "relaxed.sys", "fence.sc.sys+relaxed / volatile poll", "release / acquire+nanosleep(64)"};
  for (int mode = 0; mode < 4; ++mode) {
    CK(cudaSetDevice(0)); CK(cudaMemset(f0, 0, 4096));
    CK(cudaSetDevice(1)); CK(cudaMemset(f1, 0, 4096)); CK(cudaDeviceSynchronize());
    const int iters = 2000;
    CK(cudaSetDevice(1)); pingpong<<<1, 1>>>(f0, f1, iters, mode, 0, o1);
    CK(cudaSetDevice(0)); pingpong<<<1, 1>>>(f1, f0, iters, mode, 1, o0);
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
    uint64_t ns = 0; CK(cudaSetDevice(0)); CK(cudaMemcpy(&ns, o0, 8, cudaMemcpyDeviceToHost));
    printf("pingpong %-40s round trip %.3f us\n", names[mode], ns / 1e3 / iters);
  }
  // dependent loads: local vs remote
  const size_t N = 1 << 24;
  uint32_t* h = (uint32_t*)malloc(N * 4);
  for (size_t i = 0; i < N; ++i) h[i] = uint32_t((i * 2654435761ull + 12345) % N);
  uint32_t *c0, *c1;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&c0, N * 4)); CK(cudaMemcpy(c0, h, N * 4, cudaMemcpyHostToDevice));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&c1, N * 4)); CK(cudaMemcpy(c1, h, N * 4, cudaMemcpyHostToDevice));
  CK(cudaSetDevice(0));
  uint64_t r[3];
  chase<<<1, 1>>>(c0, 2000, o0); CK(cudaMemcpy(r, o0, 16, cudaMemcpyDeviceToHost));
  printf("dependent load, local HBM (64 MB span): %.3f us\n", r[0] / 1e3 / 2000);
  chase<<<1, 1>>>(c1, 2000, o0); CK(cudaMemcpy(r, o0, 16, cudaMemcpyDeviceToHost));
  printf("dependent load, peer HBM over NVLink:   %.3f us\n", r[0] / 1e3 / 2000);
  // fence cost after a bulk write
  float* big; const size_t nb = size_t(64) << 20;
  CK(cudaMalloc(&big, nb * 4));
  for (int rep = 0; rep < 2; ++rep) {
    bulk<<<1184, 256>>>(big, nb);
    fence_cost<<<1, 1>>>(o0, f1);
    CK(cudaMemcpy(r, o0, 24, cudaMemcpyDeviceToHost));
    printf("after 256 MB write: fence.sc.sys %.3f us, st.release.sys(remote) %.3f us, fence.gpu %.3f us\n", r[0] / 1e3, r[1] / 1e3, r[2] / 1e3);
  }
  // scattered stores + mask atomics into peer memory, 148 CTAs x 256 threads x 16
  float* pst; uint32_t* pm;
  CK(cudaSetDevice(1)); CK(cudaMalloc(&pst, size_t(64) << 20)); CK(cudaMalloc(&pm, size_t(16) << 20));
  float* lst; uint32_t* lm;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&lst, size_t(64) << 20)); CK(cudaMalloc(&lm, size_t(16) << 20));
  const char* sm[] = {"atomicOr_system", "red.relaxed.sys.or", "atomicOr (gpu)"};
  for (int tgt = 0; tgt < 2; ++tgt)
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(o0, 0, 8));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        scatter_remote<<<148, 256>>>(tgt ? pst : lst, tgt ? pm : lm, size_t(16) << 20, 16, mode, o0);
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        CK(cudaMemcpy(r, o0, 8, cudaMemcpyDeviceToHost));
        if (rep) printf("scatter 606k entries (%s, %s): kernel %.1f us (event), CTA max %.1f us\n", tgt ? "peer" : "local", sm[mode], ms * 1e3, r[0] / 1e3);
      }
    }
  return 0;
}
