// cold_lat.cu — what a "cold" kernel pays on B200 (diagnostics only):
// dependent-load latency to pages not touched since a 256 MB stream (TLB
// misses) vs warm pages, and per-CTA time of a large straight-line kernel on
// its first vs second launch (instruction-cache misses).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cold_lat cold_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void stream_write(float* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = 1.f;
}
// one thread: `steps` dependent loads, each `stride` bytes apart
__global__ void chase(const char* base, size_t stride, int steps, uint64_t* out) {
  uint64_t acc = 0;
  uint64_t t0 = gt();
  for (int i = 0; i < steps; ++i) {
    const uint32_t v = *(volatile const uint32_t*)(base + (size_t(i) * stride) + (acc & 1));
    acc += v;
  }
  out[0] = gt() - t0;
  out[1] = acc;
}
// every CTA: one load from its own page (stride apart), timed per CTA
__global__ void spread(const char* base, size_t stride, uint64_t* out) {
  if (threadIdx.x) return;
  uint64_t t0 = gt();
  const uint32_t v = *(volatile const uint32_t*)(base + size_t(blockIdx.x) * stride);
  uint64_t t1 = gt();
  out[blockIdx.x] = (t1 - t0) + (v == 12345u ? 1 : 0);
}

#define BODY(i) x = x * 1.000001f + float(i); y = y * 0.999999f - x;
#define B10(i) BODY(i##0) BODY(i##1) BODY(i##2) BODY(i##3) BODY(i##4) BODY(i##5) BODY(i##6) BODY(i##7) BODY(i##8) BODY(i##9)
#define B100(i) B10(i##0) B10(i##1) B10(i##2) B10(i##3) B10(i##4) B10(i##5) B10(i##6) B10(i##7) B10(i##8) B10(i##9)
__global__ void bigcode(float* out, uint64_t* t) {
  float x = threadIdx.x, y = blockIdx.x;
  uint64_t t0 = gt();
  B100(1) B100(2) B100(3) B100(4)
  uint64_t t1 = gt();
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
  if (x == 0.123f) out[0] = y;
}

int main() {
  const size_t big = size_t(256) << 20;
  char* buf; float* flush; uint64_t* o; float* fo;
  CK(cudaMalloc(&buf, size_t(1) << 30)); CK(cudaMalloc(&flush, big)); CK(cudaMalloc(&o, 1 << 20)); CK(cudaMalloc(&fo, 64));
  CK(cudaMemset(buf, 0, size_t(1) << 30));
  uint64_t h[1024];
  for (int rep = 0; rep < 2; ++rep) {
    stream_write<<<1184, 256>>>(flush, big / 4);
    chase<<<1, 1>>>(buf, size_t(2) << 20, 256, o);  // 256 distinct 2 MB pages
    CK(cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost));
    printf("after stream: dependent load, new 2MB page each: %.3f us\n", h[0] / 1e3 / 256);
    chase<<<1, 1>>>(buf, size_t(2) << 20, 256, o);
    CK(cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost));
    printf("again (pages warm in TLB/L2):                  %.3f us\n", h[0] / 1e3 / 256);
    stream_write<<<1184, 256>>>(flush, big / 4);
    chase<<<1, 1>>>(buf + 4096, 64 * 1024, 256, o);  // 256 lines in 16 MB
    CK(cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost));
    printf("after stream: dependent load, 64KB apart (8 pages): %.3f us\n", h[0] / 1e3 / 256);
    stream_write<<<1184, 256>>>(flush, big / 4);
    spread<<<1024, 32>>>(buf + 8192, 256 * 1024, o);  // 1024 CTAs over 256 MB
    CK(cudaMemcpy(h, o, 8 * 1024, cudaMemcpyDeviceToHost));
    uint64_t mx = 0, sum = 0; for (int i = 0; i < 1024; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("after stream: 1024 CTAs one cold load each: mean %.3f us max %.3f us\n", sum / 1e3 / 1024, mx / 1e3);
  }
  for (int rep = 0; rep < 3; ++rep) {
    if (rep == 2) stream_write<<<1184, 256>>>(flush, big / 4);
    bigcode<<<1184, 256>>>(fo, o);
    CK(cudaMemcpy(h, o, 8 * 1024, cudaMemcpyDeviceToHost));
    uint64_t mx = 0, sum = 0; for (int i = 0; i < 1024; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("bigcode launch %d%s: per-CTA mean %.3f us max %.3f us\n", rep, rep == 2 ? " (after 256MB stream)" : "", sum / 1e3 / 1024, mx / 1e3);
  }
  return 0;
}
