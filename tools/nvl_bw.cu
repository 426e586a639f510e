// NVLink peer-access patterns on B200 (diagnostics for the merge's data path).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_bw tools/nvl_bw.cu && tools/nvl_bw
// GPU 0 reads / writes GPU 1's memory with: coalesced 16-byte loads (many in
// flight), coalesced stores, and the merge's pattern — one ~330-byte piece per
// 32 KB slot (a K1 tile's entries) — by plain loads, cp.async (LDGSTS) and TMA
// bulk copies.  Prints GB/s per pattern.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void rd_coalesced(const float4* __restrict__ src, size_t n4, float* out) {
  float acc = 0.f;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    acc += a.x + b.y + c.z + d.w;
  }
  for (; i < n4; i += stride) acc += src[i].x;
  if (acc == 12345.f) out[0] = acc;
}
__global__ void wr_coalesced(float4* dst, size_t n4) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) dst[i] = make_float4(1, 2, 3, 4);
}
// pieces: `pieces` slots of 32 KB, 336 bytes used at the start of each (21 x 16 B)
__global__ void rd_pieces_ldg(const uint4* __restrict__ src, int pieces, float* out) {
  uint32_t acc = 0;
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int p = warp; p < pieces; p += nwarps * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int pp = p + u * nwarps;
      v[u] = (pp < pieces && lane < 21) ? src[size_t(pp) * 2048 + lane] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x;
  }
  if (acc == 12345u) out[0] = float(acc);
}
// CTA-span order: CTA b walks pieces [b * span, (b + 1) * span) (the merge's
// contiguous tile spans); 8 warps take consecutive pieces of the span
__global__ void rd_pieces_span(const uint4* __restrict__ src, int pieces, float* out) {
  uint32_t acc = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int span = (pieces + gridDim.x - 1) / gridDim.x;
  const int p0 = blockIdx.x * span, p1 = min(pieces, p0 + span);
  for (int p = p0 + w; p < p1; p += nw * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int pp = p + u * nw;
      v[u] = (pp < p1 && lane < 21) ? src[size_t(pp) * 2048 + lane] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x;
  }
  if (acc == 12345u) out[0] = float(acc);
}
__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(s))), "l"(g) : "memory");
}
__global__ void rd_pieces_ldgsts(const uint4* __restrict__ src, int pieces, float* out) {
  __shared__ uint4 buf[8][8][32];  // 8 stages x 8 warps x 32 lanes
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  int st = 0;
  for (int p = warp; p < pieces; p += nwarps) {
    if (lane < 21) cp16(&buf[st][w][lane], &src[size_t(p) * 2048 + lane]);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 6;" ::: "memory");
    acc += buf[(st + 1) & 7][w][lane].x;
    st = (st + 1) & 7;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 12345u) out[0] = float(acc);
}
__global__ void rd_pieces_tma(const uint4* __restrict__ src, int pieces, float* out) {
  __shared__ __align__(128) uint4 buf[8][24];
  __shared__ __align__(8) uint64_t mb[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(uint32_t(__cvta_generic_to_shared(&mb[s]))));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t ph = 0, acc = 0;
  int issued = 0, done = 0;
  for (int p = blockIdx.x; p < pieces || done < issued; ) {
    while (issued - done < 8 && p < pieces) {
      const int s = issued & 7;
      const uint32_t m = uint32_t(__cvta_generic_to_shared(&mb[s]));
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 336;" ::"r"(m) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 336, [%2];" ::"r"(
                       uint32_t(__cvta_generic_to_shared(&buf[s][0]))), "l"(&src[size_t(p) * 2048]), "r"(m) : "memory");
      ++issued;
      p += gridDim.x;
    }
    if (done < issued) {
      const int s = done & 7;
      const uint32_t m = uint32_t(__cvta_generic_to_shared(&mb[s]));
      asm volatile("{ .reg .pred q; W: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W; }" ::"r"(m),
                   "r"((ph >> s) & 1u) : "memory");
      ph ^= 1u << s;
      acc += buf[s][0].x;
      ++done;
    }
  }
  if (acc == 12345u) out[0] = float(acc);
}

int main(int argc, char** argv) {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("needs 2 GPUs\n"); return 0; }
  const size_t bytes = size_t(argc > 1 ? atoi(argv[1]) : 1) << 30;  // GiB per buffer
  void *b0, *b1;
  float* out;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(b1, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, double moved, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.1f GB/s  (%.3f ms per pass)\n", name, moved * 5 / (ms * 1e-3) / 1e9, ms / 5);
  };
  const size_t n4 = bytes / 16;
  timeit("remote read, coalesced 16 B loads", double(bytes), [&] { rd_coalesced<<<sms * 8, 256>>>((const float4*)b1, n4, out); });
  timeit("local read, coalesced 16 B loads", double(bytes), [&] { rd_coalesced<<<sms * 8, 256>>>((const float4*)b0, n4, out); });
  timeit("remote write, coalesced 16 B stores", double(bytes), [&] { wr_coalesced<<<sms * 8, 256>>>((float4*)b1, n4); });
  const int pieces = int(bytes / 32768);
  timeit("remote 336 B pieces / 32 KB slot, LDG", double(pieces) * 336, [&] { rd_pieces_ldg<<<sms * 8, 256>>>((const uint4*)b1, pieces, out); });
  timeit("remote 336 B pieces, CTA-span order, LDG", double(pieces) * 336, [&] { rd_pieces_span<<<sms * 2, 256>>>((const uint4*)b1, pieces, out); });
  timeit("remote 336 B pieces / 32 KB slot, LDGSTS", double(pieces) * 336, [&] { rd_pieces_ldgsts<<<sms * 8, 256>>>((const uint4*)b1, pieces, out); });
  timeit("remote 336 B pieces / 32 KB slot, TMA bulk", double(pieces) * 336, [&] { rd_pieces_tma<<<sms * 8, 32>>>((const uint4*)b1, pieces, out); });
  // both GPUs at once: GPU 0 reads GPU 1's buffer while GPU 1 reads GPU 0's (the merge's all-to-all)
  {
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    float* out1;
    CK(cudaMalloc(&out1, 64));
    cudaStream_t s1;
    cudaStreamCreate(&s1);
    CK(cudaSetDevice(0));
    cudaStream_t s0;
    cudaStreamCreate(&s0);
    auto both = [&](bool pieces_mode) {
      for (int r = 0; r < 5; ++r) {
        CK(cudaSetDevice(0));
        if (pieces_mode) rd_pieces_ldg<<<sms * 8, 256, 0, s0>>>((const uint4*)b1, pieces, out);
        else rd_coalesced<<<sms * 8, 256, 0, s0>>>((const float4*)b1, n4, out);
        CK(cudaSetDevice(1));
        if (pieces_mode) rd_pieces_ldg<<<sms * 8, 256, 0, s1>>>((const uint4*)b0, pieces, out1);
        else rd_coalesced<<<sms * 8, 256, 0, s1>>>((const float4*)b0, n4, out1);
      }
      CK(cudaSetDevice(0));
      return 0;
    };
    for (int mode = 0; mode < 2; ++mode) {
      both(mode);
      CK(cudaSetDevice(1));
      cudaDeviceSynchronize();
      CK(cudaSetDevice(0));
      cudaDeviceSynchronize();
      cudaEvent_t a0, a1;
      cudaEventCreate(&a0);
      cudaEventCreate(&a1);
      cudaEventRecord(a0, s0);
      both(mode);
      cudaEventRecord(a1, s0);
      cudaEventSynchronize(a1);
      CK(cudaSetDevice(1));
      cudaDeviceSynchronize();
      CK(cudaSetDevice(0));
      float ms = 0;
      cudaEventElapsedTime(&ms, a0, a1);
      const double moved = mode ? double(pieces) * 336 : double(bytes);
      printf("%-44s %8.1f GB/s per GPU\n", mode ? "BOTH ways at once: 336 B pieces, LDG" : "BOTH ways at once: coalesced reads",
             moved * 5 / (ms * 1e-3) / 1e9);
    }
  }
  timeit("local 336 B pieces / 32 KB slot, LDG", double(pieces) * 336, [&] { rd_pieces_ldg<<<sms * 8, 256>>>((const uint4*)b0, pieces, out); });
  timeit("local 336 B pieces / 32 KB slot, TMA bulk", double(pieces) * 336, [&] { rd_pieces_tma<<<sms * 8, 32>>>((const uint4*)b0, pieces, out); });
  return 0;
}
