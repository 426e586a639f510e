// okt_topk.cu — exact top-k trim for the Table-1 TopkA baseline
// (collectives.cpp:152-159 topka_allreduce -> topk_exact, sparse.cpp:43-71).
// The radix select gives the k-th largest magnitude th exactly; the selection
// {|v| >= th} (coordinate order) then keeps every |v| > th and, of the entries
// equal to th, the first k - #{|v| > th} in coordinate order — the
// reference's magnitude-descending order with ties toward the smaller index.
// Two passes over the selection in 1024-entry chunks: counts, then an
// order-preserving write at the chunk offsets the host derives from them.
#include "okt_device.cuh"
#include "okt_kernels.hpp"

namespace okt {

constexpr int kTrimPer = 4;                       // entries per thread
constexpr int kTrimChunk = kTrimPer * kThreads;   // 1024

__global__ void __launch_bounds__(kThreads)
    topk_count_kernel(const uint64_t* __restrict__ coo, uint64_t m, float th, uint32_t* gt_cnt,
                      uint32_t* eq_cnt) {
  __shared__ uint64_t red[kWarps];
  const uint64_t base = uint64_t(blockIdx.x) * kTrimChunk;
  uint32_t gt = 0, eq = 0;
#pragma unroll
  for (int j = 0; j < kTrimPer; ++j) {
    const uint64_t i = base + uint64_t(j) * kThreads + threadIdx.x;
    if (i < m) {
      const float a = fabsf(coo_val(coo[i]));
      gt += a > th ? 1u : 0u;
      eq += a == th ? 1u : 0u;
    }
  }
  const uint64_t sg = block_sum(gt, red);
  const uint64_t se = block_sum(eq, red);
  if (threadIdx.x == 0) {
    gt_cnt[blockIdx.x] = uint32_t(sg);
    eq_cnt[blockIdx.x] = uint32_t(se);
  }
}

// off[c]: output position of chunk c's first kept entry; eq_before[c]: equal
// entries in chunks < c; need: equal entries kept in all.  Kept entries go to
// the AoS `aos` and/or the SoA (idx, fp64 val) outputs, whichever are non-null.
__global__ void __launch_bounds__(kThreads)
    topk_write_kernel(const uint64_t* __restrict__ coo, uint64_t m, float th, const uint64_t* off,
                      const uint64_t* eq_before, uint64_t need, uint64_t* __restrict__ aos,
                      uint32_t* __restrict__ out_idx, double* __restrict__ out_val) {
  __shared__ uint32_t s_w[kWarps], s_we[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // thread-contiguous entries so that a thread's keep decisions follow coordinate order
  const uint64_t base = uint64_t(blockIdx.x) * kTrimChunk + uint64_t(threadIdx.x) * kTrimPer;
  uint64_t e[kTrimPer];
  bool gt[kTrimPer], eq[kTrimPer];
  uint32_t n_eq = 0;
#pragma unroll
  for (int j = 0; j < kTrimPer; ++j) {
    const uint64_t i = base + j;
    e[j] = i < m ? coo[i] : 0ull;
    const float a = fabsf(coo_val(e[j]));
    gt[j] = i < m && a > th;
    eq[j] = i < m && a == th;
    n_eq += eq[j] ? 1u : 0u;
  }
  // exclusive prefix of the equal entries within the chunk
  uint32_t inc_e = n_eq;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, inc_e, o);
    if (lane >= o) inc_e += x;
  }
  if (lane == 31) s_we[warp] = inc_e;
  __syncthreads();
  uint32_t wpre_e = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) wpre_e += (w < warp) ? s_we[w] : 0u;
  uint64_t eq_rank = eq_before[blockIdx.x] + wpre_e + inc_e - n_eq;
  bool keep[kTrimPer];
  uint32_t n_keep = 0;
#pragma unroll
  for (int j = 0; j < kTrimPer; ++j) {
    keep[j] = gt[j] || (eq[j] && eq_rank < need);
    if (eq[j]) ++eq_rank;
    n_keep += keep[j] ? 1u : 0u;
  }
  uint32_t inc = n_keep;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) wpre += (w < warp) ? s_w[w] : 0u;
  uint64_t pos = off[blockIdx.x] + wpre + inc - n_keep;
#pragma unroll
  for (int j = 0; j < kTrimPer; ++j)
    if (keep[j]) {
      if (aos) aos[pos] = e[j];
      if (out_idx) {
        out_idx[pos] = coo_idx(e[j]);
        out_val[pos] = double(coo_val(e[j]));
      }
      ++pos;
    }
}

cudaError_t launch_topk_count(Launch& L, const uint64_t* coo, uint64_t m, float th, uint32_t* gt_cnt,
                              uint32_t* eq_cnt) {
  const uint64_t chunks = (m + kTrimChunk - 1) / kTrimChunk;
  if (!chunks) return cudaSuccess;
  topk_count_kernel<<<unsigned(chunks), kThreads, 0, L.s>>>(coo, m, th, gt_cnt, eq_cnt);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_topk_write(Launch& L, const uint64_t* coo, uint64_t m, float th, const uint64_t* off,
                              const uint64_t* eq_before, uint64_t need, uint64_t* aos, uint32_t* out_idx,
                              double* out_val) {
  const uint64_t chunks = (m + kTrimChunk - 1) / kTrimChunk;
  if (!chunks) return cudaSuccess;
  topk_write_kernel<<<unsigned(chunks), kThreads, 0, L.s>>>(coo, m, th, off, eq_before, need, aos, out_idx,
                                                                out_val);
  ++L.launches;
  return cudaGetLastError();
}

}  // namespace okt
