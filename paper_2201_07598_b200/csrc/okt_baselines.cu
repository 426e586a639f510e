// okt_baselines.cu — kernels of the Table-1 comparison collectives
// (collectives.cpp:152-354): TopkA, gTopk, TopkDSA, Gaussiank.
//
//  * exact top-k trim (topk_exact, sparse.cpp:43-92): after the radix select
//    of the k-th largest magnitude th, keep every |v| > th and, of the
//    entries equal to th, the first k - #{|v| > th} in coordinate order — the
//    reference's magnitude-descending order with ties toward the smaller
//    index, re-sorted by coordinate;
//  * merge of two sorted COO lists (merge_two, sparse.cpp:206-237): each entry
//    finds its merged position by binary search in the other list, then the
//    heads of equal-index pairs emit the pair's sum;
//  * dense fp64 windows of TopkDSA (densify, window += half, COO scatter-add,
//    nonzero extraction — collectives.cpp:167-297);
//  * the window adds of the dense fp64 recursive-halving allreduce
//    (collectives.cpp:89-150);
//  * Gaussiank moments (sparse.cpp:167-188) with a fixed-shape deterministic
//    fp64 reduction, and the |v| >= th count of the 0.9 rescaling loop.
//
// Every order-preserving compaction runs in 1024-entry chunks: a count pass,
// the host's exclusive prefix over the chunk counts, a write pass.
#include "okt_device.cuh"
#include "okt_kernels.hpp"

namespace okt {

constexpr int kPer = 4;                      // entries per thread
constexpr int kChunk = kPer * kThreads;      // 1024 == kTopkTrimChunk
static_assert(kChunk == kTopkTrimChunk, "chunk size");

// ---- sources ------------------------------------------------------------------------
struct SrcAos {  // AoS (u32 idx | f32 val << 32)
  const uint64_t* e;
  __device__ __forceinline__ void load(uint64_t i, uint32_t& idx, double& v) const {
    const uint64_t x = e[i];
    idx = coo_idx(x);
    v = double(coo_val(x));
  }
};
struct SrcSoa {  // SoA (u32 idx, f64 val)
  const uint32_t* idx;
  const double* val;
  __device__ __forceinline__ void load(uint64_t i, uint32_t& ix, double& v) const {
    ix = idx[i];
    v = val[i];
  }
};

// Exclusive prefix over the CTA of one u32 per thread (thread order).
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t x, uint32_t* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint32_t pre = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) pre += (w < warp) ? s_w[w] : 0u;
  __syncthreads();  // s_w reusable
  return pre + inc - x;
}

// ---- exact top-k trim -----------------------------------------------------------------
template <class Src>
__global__ void __launch_bounds__(kThreads)
    trim_count_kernel(Src src, uint64_t m, double th, uint32_t* gt_cnt, uint32_t* eq_cnt) {
  __shared__ uint64_t red[kWarps];
  const uint64_t base = uint64_t(blockIdx.x) * kChunk;
  uint32_t gt = 0, eq = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint64_t i = base + uint64_t(j) * kThreads + threadIdx.x;
    if (i < m) {
      uint32_t ix;
      double v;
      src.load(i, ix, v);
      const double a = fabs(v);
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

// off[c]: output position of chunk c's first kept entry; eq_before[c]: ties in
// chunks < c; need: ties kept in all.  Kept entries go to the AoS `aos` (AoS
// sources only) and/or the SoA (idx, fp64 val) outputs, whichever are non-null.
template <class Src>
__global__ void __launch_bounds__(kThreads)
    trim_write_kernel(Src src, uint64_t m, double th, const uint64_t* off, const uint64_t* eq_before,
                      uint64_t need, uint64_t* __restrict__ aos, uint32_t* __restrict__ out_idx,
                      double* __restrict__ out_val) {
  __shared__ uint32_t s_w[kWarps];
  // thread-contiguous entries: a thread's keep decisions follow coordinate order
  const uint64_t base = uint64_t(blockIdx.x) * kChunk + uint64_t(threadIdx.x) * kPer;
  uint32_t ix[kPer];
  double v[kPer];
  bool gt[kPer], eq[kPer];
  uint32_t n_eq = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint64_t i = base + j;
    ix[j] = 0;
    v[j] = 0.0;
    if (i < m) src.load(i, ix[j], v[j]);
    const double a = fabs(v[j]);
    gt[j] = i < m && a > th;
    eq[j] = i < m && a == th;
    n_eq += eq[j] ? 1u : 0u;
  }
  uint64_t eq_rank = eq_before[blockIdx.x] + cta_excl_scan(n_eq, s_w);
  bool keep[kPer];
  uint32_t n_keep = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    keep[j] = gt[j] || (eq[j] && eq_rank < need);
    if (eq[j]) ++eq_rank;
    n_keep += keep[j] ? 1u : 0u;
  }
  uint64_t pos = off[blockIdx.x] + cta_excl_scan(n_keep, s_w);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    if (keep[j]) {
      if (aos) aos[pos] = coo_pack(ix[j], float(v[j]));
      if (out_idx) {
        out_idx[pos] = ix[j];
        out_val[pos] = v[j];
      }
      ++pos;
    }
  }
}

// ---- flagged compactions ----------------------------------------------------------------
// Heads of the merged sequence (equal-index pairs are adjacent, at most two).
struct SelMergeHeads {
  const uint32_t* ti;
  const double* tv;
  uint64_t N;
  uint32_t* oi;
  double* ov;
  __device__ __forceinline__ bool keep(uint64_t p) const { return p == 0 || ti[p] != ti[p - 1]; }
  __device__ __forceinline__ void emit(uint64_t p, uint64_t pos) const {
    const uint32_t x = ti[p];
    double s = tv[p];
    if (p + 1 < N && ti[p + 1] == x) s = s + tv[p + 1];
    oi[pos] = x;
    ov[pos] = s;
  }
};
// Nonzero coordinates of a dense fp64 window starting at coordinate lo.
struct SelDenseNz {
  const double* w;
  uint64_t lo;
  uint32_t* oi;
  double* ov;
  __device__ __forceinline__ bool keep(uint64_t i) const { return w[i] != 0.0; }
  __device__ __forceinline__ void emit(uint64_t i, uint64_t pos) const {
    oi[pos] = uint32_t(lo + i);
    ov[pos] = w[i];
  }
};
// AoS (f32) -> SoA (f64), everything kept.
struct SelAosAll {
  const uint64_t* e;
  uint32_t* oi;
  double* ov;
  __device__ __forceinline__ bool keep(uint64_t) const { return true; }
  __device__ __forceinline__ void emit(uint64_t i, uint64_t pos) const {
    oi[pos] = coo_idx(e[i]);
    ov[pos] = double(coo_val(e[i]));
  }
};

template <class Sel>
__global__ void __launch_bounds__(kThreads) flag_count_kernel(Sel sel, uint64_t N, uint32_t* cnt) {
  __shared__ uint64_t red[kWarps];
  const uint64_t base = uint64_t(blockIdx.x) * kChunk;
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint64_t i = base + uint64_t(j) * kThreads + threadIdx.x;
    if (i < N && sel.keep(i)) ++c;
  }
  const uint64_t s = block_sum(c, red);
  if (threadIdx.x == 0) cnt[blockIdx.x] = uint32_t(s);
}

template <class Sel>
__global__ void __launch_bounds__(kThreads) flag_write_kernel(Sel sel, uint64_t N, const uint64_t* off) {
  __shared__ uint32_t s_w[kWarps];
  const uint64_t base = uint64_t(blockIdx.x) * kChunk + uint64_t(threadIdx.x) * kPer;
  bool keep[kPer];
  uint32_t n = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    keep[j] = base + j < N && sel.keep(base + j);
    n += keep[j] ? 1u : 0u;
  }
  uint64_t pos = off[blockIdx.x] + cta_excl_scan(n, s_w);
#pragma unroll
  for (int j = 0; j < kPer; ++j)
    if (keep[j]) sel.emit(base + j, pos++);
}

// ---- merge of two sorted COO lists ------------------------------------------------------
__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ uint64_t upper_bound_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merged position of every entry (A before B on equal indices).
__global__ void __launch_bounds__(kThreads)
    merge_rank_kernel(const uint32_t* __restrict__ ai, const double* __restrict__ av, uint64_t na,
                      const uint32_t* __restrict__ bi, const double* __restrict__ bv, uint64_t nb,
                      uint32_t* __restrict__ ti, double* __restrict__ tv) {
  const uint64_t N = na + nb;
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < N; i += uint64_t(gridDim.x) * kThreads) {
    if (i < na) {
      const uint32_t x = ai[i];
      const uint64_t p = i + lower_bound_u32(bi, nb, x);
      ti[p] = x;
      tv[p] = av[i];
    } else {
      const uint64_t j = i - na;
      const uint32_t x = bi[j];
      const uint64_t p = j + upper_bound_u32(ai, na, x);
      ti[p] = x;
      tv[p] = bv[j];
    }
  }
}

// [lower_bound(lo), lower_bound(hi)) of a sorted index list (sparse_slice).
__global__ void slice_bounds_kernel(const uint32_t* idx, uint64_t n, uint64_t lo, uint64_t hi, uint64_t* out) {
  if (threadIdx.x == 0) {
    out[0] = lo > 0xffffffffull ? n : lower_bound_u32(idx, n, uint32_t(lo));
    out[1] = hi > 0xffffffffull ? n : lower_bound_u32(idx, n, uint32_t(hi));
  }
}

// ---- dense fp64 windows ----------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
    window_scatter_kernel(const uint32_t* __restrict__ idx, const double* __restrict__ val, uint64_t nnz,
                          uint64_t lo, double* __restrict__ win, bool add) {
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < nnz; i += uint64_t(gridDim.x) * kThreads) {
    double* d = win + (idx[i] - lo);
    *d = add ? *d + val[i] : val[i];
  }
}
__global__ void __launch_bounds__(kThreads)
    window_add_kernel(double* __restrict__ win, const double* __restrict__ in, uint64_t W) {
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < W; i += uint64_t(gridDim.x) * kThreads)
    win[i] = win[i] + in[i];
}

// ---- Gaussiank moments ------------------------------------------------------------------
// Fixed shape (kMomentCtas CTAs, grid-stride, CTA tree) so the fp64 result
// does not depend on the device.
constexpr int kMomentCtas = 1024;

template <bool CENTERED>
__global__ void __launch_bounds__(kThreads)
    moment_partial_kernel(const float* __restrict__ g, uint64_t n, const double* d_mean, double* partial) {
  __shared__ double red[kThreads];
  const double mean = CENTERED ? *d_mean : 0.0;
  double s = 0.0;
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += uint64_t(kMomentCtas) * kThreads) {
    const double v = double(g[i]);
    if (CENTERED) {
      const double d = v - mean;
      s += d * d;
    } else {
      s += v;
    }
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// out = (sum of partials) / div, in a fixed tree.
__global__ void __launch_bounds__(kThreads) moment_final_kernel(const double* partial, double div, double* out) {
  __shared__ double red[kThreads];
  double s = 0.0;
  for (int i = threadIdx.x; i < kMomentCtas; i += kThreads) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0] / div;
}

__global__ void __launch_bounds__(kThreads)
    count_ge_kernel(const float* __restrict__ g, uint64_t n, double th, unsigned long long* cnt) {
  __shared__ uint64_t red[kWarps];
  uint32_t c = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += uint64_t(gridDim.x) * kThreads)
    c += fabs(double(g[i])) >= th ? 1u : 0u;
  const uint64_t s = block_sum(c, red);
  if (threadIdx.x == 0 && s) atomicAdd(cnt, (unsigned long long)s);
}

// ---- launchers ---------------------------------------------------------------------------
namespace {
unsigned chunks_of(uint64_t m) { return unsigned((m + kChunk - 1) / kChunk); }
unsigned stride_grid(uint64_t n) {
  const uint64_t want = (n + kThreads - 1) / kThreads;
  return unsigned(want < 4096 ? (want ? want : 1) : 4096);
}
template <class Sel>
cudaError_t flag_count(Launch& L, const Sel& sel, uint64_t N, uint32_t* cnt) {
  if (!N) return cudaSuccess;
  flag_count_kernel<Sel><<<chunks_of(N), kThreads, 0, L.s>>>(sel, N, cnt);
  ++L.launches;
  return cudaGetLastError();
}
template <class Sel>
cudaError_t flag_write(Launch& L, const Sel& sel, uint64_t N, const uint64_t* off) {
  if (!N) return cudaSuccess;
  flag_write_kernel<Sel><<<chunks_of(N), kThreads, 0, L.s>>>(sel, N, off);
  ++L.launches;
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_topk_count(Launch& L, const uint64_t* aos, const uint32_t* idx, const double* val, uint64_t m,
                              double th, uint32_t* gt_cnt, uint32_t* eq_cnt) {
  if (!m) return cudaSuccess;
  if (aos) trim_count_kernel<SrcAos><<<chunks_of(m), kThreads, 0, L.s>>>(SrcAos{aos}, m, th, gt_cnt, eq_cnt);
  else trim_count_kernel<SrcSoa><<<chunks_of(m), kThreads, 0, L.s>>>(SrcSoa{idx, val}, m, th, gt_cnt, eq_cnt);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_topk_write(Launch& L, const uint64_t* aos_in, const uint32_t* idx, const double* val, uint64_t m,
                              double th, const uint64_t* off, const uint64_t* eq_before, uint64_t need,
                              uint64_t* aos, uint32_t* out_idx, double* out_val) {
  if (!m) return cudaSuccess;
  if (aos_in)
    trim_write_kernel<SrcAos><<<chunks_of(m), kThreads, 0, L.s>>>(SrcAos{aos_in}, m, th, off, eq_before, need, aos,
                                                                  out_idx, out_val);
  else
    trim_write_kernel<SrcSoa><<<chunks_of(m), kThreads, 0, L.s>>>(SrcSoa{idx, val}, m, th, off, eq_before, need,
                                                                  nullptr, out_idx, out_val);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_merge_rank(Launch& L, const uint32_t* ai, const double* av, uint64_t na, const uint32_t* bi,
                              const double* bv, uint64_t nb, uint32_t* ti, double* tv) {
  if (!(na + nb)) return cudaSuccess;
  merge_rank_kernel<<<stride_grid(na + nb), kThreads, 0, L.s>>>(ai, av, na, bi, bv, nb, ti, tv);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_merge_heads(Launch& L, const uint32_t* ti, const double* tv, uint64_t N, uint32_t* cnt,
                               const uint64_t* off, uint32_t* oi, double* ov) {
  const SelMergeHeads sel{ti, tv, N, oi, ov};
  return off ? flag_write(L, sel, N, off) : flag_count(L, sel, N, cnt);
}

cudaError_t launch_dense_nonzero(Launch& L, const double* w, uint64_t W, uint64_t lo, uint32_t* cnt,
                                 const uint64_t* off, uint32_t* oi, double* ov) {
  const SelDenseNz sel{w, lo, oi, ov};
  return off ? flag_write(L, sel, W, off) : flag_count(L, sel, W, cnt);
}

cudaError_t launch_aos_to_soa(Launch& L, const uint64_t* aos, uint64_t m, const uint64_t* off, uint32_t* oi,
                              double* ov) {
  return flag_write(L, SelAosAll{aos, oi, ov}, m, off);
}

cudaError_t launch_slice_bounds(Launch& L, const uint32_t* idx, uint64_t n, uint64_t lo, uint64_t hi,
                                uint64_t* out) {
  slice_bounds_kernel<<<1, 32, 0, L.s>>>(idx, n, lo, hi, out);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_window_scatter(Launch& L, const uint32_t* idx, const double* val, uint64_t nnz, uint64_t lo,
                                  double* win, bool add) {
  if (!nnz) return cudaSuccess;
  window_scatter_kernel<<<stride_grid(nnz), kThreads, 0, L.s>>>(idx, val, nnz, lo, win, add);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_window_add(Launch& L, double* win, const double* in, uint64_t W) {
  if (!W) return cudaSuccess;
  window_add_kernel<<<stride_grid(W), kThreads, 0, L.s>>>(win, in, W);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_moments(Launch& L, const float* g, uint64_t n, double* partial, double* d_mean, double* d_var) {
  moment_partial_kernel<false><<<kMomentCtas, kThreads, 0, L.s>>>(g, n, nullptr, partial);
  moment_final_kernel<<<1, kThreads, 0, L.s>>>(partial, double(n), d_mean);
  moment_partial_kernel<true><<<kMomentCtas, kThreads, 0, L.s>>>(g, n, d_mean, partial);
  moment_final_kernel<<<1, kThreads, 0, L.s>>>(partial, double(n - 1), d_var);
  L.launches += 4;
  return cudaGetLastError();
}

cudaError_t launch_count_ge(Launch& L, const float* g, uint64_t n, double th, unsigned long long* cnt) {
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), L.s);
  if (e != cudaSuccess) return e;
  count_ge_kernel<<<stride_grid(n) < 1184 ? stride_grid(n) : 1184, kThreads, 0, L.s>>>(g, n, th, cnt);
  ++L.launches;
  return cudaGetLastError();
}

}  // namespace okt
