// okt_device.cuh — device building blocks shared by the Ok-Topk kernels.
//
// Every order-preserving compaction on the path (local selection, region
// merge, survivor filter, index intersection) runs in two phases:
//   phase A  CTA c owns a contiguous chunk of tiles and compacts its selected
//            entries into its own staging window (chunk-local positions).  One
//            __syncthreads per tile; no CTA ever waits on another, so the
//            streaming pass runs at HBM speed.
//   phase B  one CTA per chunk: exclusive prefix of the chunk counts, then a
//            coalesced copy of the chunk's entries to their final positions.
// Round-1 measurement (profiles/r01_k1_lookback_raw.csv): a single-pass
// decoupled look-back version of K1 spent 64% of its cycles at the CTA
// barrier behind the look-back warp and ran at 30% of HBM peak, while the
// same streaming pass without the look-back ran at 91%.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Device-side invariant checks of the debug build (make DEBUG_CHECKS=1 ->
// libokt_checked.so): an out-of-range position or count traps the kernel with
// a message.  compute-sanitizer is refused on the GPU pool these kernels are
// tested on, so the checked build plus the oracle comparisons stand in for
// memcheck; in the product build the macro is empty.
#ifdef OKT_DEBUG_CHECKS
#include <cstdio>
#define OKT_DCHECK(cond, what, a, b)                                                                      \
  do {                                                                                                    \
    if (!(cond)) {                                                                                        \
      printf("OKT_DCHECK failed: %s (%llu, %llu) block %d thread %d\n", what, (unsigned long long)(a),    \
             (unsigned long long)(b), int(blockIdx.x), int(threadIdx.x));                                 \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
#define OKT_DCHECK(cond, what, a, b) \
  do {                               \
  } while (0)
#endif

namespace okt {

constexpr int kMaxP = 8;                     // ranks per world (one HGX box)
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kJ = 4;                        // groups per thread per tile
static_assert(kJ * kWarps == 32, "tile scan table must be one warp wide");

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Element (j, warp, lane, c) of a tile sits at tile offset
// j*C*kThreads + (warp*32 + lane)*C + c, so output order is (j, warp, lane, c).
// Lane 0 of each warp writes its per-j selected counts into the 32-entry
// table; after one barrier every warp scans the table itself.  The table is
// double-buffered by the caller (tile parity), which makes the second barrier
// unnecessary.  Returns the tile's selected total; grp[j] receives the
// exclusive offset of (j, this warp) inside the tile.
template <int C>
__device__ __forceinline__ uint32_t tile_offsets(uint32_t* tbl, const unsigned (&bal)[kJ][C],
                                                 uint32_t (&grp)[kJ]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < C; ++q) c += __popc(bal[j][q]);
      tbl[j * kWarps + warp] = c;
    }
  }
  __syncthreads();
  const uint32_t v = tbl[lane];
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t excl = incl - v;
#pragma unroll
  for (int j = 0; j < kJ; ++j) grp[j] = __shfl_sync(0xffffffffu, excl, j * kWarps + warp);
  return __shfl_sync(0xffffffffu, incl, 31);
}

// Rank of element (j, c) of this thread inside its (j, warp) group.
template <int C>
__device__ __forceinline__ uint32_t rank_in_group(const unsigned (&bal)[kJ][C], int j, int c) {
  const unsigned lt = lanemask_lt();
  const unsigned me = 1u << (threadIdx.x & 31);
  uint32_t r = 0;
#pragma unroll
  for (int q = 0; q < C; ++q) {
    r += __popc(bal[j][q] & lt);
    if (q < c) r += (bal[j][q] & me) ? 1u : 0u;
  }
  return r;
}

// CTA-wide sum of one u32 per thread (all threads get the result).
// This thread's share of sum_{q < n} p[q * step]: U independent (predicated)
// loads in flight per round, so a CTA sums thousands of counts in about one
// memory round trip instead of one per loop iteration.
template <int U = 16>
__device__ __forceinline__ uint64_t strided_sum(const uint32_t* p, uint32_t n, uint32_t step = 1) {
  uint64_t acc = 0;
  for (uint32_t q0 = 0; q0 < n; q0 += U * kThreads) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = q0 + uint32_t(u) * kThreads + threadIdx.x;
      v[u] = q < n ? p[uint64_t(q) * step] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  return acc;
}

// A random 4-byte gather of a model / residual word (one per u entry): L2
// only, with the 64-byte L2 prefetch-size hint.  Without a hint each such
// gather pulled 128 B from DRAM (ncu at n = 340M, 3.4M gathers: phase B read
// 445 MB in 161 us; with .L2::64B 275 MB in 144 us).  OKT_RAND_LD (A/B
// builds): 0 no hint, 1 .L2::64B, 2 .L2::128B, 3 .L2::256B (487 MB).
#ifndef OKT_RAND_LD
#define OKT_RAND_LD 1
#endif
__device__ __forceinline__ float ld_rand(const float* p) {
  float v;
#if OKT_RAND_LD == 1
  asm("ld.global.cg.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
#elif OKT_RAND_LD == 2
  asm("ld.global.cg.L2::128B.f32 %0, [%1];" : "=f"(v) : "l"(p));
#elif OKT_RAND_LD == 3
  asm("ld.global.cg.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p));
#else
  v = __ldcg(p);
#endif
  return v;
}

__device__ __forceinline__ uint64_t block_sum(uint64_t v, uint64_t* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  uint64_t t = 0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

// Smallest float f with (double)f >= th (th >= 0): |a| >= th  <=>  |a| >= f for
// every finite float a, so the select predicate runs in fp32.
__device__ __forceinline__ float ceil_to_float(double th) {
  float f = __double2float_rn(th);
  if (double(f) < th) f = nextafterf(f, __int_as_float(0x7f800000));
  return f;
}

__device__ __forceinline__ uint64_t coo_pack(uint32_t idx, float v) {
  return (uint64_t(__float_as_uint(v)) << 32) | uint64_t(idx);
}
__device__ __forceinline__ uint32_t coo_idx(uint64_t e) { return uint32_t(e); }
__device__ __forceinline__ float coo_val(uint64_t e) {
  return __uint_as_float(uint32_t(e >> 32));
}

// The reference's stride-doubling bracket sum (oktopk.cpp sparse_sum over
// the P sources of one coordinate; absent sources leave their bracket slot
// empty) in fp64 over values already in registers; bit r of `bits`: source r
// present.
template <int P>
__device__ __forceinline__ double bracket_regs(const float (&v)[P], uint32_t bits) {
  double a[P];
  bool h[P];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    h[q] = (bits >> q) & 1u;
    a[q] = h[q] ? double(v[q]) : 0.0;
  }
#pragma unroll
  for (int s = P >> 1; s >= 1; s >>= 1) {
#pragma unroll
    for (int q = 0; q < s; ++q) {
      if (h[q] && h[q + s]) a[q] = a[q] + a[q + s];
      else if (h[q + s]) a[q] = a[q + s];
      h[q] = h[q] || h[q + s];
    }
  }
  return a[0];
}
}  // namespace okt
