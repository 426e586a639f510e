// okt_device.cuh — device building blocks shared by the Ok-Topk kernels.
//
// Every order-preserving compaction on the path (local selection, region
// merge, survivor filter, index intersection) is a single-pass decoupled
// look-back scan: a tile publishes its aggregate, one warp walks predecessors
// 32 at a time, and the tile's entries are written straight to their final
// positions.  Tile IDs come from an atomic counter (not blockIdx), so a tile
// only ever waits on tiles already owned by running CTAs: deadlock-free even
// when several ranks' kernels share one GPU.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace okt {

constexpr int kMaxP = 8;                     // ranks per world (one HGX box)
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kJ = 4;                        // groups per thread per tile
constexpr int kC = 4;                        // elements per group (one 16 B vector)
constexpr int kTile = kJ * kC * kThreads;    // 4096 elements per tile
static_assert(kJ * kWarps == 32, "tile scan table must be one warp wide");

// ---- look-back status words --------------------------------------------------
// [63:62] flag (1 = aggregate, 2 = inclusive prefix), [61:32] launch epoch,
// [31:0] value.  Flag, epoch and value travel in one 64-bit store, so no
// fences are needed between them; the epoch makes stale words from earlier
// launches invisible, so the array is never cleared.
constexpr uint64_t kFlagAgg = 1ull;
constexpr uint64_t kFlagPre = 2ull;

__device__ __forceinline__ uint64_t pack_status(uint64_t flag, uint32_t epoch,
                                                uint32_t v) {
  return (flag << 62) | (uint64_t(epoch & 0x3fffffffu) << 32) | uint64_t(v);
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Warp-collective: publish `agg` for `tile` and return the exclusive prefix of
// all earlier tiles.  Every lane returns the same value.
__device__ __forceinline__ uint32_t lookback(uint64_t* status, uint32_t tile,
                                             uint32_t epoch, uint32_t agg) {
  const int lane = threadIdx.x & 31;
  const uint32_t ep = epoch & 0x3fffffffu;
  if (tile == 0) {
    if (lane == 0) st_relaxed(&status[0], pack_status(kFlagPre, epoch, agg));
    return 0;
  }
  if (lane == 0) st_relaxed(&status[tile], pack_status(kFlagAgg, epoch, agg));
  uint32_t excl = 0;
  int64_t pred = int64_t(tile) - 1;
  while (true) {
    const int64_t idx = pred - lane;
    uint32_t flag = uint32_t(kFlagPre), val = 0;
    if (idx >= 0) {
      uint64_t s;
      int spins = 0;
      while (true) {
        s = ld_relaxed(&status[idx]);
        if (uint32_t((s >> 32) & 0x3fffffffu) == ep && (s >> 62) != 0) break;
        if (++spins > 8) __nanosleep(32);
      }
      flag = uint32_t(s >> 62);
      val = uint32_t(s);
    }
    const unsigned pre = __ballot_sync(0xffffffffu, flag == uint32_t(kFlagPre));
    const int first = pre ? (__ffs(pre) - 1) : 32;
    uint32_t contrib = (lane <= first) ? val : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
    excl += contrib;
    if (pre) break;
    pred -= 32;
  }
  if (lane == 0) st_relaxed(&status[tile], pack_status(kFlagPre, epoch, excl + agg));
  return excl;
}

// ---- tile scan ---------------------------------------------------------------
// Element (j, warp, lane, c) of a tile sits at tile offset
// j*kC*kThreads + (warp*32 + lane)*kC + c, so output order is (j, warp, lane, c).
// Each thread passes one ballot per (j, c); the per-(j, warp) counts form a
// 32-entry table that warp 0 scans before the look-back.
struct TileScanSmem {
  uint32_t cnt[kJ * kWarps];
  uint32_t base;
  uint32_t tile;
};

// All threads call.  On return s.base is the tile's exclusive prefix and
// s.cnt[j*kWarps + w] the exclusive offset of (j, w) inside the tile.  The
// CTA that owns the last tile stores the grand total to *d_total.
template <int C>
__device__ __forceinline__ void tile_scan(TileScanSmem& s, const unsigned (&bal)[kJ][C],
                                          uint32_t tile, uint32_t num_tiles,
                                          uint64_t* status, uint32_t epoch,
                                          uint64_t* d_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < C; ++q) c += __popc(bal[j][q]);
      s.cnt[j * kWarps + warp] = c;
    }
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t v = s.cnt[lane];
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = lookback(status, tile, epoch, total);
    s.cnt[lane] = incl - v;
    if (lane == 0) {
      s.base = excl;
      if (tile + 1 == num_tiles && d_total) *d_total = uint64_t(excl) + total;
    }
  }
  __syncthreads();
}

// Rank of element (j, c) of this thread inside its (j, warp) group.
template <int C>
__device__ __forceinline__ uint32_t rank_in_group(const unsigned (&bal)[kJ][C], int j,
                                                  int c) {
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

// Dynamic tile fetch: one atomic per tile on ctr[0]; the last CTA to leave
// resets the counter pair so the next launch on the stream starts at 0.
__device__ __forceinline__ uint32_t fetch_tile(uint32_t* ctr, uint32_t& s_tile) {
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctr[0], 1u);
  __syncthreads();
  const uint32_t t = s_tile;
  __syncthreads();  // every thread has read s_tile before thread 0 may refill it
  return t;
}
__device__ __forceinline__ void retire_cta(uint32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctr[1], 1u) == gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
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

}  // namespace okt
