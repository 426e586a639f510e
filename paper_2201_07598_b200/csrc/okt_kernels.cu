// okt_kernels.cu — sm_100a kernels of the Ok-Topk sparse allreduce.
//
// Everything here is HBM- or latency-bound integer/byte work: 128-bit
// coalesced streaming loads, warp-ballot compaction in two phases (see
// okt_device.cuh), and O(k) scatters.  No tensor cores: nothing on this path
// is a contraction.
//
// Reference functions each kernel replaces (proj/core/src/...):
//   k1_kernel          trainer.cpp:423-435 make_accumulator, sparse.cpp:14-19
//                      all_finite, sparse.cpp:94-106 select_by_threshold(Dense)
//   radix_*            oktopk.cpp:12-26 th_re_evaluate -> sparse.cpp:43-80 topk_from
//   scatter/region_scan sparse.cpp:206-257 sparse_sum (stride-doubling bracket)
//   filter_kernel      sparse.cpp:108-120 select_by_threshold(Sparse)
//   apply_kernel       oktopk.cpp:299-302 set_intersection, trainer.cpp:478-479
//                      residual zero, trainer.cpp:437-442 apply_sparse_update
//   proposals/cuts     oktopk.cpp:28-61 space_repartition
//   slice_offsets      sparse.cpp:190-202 sparse_slice (lower_bound)
#include "okt_device.cuh"
#include "okt_kernels.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>

namespace okt {

namespace {

template <typename K>
int resident_ctas(K kernel, int threads, int sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return per_sm * sms;
}

// First tile of chunk c when `tiles` tiles are split evenly over G chunks:
// floor(c * tiles / G), in 32-bit arithmetic whenever the product fits (the
// 64-bit division is a called subroutine).
__device__ __forceinline__ uint64_t split_at(uint32_t c, uint64_t tiles, uint32_t G) {
  const uint64_t m = uint64_t(c) * tiles;
  return m <= 0xffffffffull ? uint64_t(uint32_t(m) / G) : m / G;
}

// Same, for launches whose host side checked tiles * G < 2^32.
__device__ __forceinline__ uint32_t split_at32(uint32_t c, uint32_t tiles, uint32_t G) { return c * tiles / G; }

__device__ __forceinline__ bool nonfinite(float a) {
  return (__float_as_uint(a) & 0x7f800000u) == 0x7f800000u;
}

uint32_t chunks_for(uint64_t tiles, int resident, int max_chunks) {
  uint64_t g = std::min<uint64_t>(tiles, uint64_t(resident));
  g = std::min<uint64_t>(g, uint64_t(max_chunks));
  return uint32_t(std::max<uint64_t>(g, 1));
}

}  // namespace

size_t stage_entries(uint64_t count, int tile, int max_chunks) {
  return size_t((count + tile - 1) / tile + uint64_t(max_chunks)) * size_t(tile);
}

// =============================================================================
// Phase B: chunk prefix + copy to final positions
// =============================================================================
// MODE 0: AoS u64 -> AoS u64; 1: AoS u64 -> SoA (u32, f32 widened to f64);
//      2: SoA -> SoA; 3: u32 -> u32; 4: SoA (u32, f64 holding an f32) -> AoS u64.
#ifndef OKT_COMPACT_BATCH
#define OKT_COMPACT_BATCH 4
#endif
constexpr int kCompactBatch = OKT_COMPACT_BATCH;

// A CTA copies a group of consecutive chunks (up to kThreads; one chunk per
// CTA for the static-chunk producers, a few tiles for K1's per-tile staging):
// the group's counts are block-scanned, the group total is published in
// agg[blockIdx.x] (tagged with the launch), and the group's exclusive prefix is
// the sum of the lower CTAs' published totals (a decoupled look-back over
// aggregates only: every CTA publishes before it waits, and the grid is one
// wave, so nobody waits on a CTA that waits).  The group's first entries are
// loaded while the look-back completes.  Round 1 summed every lower chunk
// count per CTA instead (O(G^2 / per) L2 reads: 0.28 ms at 340M).
__device__ __forceinline__ void agg_publish(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t agg_load(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// APPLY (P = 1 EF step, MODE 1): the model half of K7 on every entry of u,
// w[i] = float(double(w[i]) - v) (trainer.cpp:437-442, P = 1; K1 already
// zeroed the residual); skipped when K1 met a non-finite accumulator (the
// reference throws before touching the model).  Entries go in batches of
// kCompactBatch per thread: staging loads, then the model gathers, then the
// stores, so every random access of the batch is in flight together.
template <int MODE, bool APPLY>
__global__ void __launch_bounds__(kThreads)
    compact_kernel(const uint64_t* __restrict__ s64, const uint32_t* __restrict__ sidx,
                   const double* __restrict__ sval, const uint32_t* __restrict__ counts,
                   const uint32_t* __restrict__ counts2, uint32_t g2, uint32_t G, uint64_t cap_host,
                   const uint64_t* d_cap, uint64_t* __restrict__ o64, uint32_t* oidx, double* oval,
                   uint64_t* d_total, uint64_t* d_total2, uint64_t* agg, ApplyArgs ap) {
  __shared__ uint64_t red[kWarps];
  __shared__ uint32_t s_pre[kThreads + 1];
  __shared__ uint32_t s_wt[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    trace_stamp(ap.trace, kTrCompact, 0);
    if (blockIdx.x == 0 && ap.d_flags_next) *ap.d_flags_next = 0;  // (nobody uses it during this step)
  }
  const uint32_t c0 = uint32_t(split_at(blockIdx.x, G, gridDim.x));
  const uint32_t c1 = uint32_t(split_at(blockIdx.x + 1, G, gridDim.x));
  const int nc = int(c1 - c0);
  const uint64_t cap = d_cap ? *d_cap : cap_host;
  // group prefix (block scan)
  const uint32_t v = tid < nc ? counts[c0 + tid] : 0u;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_wt[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) wpre += (w < warp) ? s_wt[w] : 0u;
  if (tid < nc) s_pre[tid + 1] = wpre + incl;
  if (tid == 0) s_pre[0] = 0;
  __syncthreads();
  const uint64_t cnt = s_pre[nc];
  const uint64_t tag = uint64_t(ap.tag) << 32;
  if (tid == 0) agg_publish(&agg[blockIdx.x], tag | cnt);
  if (tid == 0) trace_stamp(ap.trace, kTrCompact, 1);
  auto src_of = [&](uint64_t j) {  // staging position of the group's j-th entry
    int lo = 0, hi = nc - 1;          // last k with s_pre[k] <= j
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= j) lo = mid;
      else hi = mid - 1;
    }
    OKT_DCHECK(j - s_pre[lo] < cap, "compact: entry beyond its chunk", j - s_pre[lo], cap);
    return uint64_t(c0 + lo) * cap + (j - s_pre[lo]);
  };
  constexpr int B = kCompactBatch;
  uint64_t e64[B];
  uint32_t ei[B];
  double ev[B];
  float wv[B];
  auto load_batch = [&](uint64_t j0) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint64_t j = j0 + uint64_t(b) * kThreads;
      e64[b] = 0;
      ei[b] = 0;
      ev[b] = 0.0;
      if (j < cnt) {
        const uint64_t sj = src_of(j);
        if (MODE == 0 || MODE == 1) e64[b] = s64[sj];
        if (MODE == 2 || MODE == 3 || MODE == 4) ei[b] = sidx[sj];
        if (MODE == 2 || MODE == 4) ev[b] = sval[sj];
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (MODE == 1) {
        ei[b] = coo_idx(e64[b]);
        ev[b] = double(coo_val(e64[b]));
      }
      // (L2-only 4-byte gathers: through L1 each random word pulled a whole
      // 128-byte line from DRAM — 445 MB read for 3.4M words at 340M, ncu)
      wv[b] = (APPLY && j0 + uint64_t(b) * kThreads < cnt) ? ld_rand(ap.w + ei[b]) : 0.f;
    }
  };
  // The first batch is loaded before the global prefix is known: only the
  // output positions depend on it.
  load_batch(tid);
  // look-back over the lower CTAs' group totals of this launch
  uint64_t pre = 0;
  for (uint32_t b = tid; b < blockIdx.x; b += kThreads) {
    uint64_t a;
    do {
      a = agg_load(&agg[b]);
    } while ((a & 0xffffffff00000000ull) != tag);
    pre += uint32_t(a);
  }
  pre = block_sum(pre, red);
  if (tid == 0) trace_stamp(ap.trace, kTrCompact, 3);
  const bool last = blockIdx.x == gridDim.x - 1;
  if (last) {  // the totals (and the step's scalars, straight into mapped host memory: no D2H node)
    uint64_t s2 = counts2 ? strided_sum(counts2, g2) : 0;
    if (counts2) s2 = block_sum(s2, red);
    if (tid == 0) {
      *d_total = pre + cnt;
      if (counts2) *d_total2 = s2;
      if (ap.hout) {
        ap.hout->m = counts2 ? s2 : 0;
        ap.hout->S = pre + cnt;
        ap.hout->flags = *reinterpret_cast<volatile uint32_t*>(ap.d_flags);  // (K1 has finished)
        ap.hout->seq = ap.seq;
      }
    }
  }
  const bool skip = APPLY && (*ap.d_flags & 1u);  // non-finite step: the model stays as it was
  bool bad = false;
  for (uint64_t j0 = tid;; j0 += uint64_t(B) * kThreads) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint64_t j = j0 + uint64_t(b) * kThreads;
      if (j >= cnt) continue;
      if (MODE == 0) o64[pre + j] = e64[b];
      else if (MODE == 4) o64[pre + j] = coo_pack(ei[b], float(ev[b]));
      else if (MODE == 3) oidx[pre + j] = ei[b];
      else {
        oidx[pre + j] = ei[b];
        oval[pre + j] = ev[b];
      }
      if (APPLY && !skip) {
        const float nw = float(double(wv[b]) - ev[b]);
        ap.w[ei[b]] = nw;
        bad |= nonfinite(nw);
      }
    }
    if (j0 + uint64_t(B) * kThreads >= cnt) break;
    load_batch(j0 + uint64_t(B) * kThreads);
  }
  if (APPLY && __syncthreads_or(bad) && tid == 0) {
    atomicOr(ap.d_flags, 4u);
    if (ap.hout) *reinterpret_cast<volatile uint32_t*>(&ap.hout->bad_iter) = 1u;  // (error path only)
  }
  if (lane == 0) trace_stamp(ap.trace, kTrCompact, 2);
}

const void* compact_graph_kernel(bool apply) {
  return apply ? reinterpret_cast<const void*>(compact_kernel<1, true>)
               : reinterpret_cast<const void*>(compact_kernel<1, false>);
}

// G chunks of `cap` entries (cap_host, or *d_cap when set); counts2: g2
// partial sums (0 = none).
template <int MODE>
static cudaError_t launch_compact(Launch& L, const Stage& S, uint32_t G, uint64_t cap_host,
                                  const uint64_t* d_cap, uint32_t g2, uint64_t* o64, uint32_t* oidx,
                                  double* oval, uint64_t* d_total, uint64_t* d_total2,
                                  const ApplyArgs* ap = nullptr) {
  // one chunk per CTA while the grid fits one wave, then groups of up to
  // kThreads chunks; the grid never exceeds one wave (the look-back waits on
  // lower CTAs)
  static std::atomic<int> cap{0};  // (resident CTAs; benign concurrent first use)
  if (!cap) cap = resident_ctas(compact_kernel<MODE, true>, kThreads, L.sms);
  const uint32_t slots = uint32_t(std::min(cap.load(), S.max_chunks));
  const uint32_t per = std::min<uint32_t>(kThreads, std::max<uint32_t>(1, (G + slots - 1) / slots));
  const uint32_t GB = std::max<uint32_t>(1, (G + per - 1) / per);
  const uint32_t* c2 = g2 ? S.counts2 : nullptr;
  ApplyArgs a = ap ? *ap : ApplyArgs{};
  if (!a.tag) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(L.s, &cs);
    if (cs == cudaStreamCaptureStatusActive) {
      // captured into a graph, the launch's arguments (its tag) repeat at every
      // replay: clear the look-back words in the graph first and use tag 1
      // (the counter below starts at 2, so no direct launch reuses it)
      const cudaError_t e = cudaMemsetAsync(S.agg, 0, sizeof(uint64_t) * GB, L.s);
      if (e != cudaSuccess) return e;
      a.tag = 1;
    } else {
      a.tag = ++*S.tag_ctr;
      if (a.tag < 2) a.tag = *S.tag_ctr = 2;  // (0 never tags a launch; 1 is the graphs')
    }
  }
  if (MODE == 1 && a.k7)
    compact_kernel<MODE, true><<<GB, kThreads, 0, L.s>>>(S.s64, S.sidx, S.sval, S.counts, c2, g2, G, cap_host, d_cap,
                                                         o64, oidx, oval, d_total, d_total2, S.agg, a);
  else
    compact_kernel<MODE, false><<<GB, kThreads, 0, L.s>>>(S.s64, S.sidx, S.sval, S.counts, c2, g2, G, cap_host, d_cap,
                                                          o64, oidx, oval, d_total, d_total2, S.agg, a);
  ++L.launches;
  return cudaGetLastError();
}

// =============================================================================
// K1: fused accumulate / select / compact (phase A)
// =============================================================================
// APPLY (single rank, DUAL): u = the emitted set, and every entry of u is in
// the local selection (indexes = u), so the residual half of K7 runs here, in
// the tile that emits the entry: the residual word is stored as 0 instead of
// acc (trainer.cpp:478-479; no extra bytes on the ACCUM pass, a 4-byte store
// per entry on the select-only refresh pass).  The residual buffer written
// here is committed only when the step succeeds.  The model half (w -= u)
// stays in phase B, after the whole grid's finiteness is known: a model
// update inside K1 put a dependent DRAM round trip into every tile and
// slowed K1 from 0.60 to 1.02 ms at n = 340M (round-2 launch list).
template <bool ACCUM, bool SELECT, bool HIST, bool VEC, bool DUAL, bool APPLY>
__global__ void __launch_bounds__(kThreads, VEC ? 4 : 3)
    k1_kernel(const float* __restrict__ g, const float* eps_in, float* eps_out, float alpha, uint64_t n,
              uint32_t tiles, uint32_t* tile_ctr, const double* __restrict__ d_th,
              const double* __restrict__ d_th2, uint64_t* __restrict__ stg, uint32_t* counts,
              uint32_t* counts2, uint32_t* d_flags, uint32_t* d_hist, const StepPtrs* ind, K1P2P p2p, K1Apply ka) {
  static_assert(!APPLY || (DUAL && SELECT), "the fused apply is the single-rank dual-threshold select");
  constexpr int C = 4, TILE = kJ * C * kThreads;
  // Tiles are handed out dynamically (a ticket counter; the prefetched next
  // ticket hides its round trip), so every CTA streams until the input is
  // exhausted instead of a statically assigned range finishing unevenly.
  // Each tile compacts its selected entries into its own staging slot
  // [tile * TILE, ...) with its count in counts[tile]: the tile order is the
  // coordinate order, whichever CTA ran the tile.
  // P2P mode: the staging, the counts and, per tile, the number of entries
  // below every cut live in this rank's window; peers read each tile's slice
  // for their region in place ([lt[t][r], lt[t][r+1])).
  __shared__ uint64_t s_cut[kMaxP];
  __shared__ uint32_t s_below[2][kMaxP];
  __shared__ uint32_t s_tile[2];
  // (the P2P path always runs the vectorised, single-threshold variants)
  const bool p2p_on = VEC && !DUAL && p2p.tab != nullptr;
  const int lt_P = p2p_on ? p2p.tab->P : 0;
  const int me_rank = p2p_on ? p2p.tab->rank : 0;
  uint32_t* lt_out = nullptr;
  const int p2p_par = p2p_on ? (p2p.par_v >= 0 ? p2p.par_v : p2p.sp->par) : 0;
  if (p2p_on && p2p.sp_out && blockIdx.x == 0) {
    // argument-fed step: publish the step block for the later kernels of the
    // step (they start after this grid) and clear the plan
    if (threadIdx.x == 0) *p2p.sp_out = p2p.spv;
    uint32_t* pz = reinterpret_cast<uint32_t*>(p2p.plan_zero);
    for (int i = threadIdx.x; i < int(sizeof(P2PPlan) / 4); i += blockDim.x) pz[i] = 0u;
  }
  if (p2p_on) {
    const int me = p2p.tab->rank, par = p2p_par;
    stg = p2p.tab->kstg[me][par];
    counts = p2p.tab->kcnt[me][par];
    lt_out = p2p.tab->klt[me][par];
    if (threadIdx.x < lt_P) {
      s_cut[threadIdx.x] = p2p.cuts[threadIdx.x];
      s_below[0][threadIdx.x] = 0;
      s_below[1][threadIdx.x] = 0;
    }
  }
  uint64_t* const trace = p2p_on ? p2p.tab->trace : (ind ? ind->trace : nullptr);
  if (trace && threadIdx.x == 0) trace_stamp(trace, kTrK1, 0);
  if (ind) {
    g = ind->g;
    eps_in = ind->eps_in;
    eps_out = ind->eps_out;
    alpha = ind->alpha;
  }
  __shared__ uint32_t tbl[2][32];
  __shared__ uint32_t s_hist[HIST ? 2048 : 1];
  __shared__ uint64_t red[kWarps];
  const int tid = threadIdx.x;
  float tf = 0.f, tf_loc = 0.f;
  if (SELECT) {
    const double lth = *d_th;
    tf_loc = ceil_to_float(lth);
    tf = DUAL ? ceil_to_float(fmax(lth, *d_th2)) : tf_loc;
  }
  if (HIST) {
    for (int i = tid; i < 2048; i += kThreads) s_hist[i] = 0;
    __syncthreads();
  }
  bool bad = false;
  uint32_t mloc = 0;
  // P2P: this CTA's share of the totals, slot d < P (below cut d) kept by
  // thread d, slot kMaxP (all) by thread 0 (in shared memory: K1's P2P
  // variant is at its 64-register cap; < 2^32 — fewer entries than n < 2^32)
  __shared__ uint32_t s_tot[kMaxP + 1];
  if (tid <= kMaxP) s_tot[tid] = 0;  // (each slot read and written by one thread only)
  if (tid == 0) s_tile[0] = atomicAdd(&tile_ctr[0], 1u);
  __syncthreads();
  for (int parity = 0;; parity ^= 1) {
    const uint32_t tile = s_tile[parity];
    if (tile >= tiles) break;
    // next ticket, read after this tile's barrier
    if (tid == 0) s_tile[parity ^ 1] = atomicAdd(&tile_ctr[0], 1u);
    const uint64_t base = uint64_t(tile) * TILE;
    uint64_t* out = stg + base;
    float a[kJ][C];
    bool valid[kJ][C];
    if (VEC && base + TILE <= n) {
      float4 gv[kJ], ev[kJ];
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const uint64_t e0 = base + uint64_t(j) * (C * kThreads) + uint64_t(tid) * C;
        gv[j] = __ldcs(reinterpret_cast<const float4*>(g + e0));
        if (ACCUM) ev[j] = __ldcs(reinterpret_cast<const float4*>(eps_in + e0));
      }
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        if (ACCUM) {
          a[j][0] = fmaf(alpha, gv[j].x, ev[j].x);
          a[j][1] = fmaf(alpha, gv[j].y, ev[j].y);
          a[j][2] = fmaf(alpha, gv[j].z, ev[j].z);
          a[j][3] = fmaf(alpha, gv[j].w, ev[j].w);
          const uint64_t e0 = base + uint64_t(j) * (C * kThreads) + uint64_t(tid) * C;
          float4 st = make_float4(a[j][0], a[j][1], a[j][2], a[j][3]);
          if (APPLY || (p2p_on && p2p.zero_sel)) {  // the residual of an entry of u / the local selection is 0
            if (fabsf(st.x) >= tf) st.x = 0.f;
            if (fabsf(st.y) >= tf) st.y = 0.f;
            if (fabsf(st.z) >= tf) st.z = 0.f;
            if (fabsf(st.w) >= tf) st.w = 0.f;
          }
          // (single rank: nothing reads the residual again this step -> streaming store)
          if (APPLY) __stcs(reinterpret_cast<float4*>(eps_out + e0), st);
          else *reinterpret_cast<float4*>(eps_out + e0) = st;
        } else {
          a[j][0] = gv[j].x;
          a[j][1] = gv[j].y;
          a[j][2] = gv[j].z;
          a[j][3] = gv[j].w;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          valid[j][c] = true;
          bad |= nonfinite(a[j][c]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const uint64_t e = base + uint64_t(j) * (C * kThreads) + uint64_t(tid) * C + c;
          valid[j][c] = e < n;
          float x = 0.f;
          if (valid[j][c]) {
            x = g[e];
            if (ACCUM) {
              x = fmaf(alpha, x, eps_in[e]);
              eps_out[e] = ((APPLY || (p2p_on && p2p.zero_sel)) && fabsf(x) >= tf) ? 0.f : x;
            }
            bad |= nonfinite(x);
          }
          a[j][c] = x;
        }
      }
    }
    if (HIST) {
#pragma unroll
      for (int j = 0; j < kJ; ++j)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (valid[j][c]) atomicAdd(&s_hist[(__float_as_uint(a[j][c]) & 0x7fffffffu) >> 20], 1u);
    }
    if (SELECT) {
      unsigned bal[kJ][C];
      bool pred[kJ][C];
#pragma unroll
      for (int j = 0; j < kJ; ++j)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float m = fabsf(a[j][c]);
          pred[j][c] = valid[j][c] && m >= tf;
          if (DUAL) mloc += (valid[j][c] && m >= tf_loc) ? 1u : 0u;
          bal[j][c] = __ballot_sync(0xffffffffu, pred[j][c]);
        }
      // A cut inside this tile: the entries below it are a prefix of the
      // tile's order, counted here (warp reduce + one smem add per warp).
      uint32_t cut_mask = 0;
      if (p2p_on) {
        for (int d = 0; d < lt_P; ++d) {
          const uint64_t cut = s_cut[d];
          if (cut >= base && cut < base + TILE) {
            cut_mask |= 1u << d;
            uint32_t below = 0;
#pragma unroll
            for (int j = 0; j < kJ; ++j)
#pragma unroll
              for (int c = 0; c < C; ++c)
                below += (pred[j][c] && base + uint64_t(j) * (C * kThreads) + uint64_t(tid) * C + c < cut) ? 1u : 0u;
            below = __reduce_add_sync(0xffffffffu, below);
            if ((tid & 31) == 0 && below) atomicAdd(&s_below[parity][d], below);
          }
        }
      }
      uint32_t grp[kJ];
      const uint32_t total = tile_offsets<C>(tbl[parity], bal, grp);
      if (tid == 0) counts[tile] = total;
      if (tid < lt_P) {
        // a cut inside the tile: the count below it; else all or nothing
        const uint32_t below = ((cut_mask >> tid) & 1u) ? s_below[parity][tid] : (s_cut[tid] <= base ? 0u : total);
        lt_out[uint64_t(tile) * kMaxP + tid] = below;
        s_tot[tid] += below;
        if (tid == 0) s_tot[kMaxP] += total;
        s_below[parity][tid] = 0;  // reused two tiles later, after two barriers
      }
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if (pred[j][c]) {
            const uint32_t pos = grp[j] + rank_in_group<C>(bal, j, c);
            OKT_DCHECK(pos < uint32_t(TILE), "k1: staged position beyond the tile", pos, tile);
            const uint64_t e = base + uint64_t(j) * (C * kThreads) + uint64_t(tid) * C + c;
            out[pos] = coo_pack(uint32_t(e), a[j][c]);
            if (APPLY && !ACCUM) ka.zero[e] = 0.f;
          }
        }
      }
    } else {
      __syncthreads();  // orders the next-ticket write (SELECT: inside tile_offsets)
    }
  }
  if (DUAL) {
    const uint64_t s = block_sum(mloc, red);
    if (tid == 0) counts2[blockIdx.x] = uint32_t(s);
  }
  if (p2p_on && p2p.tot_acc && tid < lt_P) {
    if (s_tot[tid]) atomicAdd(reinterpret_cast<unsigned long long*>(&p2p.tot_acc[tid]), (unsigned long long)s_tot[tid]);
    if (tid == 0 && s_tot[kMaxP])
      atomicAdd(reinterpret_cast<unsigned long long*>(&p2p.tot_acc[kMaxP]), (unsigned long long)s_tot[kMaxP]);
  }
  if (__syncthreads_or(bad) && tid == 0) {
    atomicOr(d_flags, 1u);
  }
  if (HIST) {
    for (int i = tid; i < 2048; i += kThreads)
      if (s_hist[i]) atomicAdd(&d_hist[i], s_hist[i]);
  }
  if (tid == 0) {
    // the last CTA out re-arms the ticket counter for the next launch
    __threadfence();
    if (atomicAdd(&tile_ctr[1], 1u) == gridDim.x - 1) {
      tile_ctr[0] = 0;
      tile_ctr[1] = 0;
      if (p2p_on && p2p.tot_acc) {
        // every CTA's counts are in: publish the totals (and clear them)
        const uint64_t all = atomicExch(reinterpret_cast<unsigned long long*>(&p2p.tot_acc[kMaxP]), 0ull);
        for (int d = 0; d <= lt_P; ++d) {
          const uint64_t o = d < lt_P ? atomicExch(reinterpret_cast<unsigned long long*>(&p2p.tot_acc[d]), 0ull) : all;
          p2p.d_off[d] = o;
          if (p2p.hout) p2p.hout->off[d] = o;
        }
        *p2p.d_m = all;
        if (p2p.hout) {
          p2p.hout->m = all;
          p2p.hout->seq_tot = p2p.par_v >= 0 ? p2p.spv.epoch : p2p.sp->epoch;
        }
      }
      __threadfence();
    }
  }
  if (p2p_on && blockIdx.x == 0 && tid == 0) {
    // Chunk geometry for the peers; the status and the L-ready flags are
    // published by the next kernel on the stream (the P2P scatter) once every
    // CTA of this one has finished: a system fence issued here, while the grid
    // still streams, would wait for that traffic to drain (tools/fence_lat.cu).
    P2PPub* pub = &p2p.tab->hdr[me_rank]->pub[p2p_par];
    pub->k1_G = tiles;  // chunk = tile
    pub->k1_cap = TILE;
  }
  if (trace && (tid & 31) == 0) trace_stamp(trace, kTrK1, 2);
}

template <bool ACCUM, bool SELECT, bool HIST, bool DUAL, bool APPLY = false>
static cudaError_t k1_dispatch(Launch& L, const Stage& S, bool vec, const float* g, const float* eps_in,
                               float* eps_out, float alpha, uint64_t n, const double* d_th,
                               const double* d_th2, const OutCoo& out, uint64_t* d_m, uint64_t* d_m2,
                               uint32_t* d_flags, uint32_t* d_hist, const ApplyArgs* ap, const K1P2P* p2p,
                               const StepPtrs* ind) {
  constexpr int TILE = kJ * 4 * kThreads;
  const uint64_t tiles = (n + TILE - 1) / TILE;
  auto kern = vec ? k1_kernel<ACCUM, SELECT, HIST, true, DUAL, APPLY> : k1_kernel<ACCUM, SELECT, HIST, false, DUAL, APPLY>;
  K1Apply ka{};
  if (APPLY) ka.zero = ACCUM ? nullptr : const_cast<float*>(g);  // the select-only pass reads acc in place
  static std::atomic<int> cap_v{0}, cap_s{0};
  std::atomic<int>& cap = vec ? cap_v : cap_s;
  if (!cap) cap = resident_ctas(kern, kThreads, L.sms);
  const uint32_t G = chunks_for(tiles, cap, S.max_chunks);  // persistent CTAs
  if (tiles > S.max_tiles) return cudaErrorInvalidValue;         // counts / staging capacity
  // Profiling events: inside a stream capture they must be external event
  // nodes (re-recorded at every graph launch); outside, plain records.
  cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
  if (L.k1_event) cudaStreamIsCapturing(L.s, &cap_st);
  const unsigned ev_flags = cap_st == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  if (L.k1_event) cudaEventRecordWithFlags(L.k1_event(L.k1_ctx), L.s, ev_flags);
  kern<<<G, kThreads, 0, L.s>>>(g, eps_in, eps_out, alpha, n, uint32_t(tiles), S.tile_ctr, d_th, d_th2, S.s64,
                                S.counts, S.counts2, d_flags, d_hist, ind, p2p ? *p2p : K1P2P{}, ka);
  if (L.k1_event) cudaEventRecordWithFlags(L.k1_event(L.k1_ctx), L.s, ev_flags);
  ++L.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !SELECT) return e;
  if (p2p) return cudaSuccess;  // peers consume the per-tile staging in place
  // chunks = tiles; counts2 holds one partial sum per K1 CTA
  if (out.aos)
    return launch_compact<0>(L, S, uint32_t(tiles), TILE, nullptr, DUAL ? G : 0, out.aos, nullptr, nullptr, d_m, d_m2);
  return launch_compact<1>(L, S, uint32_t(tiles), TILE, nullptr, DUAL ? G : 0, nullptr, out.idx, out.val, d_m, d_m2,
                           ap);
}

cudaError_t launch_k1(Launch& L, const Stage& S, K1Mode mode, const float* g, const float* eps_in,
                      float* eps_out, float alpha, uint64_t n, const double* d_th, const double* d_th2,
                      const OutCoo& out, uint64_t* d_m, uint64_t* d_m2, uint32_t* d_flags, uint32_t* d_hist,
                      const ApplyArgs* ap, const K1P2P* pub, const StepPtrs* ind) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool vec = al(g);
  if (mode != K1Mode::kSelect) vec = vec && al(eps_in) && al(eps_out);
  const bool dual = d_th2 != nullptr;
  const bool apply = dual && ap && ap->k7;  // K7 fused into the single-rank select (K1Apply)
  if (apply && mode == K1Mode::kSelect)
    return k1_dispatch<false, true, false, true, true>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out, d_m,
                                                       d_m2, d_flags, d_hist, ap, pub, ind);
  if (apply && mode == K1Mode::kAccumSelect)
    return k1_dispatch<true, true, false, true, true>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out, d_m,
                                                      d_m2, d_flags, d_hist, ap, pub, ind);
  switch (mode) {
    case K1Mode::kSelect:
      return dual ? k1_dispatch<false, true, false, true>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out,
                                                           d_m, d_m2, d_flags, d_hist, ap, pub, ind)
                  : k1_dispatch<false, true, false, false>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2,
                                                            out, d_m, d_m2, d_flags, d_hist, ap, pub, ind);
    case K1Mode::kAccumSelect:
      return dual ? k1_dispatch<true, true, false, true>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out,
                                                          d_m, d_m2, d_flags, d_hist, ap, pub, ind)
                  : k1_dispatch<true, true, false, false>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out,
                                                           d_m, d_m2, d_flags, d_hist, ap, pub, ind);
    case K1Mode::kAccumHist:
      return k1_dispatch<true, false, true, false>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out, d_m,
                                                   d_m2, d_flags, d_hist, ap, pub, ind);
    case K1Mode::kAccumSelectHist:
      return k1_dispatch<true, true, true, false>(L, S, vec, g, eps_in, eps_out, alpha, n, d_th, d_th2, out, d_m,
                                                  d_m2, d_flags, d_hist, ap, pub, ind);
  }
  return cudaErrorInvalidValue;
}

// =============================================================================
// Survivor filter and K7 apply (COO lists whose length lives on the device)
// =============================================================================
constexpr int kTileK = kJ * kThreads;  // 1024 entries per tile for the O(k) passes

template <bool AOS>
__global__ void __launch_bounds__(kThreads)
    filter_kernel(const uint64_t* __restrict__ in_aos, const uint32_t* __restrict__ in_idx,
                  const double* __restrict__ in_val, const uint64_t* d_cnt_in, const double* d_th,
                  uint32_t* __restrict__ sidx, double* __restrict__ sval, uint32_t* counts,
                  uint64_t* d_cap) {
  __shared__ uint32_t tbl[2][32];
  const int tid = threadIdx.x;
  const uint64_t cnt = *d_cnt_in;
  const double th = *d_th;
  const uint64_t tiles = (cnt + kTileK - 1) / kTileK;
  const uint64_t tpc = (tiles + gridDim.x - 1) / gridDim.x;
  if (blockIdx.x == 0 && tid == 0) *d_cap = tpc * kTileK;
  const uint64_t t0 = split_at(blockIdx.x, tiles, gridDim.x), t1 = split_at(blockIdx.x + 1, tiles, gridDim.x);
  const uint64_t obase = uint64_t(blockIdx.x) * tpc * kTileK;
  uint32_t running = 0;
  int parity = 0;
  for (uint64_t tile = t0; tile < t1; ++tile, parity ^= 1) {
    uint32_t idx[kJ];
    double val[kJ];
    unsigned bal[kJ][1];
    bool pred[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const uint64_t e = tile * kTileK + uint64_t(j) * kThreads + tid;
      const bool valid = e < cnt;
      idx[j] = 0;
      val[j] = 0.0;
      if (valid) {
        if (AOS) {
          const uint64_t x = in_aos[e];
          idx[j] = coo_idx(x);
          val[j] = double(coo_val(x));
        } else {
          idx[j] = in_idx[e];
          val[j] = in_val[e];
        }
      }
      pred[j] = valid && fabs(val[j]) >= th;
      bal[j][0] = __ballot_sync(0xffffffffu, pred[j]);
    }
    uint32_t grp[kJ];
    const uint32_t total = tile_offsets<1>(tbl[parity], bal, grp);
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (pred[j]) {
        const uint64_t pos = obase + running + grp[j] + rank_in_group<1>(bal, j, 0);
        sidx[pos] = idx[j];
        sval[pos] = val[j];
      }
    running += total;
  }
  if (tid == 0) counts[blockIdx.x] = running;
}

cudaError_t launch_filter(Launch& L, const Stage& S, bool aos, const uint64_t* in_aos, const uint32_t* in_idx,
                          const double* in_val, const uint64_t* d_cnt_in, uint64_t bound, const double* d_th,
                          uint32_t* out_idx, double* out_val, uint64_t* d_cnt_out, const ApplyArgs* ap,
                          uint64_t* out_aos) {
  static std::atomic<int> cap_a{0}, cap_s{0};
  std::atomic<int>& cap = aos ? cap_a : cap_s;
  if (!cap) cap = aos ? resident_ctas(filter_kernel<true>, kThreads, L.sms)
                      : resident_ctas(filter_kernel<false>, kThreads, L.sms);
  const uint32_t G = chunks_for((bound + kTileK - 1) / kTileK, cap, S.max_chunks);
  if (aos)
    filter_kernel<true><<<G, kThreads, 0, L.s>>>(in_aos, in_idx, in_val, d_cnt_in, d_th, S.sidx, S.sval, S.counts,
                                                 S.chunk_cap);
  else
    filter_kernel<false><<<G, kThreads, 0, L.s>>>(in_aos, in_idx, in_val, d_cnt_in, d_th, S.sidx, S.sval, S.counts,
                                                  S.chunk_cap);
  ++L.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (out_aos) return launch_compact<4>(L, S, G, 0, S.chunk_cap, 0, out_aos, nullptr, nullptr, d_cnt_out, nullptr, ap);
  return launch_compact<2>(L, S, G, 0, S.chunk_cap, 0, nullptr, out_idx, out_val, d_cnt_out, nullptr, ap);
}

// K7 where every entry of u is in the local selection (one rank: indexes = u):
// eps[i] = 0 and w[i] -= v for each entry, with no gather of acc to test the
// selection and no index list to compact (the caller's indexes are u's).
__global__ void __launch_bounds__(kThreads)
    apply_u_kernel(const uint32_t* __restrict__ u_idx, const double* __restrict__ u_val, const uint64_t* d_U,
                   float* acc, float* w, uint32_t* d_flags) {
  if (*d_flags & 1u) return;  // a non-finite step touches nothing
  const uint64_t cnt = *d_U;
  constexpr int B = 4;
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  bool bad = false;
  for (uint64_t e0 = uint64_t(blockIdx.x) * kThreads + threadIdx.x; e0 < cnt; e0 += B * stride) {
    uint32_t i[B];
    double v[B];
    float wv[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint64_t e = e0 + uint64_t(b) * stride;
      i[b] = e < cnt ? u_idx[e] : 0u;
      v[b] = e < cnt ? u_val[e] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < B; ++b) wv[b] = e0 + uint64_t(b) * stride < cnt ? ld_rand(w + i[b]) : 0.f;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (e0 + uint64_t(b) * stride >= cnt) continue;
      const float nw = float(double(wv[b]) - v[b]);
      w[i[b]] = nw;
      acc[i[b]] = 0.f;
      bad |= nonfinite(nw);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(d_flags, 4u);
}

cudaError_t launch_apply_u(Launch& L, const uint32_t* u_idx, const double* u_val, const uint64_t* d_U, uint64_t bound,
                           float* acc, float* w, uint32_t* d_flags) {
  const uint64_t want = (bound + kThreads * 4 - 1) / (kThreads * 4);
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(L.sms) * 8)));
  apply_u_kernel<<<grid, kThreads, 0, L.s>>>(u_idx, u_val, d_U, acc, w, d_flags);
  ++L.launches;
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads)
    apply_kernel(const uint32_t* __restrict__ u_idx, const double* __restrict__ u_val, const uint64_t* d_U,
                 float* acc, int zero_eps, float* w, int P, const double* d_local_th,
                 uint32_t* __restrict__ sidx, uint32_t* counts, uint64_t* d_cap, uint32_t* d_flags) {
  __shared__ uint32_t tbl[2][32];
  const int tid = threadIdx.x;
  // A step whose input was non-finite applies nothing (the reference throws
  // before touching the residual or the model).
  const bool skip = (*d_flags & (1u | 8u | 16u)) != 0;  // own or a peer's failure
  const uint64_t cnt = skip ? 0 : *d_U;
  const float tf = ceil_to_float(*d_local_th);
  const double dP = double(P);
  const uint64_t tiles = (cnt + kTileK - 1) / kTileK;
  const uint64_t tpc = (tiles + gridDim.x - 1) / gridDim.x;
  if (blockIdx.x == 0 && tid == 0) *d_cap = tpc * kTileK;
  const uint64_t t0 = split_at(blockIdx.x, tiles, gridDim.x), t1 = split_at(blockIdx.x + 1, tiles, gridDim.x);
  const uint64_t obase = uint64_t(blockIdx.x) * tpc * kTileK;
  uint32_t running = 0;
  bool bad = false;
  int parity = 0;
  for (uint64_t tile = t0; tile < t1; ++tile, parity ^= 1) {
    uint32_t idx[kJ];
    double val[kJ];
    bool valid[kJ];
    float av[kJ], wv[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const uint64_t e = tile * kTileK + uint64_t(j) * kThreads + tid;
      valid[j] = e < cnt;
      idx[j] = valid[j] ? u_idx[e] : 0u;
      val[j] = valid[j] ? u_val[e] : 0.0;
    }
    // Issue every gather before any store: acc and w never alias, and the
    // entries of u are distinct, so all 2*kJ loads can be in flight together.
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      av[j] = valid[j] ? ld_rand(acc + idx[j]) : 0.f;  // (L2-only random gathers)
      wv[j] = (valid[j] && w) ? ld_rand(w + idx[j]) : 0.f;
    }
    unsigned bal[kJ][1];
    bool pred[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      pred[j] = valid[j] && fabsf(av[j]) >= tf;
      if (valid[j]) {
        if (w) {
          const float nw = float(double(wv[j]) - val[j] / dP);
          w[idx[j]] = nw;
          bad |= nonfinite(nw);
        }
        if (zero_eps && pred[j]) acc[idx[j]] = 0.f;
      }
      bal[j][0] = __ballot_sync(0xffffffffu, pred[j]);
    }
    uint32_t grp[kJ];
    const uint32_t total = tile_offsets<1>(tbl[parity], bal, grp);
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (pred[j]) sidx[obase + running + grp[j] + rank_in_group<1>(bal, j, 0)] = idx[j];
    running += total;
  }
  if (tid == 0) counts[blockIdx.x] = running;
  if (__syncthreads_or(bad) && tid == 0) atomicOr(d_flags, 4u);
}

cudaError_t launch_apply(Launch& L, const Stage& S, const uint32_t* u_idx, const double* u_val, const uint64_t* d_U,
                         uint64_t bound, float* acc, bool zero_eps, float* w, int P, const double* d_local_th,
                         uint32_t* out_indexes, uint64_t* d_nidx, uint32_t* d_flags) {
  static std::atomic<int> cap{0};
  if (!cap) cap = resident_ctas(apply_kernel, kThreads, L.sms);
  const uint32_t G = chunks_for((bound + kTileK - 1) / kTileK, cap, S.max_chunks);
  apply_kernel<<<G, kThreads, 0, L.s>>>(u_idx, u_val, d_U, acc, zero_eps ? 1 : 0, w, P, d_local_th, S.sidx, S.counts,
                                        S.chunk_cap, d_flags);
  ++L.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_compact<3>(L, S, G, 0, S.chunk_cap, 0, nullptr, out_indexes, nullptr, d_nidx, nullptr);
}

__global__ void __launch_bounds__(kThreads)
    select_flags_kernel(const uint8_t* __restrict__ sel, const PeerTab* tab, const StepPtrs* sp, const uint64_t* d_U,
                        const uint32_t* d_flags, uint32_t* __restrict__ sidx, uint32_t* counts, uint64_t* d_cap) {
  __shared__ uint32_t tbl[2][32];
  const uint32_t* __restrict__ u_idx = tab->u_idx[tab->rank][sp->par];
  const int tid = threadIdx.x;
  const uint64_t cnt = (*d_flags & (1u | 8u | 16u)) ? 0 : *d_U;
  const uint64_t tiles = (cnt + kTileK - 1) / kTileK;
  const uint64_t tpc = (tiles + gridDim.x - 1) / gridDim.x;
  if (blockIdx.x == 0 && tid == 0) *d_cap = tpc * kTileK;
  const uint64_t t0 = split_at(blockIdx.x, tiles, gridDim.x), t1 = split_at(blockIdx.x + 1, tiles, gridDim.x);
  const uint64_t obase = uint64_t(blockIdx.x) * tpc * kTileK;
  uint32_t running = 0;
  int parity = 0;
  for (uint64_t tile = t0; tile < t1; ++tile, parity ^= 1) {
    bool pred[kJ];
    uint32_t idx[kJ];
    unsigned bal[kJ][1];
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const uint64_t e = tile * kTileK + uint64_t(j) * kThreads + tid;
      pred[j] = e < cnt && sel[e];
      idx[j] = pred[j] ? u_idx[e] : 0u;
      bal[j][0] = __ballot_sync(0xffffffffu, pred[j]);
    }
    uint32_t grp[kJ];
    const uint32_t total = tile_offsets<1>(tbl[parity], bal, grp);
#pragma unroll
    for (int j = 0; j < kJ; ++j)
      if (pred[j]) sidx[obase + running + grp[j] + rank_in_group<1>(bal, j, 0)] = idx[j];
    running += total;
  }
  if (tid == 0) counts[blockIdx.x] = running;
}

cudaError_t launch_select_flags(Launch& L, const Stage& S, const uint8_t* sel, const PeerTab* d_tab,
                                const StepPtrs* sp, const uint64_t* d_U, uint64_t bound, uint32_t* out,
                                uint64_t* d_count, const uint32_t* d_flags) {
  static std::atomic<int> cap{0};
  if (!cap) cap = resident_ctas(select_flags_kernel, kThreads, L.sms);
  const uint32_t G = chunks_for((bound + kTileK - 1) / kTileK, cap, S.max_chunks);
  select_flags_kernel<<<G, kThreads, 0, L.s>>>(sel, d_tab, sp, d_U, d_flags, S.sidx, S.counts, S.chunk_cap);
  ++L.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_compact<3>(L, S, G, 0, S.chunk_cap, 0, nullptr, out, nullptr, d_count, nullptr);
}

// =============================================================================
// K3: region merge — scatter (M1) + ordered bracket scan (M2)
// =============================================================================
__global__ void __launch_bounds__(kThreads)
    scatter_kernel(Segs segs, uint64_t lo, uint64_t W, int P, uint32_t* mask, float* stage, uint32_t* d_flags) {
  const uint64_t total = segs.start[segs.nseg];
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  for (uint64_t e = uint64_t(blockIdx.x) * kThreads + threadIdx.x; e < total; e += stride) {
    int sg = 0;
    while (sg + 1 < segs.nseg && e >= segs.start[sg + 1]) ++sg;
    const uint64_t entry = segs.ptr[sg][e - segs.start[sg]];
    const uint64_t idx = coo_idx(entry);
    if (idx < lo || idx - lo >= W) {
      atomicOr(d_flags, 2u);
      continue;
    }
    const uint64_t i = idx - lo;
    const int src = segs.src[sg];
    stage[i * uint64_t(P) + src] = coo_val(entry);
    atomicOr(&mask[i >> 2], 1u << (unsigned(i & 3u) * 8u + unsigned(src)));
  }
}

cudaError_t launch_scatter(Launch& L, const Segs& segs, uint64_t lo, uint64_t W, int P, uint32_t* mask,
                           float* stage, uint32_t* d_flags) {
  const uint64_t total = segs.start[segs.nseg];
  if (total == 0) return cudaSuccess;
  const int grid = int(std::min<uint64_t>((total + kThreads - 1) / kThreads, uint64_t(L.sms) * 16));
  scatter_kernel<<<grid, kThreads, 0, L.s>>>(segs, lo, W, P, mask, stage, d_flags);
  ++L.launches;
  return cudaGetLastError();
}

// Fixed stride-doubling bracket over source ranks with absent pass-through
// (sparse.cpp:238-245, tests/test_util.hpp:124-132):
//   P=8: ((p0+p4)+(p2+p6)) + ((p1+p5)+(p3+p7))
template <int P>
__device__ __forceinline__ double bracket_sum(const float* st, uint32_t bits) {
  double a[P];
  bool h[P];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    h[q] = (bits >> q) & 1u;
    a[q] = h[q] ? double(st[q]) : 0.0;
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

// All P staged slots of one coordinate in one vector load (the row is
// P * 4 bytes, aligned to it); absent slots are loaded and ignored.
template <int P>
__device__ __forceinline__ void load_slots(const float* __restrict__ st, float (&v)[P]) {
  if constexpr (P == 1) {
    v[0] = st[0];
  } else if constexpr (P == 2) {
    const float2 x = *reinterpret_cast<const float2*>(st);
    v[0] = x.x; v[1] = x.y;
  } else {
#pragma unroll
    for (int q = 0; q < P; q += 4) {
      const float4 x = *reinterpret_cast<const float4*>(st + q);
      v[q] = x.x; v[q + 1] = x.y; v[q + 2] = x.z; v[q + 3] = x.w;
    }
  }
}
constexpr int kGather = 4;

// Thread-contiguous layout: thread t of a tile owns coordinates
// [t*32, t*32+32) (eight mask words, two 16 B loads), so its selected set is a
// 32-bit mask and the tile order is (thread, bit): one warp scan + one CTA
// barrier per tile.  The first values each thread emits are gathered from the
// staging before the barrier, so a tile costs about one memory round trip.
constexpr int kRegionCoordsPerThread = 32;
constexpr int kRegionTile = kThreads * kRegionCoordsPerThread;  // 8192 coordinates
static_assert(kRegionTile == kRegionTileHost, "staging sized for the region tile");

template <int P, bool FILTER>
__global__ void __launch_bounds__(kThreads, 2)
    region_scan_kernel(uint64_t lo, uint64_t W, uint32_t tiles, uint32_t tpc, uint32_t* mask,
                       const float* __restrict__ stage, const double* d_gth, uint32_t* sidx, double* sval,
                       uint32_t* counts) {
  __shared__ uint32_t wtot[2][kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double gth = FILTER ? *d_gth : 0.0;
  const uint64_t nwords = (W + 3) / 4;
  const uint32_t t0 = split_at32(blockIdx.x, tiles, gridDim.x);
  const uint32_t t1 = split_at32(blockIdx.x + 1, tiles, gridDim.x);
  const uint64_t obase = uint64_t(blockIdx.x) * tpc * kRegionTile;
  uint32_t running = 0;
  auto load_mask = [&](uint32_t tile, uint32_t (&m)[8]) {
    const uint64_t w = uint64_t(tile) * (kRegionTile / 4) + uint64_t(tid) * 8;
    if (w + 8 <= nwords) {
      const uint4 a = *reinterpret_cast<const uint4*>(mask + w);
      const uint4 b = *reinterpret_cast<const uint4*>(mask + w + 4);
      m[0] = a.x; m[1] = a.y; m[2] = a.z; m[3] = a.w;
      m[4] = b.x; m[5] = b.y; m[6] = b.z; m[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) m[j] = (w + j < nwords) ? mask[w + j] : 0u;
    }
  };
  uint32_t nx[8];  // the next tile's mask words, loaded one tile ahead
  if (t0 < t1) load_mask(t0, nx);
  int parity = 0;
  for (uint32_t tile = t0; tile < t1; ++tile, parity ^= 1) {
    const uint64_t w0 = uint64_t(tile) * (kRegionTile / 4) + uint64_t(tid) * 8;  // first mask word
    uint32_t mw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) mw[j] = nx[j];
    if (tile + 1 < t1) load_mask(tile + 1, nx);
    // bit c of nibble j: byte c of word j non-zero (some source present)
    uint32_t present = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      present |= (((__vcmpne4(mw[j], 0u) & 0x01010101u) * 0x01020408u) >> 24) << (4 * j);
    const uint64_t c0 = w0 * 4;  // first coordinate (region-relative)
    auto bits_of = [&](int k) {  // select tree: keeps mw[] in registers
      const int j = k >> 2;
      const uint32_t w01 = (j & 1) ? mw[1] : mw[0], w23 = (j & 1) ? mw[3] : mw[2];
      const uint32_t w45 = (j & 1) ? mw[5] : mw[4], w67 = (j & 1) ? mw[7] : mw[6];
      const uint32_t w03 = (j & 2) ? w23 : w01, w47 = (j & 2) ? w67 : w45;
      return (((j & 4) ? w47 : w03) >> (8 * (k & 3))) & 0xffu;
    };
    // The first kGather present coordinates: all their stage loads are issued
    // together (one memory round trip), and their sums stay in registers for
    // the emit below.  Threads with more present coordinates (rare at top-k
    // densities) walk the rest one by one.
    int kk[kGather];
    double vv[kGather];
    {
      uint32_t rest = present;
#pragma unroll
      for (int b = 0; b < kGather; ++b) {
        kk[b] = rest ? __ffs(rest) - 1 : -1;
        rest &= rest - 1;
      }
      float raw[kGather][P];
#pragma unroll
      for (int b = 0; b < kGather; ++b)
        if (kk[b] >= 0) load_slots<P>(stage + (c0 + kk[b]) * P, raw[b]);
#pragma unroll
      for (int b = 0; b < kGather; ++b) vv[b] = kk[b] >= 0 ? bracket_regs<P>(raw[b], bits_of(kk[b])) : 0.0;
    }
    uint32_t sel = present;
    if (FILTER) {
      sel = 0u;
#pragma unroll
      for (int b = 0; b < kGather; ++b)
        if (kk[b] >= 0 && fabs(vv[b]) >= gth) sel |= 1u << kk[b];
      uint32_t rest = present;
#pragma unroll
      for (int b = 0; b < kGather; ++b) rest &= rest - 1;
      for (; rest; rest &= rest - 1) {
        const int k = __ffs(rest) - 1;
        if (fabs(bracket_sum<P>(stage + (c0 + k) * P, bits_of(k))) >= gth) sel |= 1u << k;
      }
    }
    if (present) {
      if (w0 + 8 <= nwords) {
        *reinterpret_cast<uint4*>(mask + w0) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(mask + w0 + 4) = make_uint4(0, 0, 0, 0);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (w0 + j < nwords) mask[w0 + j] = 0u;
      }
    }
    // CTA exclusive scan of the per-thread counts.
    const uint32_t cnt = __popc(sel);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wtot[parity][warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t x = wtot[parity][w];
      wpre += (w < warp) ? x : 0u;
      total += x;
    }
    uint64_t pos = obase + running + wpre + incl - cnt;
    for (uint32_t rest = sel; rest; rest &= rest - 1, ++pos) {
      const int k = __ffs(rest) - 1;
      double v = 0.0;
      bool have = false;
#pragma unroll
      for (int b = 0; b < kGather; ++b)
        if (kk[b] == k) {
          v = vv[b];
          have = true;
        }
      if (!have) v = bracket_sum<P>(stage + (c0 + k) * P, bits_of(k));
      sidx[pos] = uint32_t(lo + c0 + k);
      sval[pos] = v;
    }
    running += total;
  }
  if (tid == 0) counts[blockIdx.x] = running;
}

template <int P, bool FILTER>
static cudaError_t region_scan_dispatch(Launch& L, const Stage& S, uint64_t lo, uint64_t W, uint32_t* mask,
                                        const float* stage, const double* d_gth, uint32_t* out_idx,
                                        double* out_val, uint64_t* d_count) {
  constexpr int TILE = kRegionTile;
  const uint64_t tiles = (W + TILE - 1) / TILE;
  static std::atomic<int> cap{0};
  if (!cap) cap = resident_ctas(region_scan_kernel<P, FILTER>, kThreads, L.sms);
  const uint32_t G = chunks_for(tiles, cap, S.max_chunks);
  if (uint64_t(tiles) * G > 0xffffffffull) return cudaErrorInvalidValue;  // split_at32's range
  const uint32_t tpc = uint32_t(std::max<uint64_t>((tiles + G - 1) / G, 1));
  region_scan_kernel<P, FILTER><<<G, kThreads, 0, L.s>>>(lo, W, uint32_t(tiles), tpc, mask, stage, d_gth, S.sidx,
                                                         S.sval, S.counts);
  ++L.launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_compact<2>(L, S, G, uint64_t(tpc) * TILE, nullptr, 0, nullptr, out_idx, out_val, d_count,
                           nullptr);
}

cudaError_t launch_region_scan(Launch& L, const Stage& S, int P, bool filter, uint64_t lo, uint64_t W,
                               uint32_t* mask, const float* stage, const double* d_gth, uint32_t* out_idx,
                               double* out_val, uint64_t* d_count) {
#define OKT_RS(PP)                                                                                          \
  return filter ? region_scan_dispatch<PP, true>(L, S, lo, W, mask, stage, d_gth, out_idx, out_val, d_count) \
                : region_scan_dispatch<PP, false>(L, S, lo, W, mask, stage, d_gth, out_idx, out_val, d_count)
  switch (P) {
    case 1: OKT_RS(1);
    case 2: OKT_RS(2);
    case 4: OKT_RS(4);
    case 8: OKT_RS(8);
  }
#undef OKT_RS
  return cudaErrorInvalidValue;
}

// =============================================================================
// K2 / K4: radix select of the k-th largest magnitude
// =============================================================================
template <int SRC>  // 0: dense f32, 1: AoS (u32 idx | f32 val << 32), 2: f64
__device__ __forceinline__ uint64_t mag_key(const void* data, uint64_t i) {
  if (SRC == 0) return uint64_t(__float_as_uint(static_cast<const float*>(data)[i]) & 0x7fffffffu);
  if (SRC == 1) return (static_cast<const uint64_t*>(data)[i] >> 32) & 0x7fffffffull;
  return uint64_t(__double_as_longlong(static_cast<const double*>(data)[i])) & 0x7fffffffffffffffull;
}

__global__ void radix_init_kernel(RadixState* rs, uint64_t k, uint64_t n_host, const uint64_t* d_n) {
  const uint64_t cnt = d_n ? *d_n : n_host;
  rs->prefix = 0;
  rs->kk = k < cnt ? k : cnt;
  rs->active = cnt > 0 ? 1u : 0u;
  rs->pad = 0;
}

template <int SRC>
__global__ void __launch_bounds__(kThreads)
    radix_hist_kernel(const void* __restrict__ data, uint64_t n_host, const uint64_t* d_n,
                      const RadixState* rs, int shift, int bits, uint32_t* hist) {
  __shared__ uint32_t sh[2048];
  const int nb = 1 << bits;
  for (int i = threadIdx.x; i < nb; i += kThreads) sh[i] = 0;
  __syncthreads();
  if (!rs->active) return;
  const uint64_t n = d_n ? *d_n : n_host;
  const uint64_t prefix = rs->prefix;
  const int hi = shift + bits;
  const uint64_t want = prefix >> hi;
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
  if (SRC == 0 && (reinterpret_cast<uintptr_t>(data) & 15u) == 0) {
    // dense f32: 16-byte loads, two in flight per thread, then the < 4 tail keys
    const float4* d4 = static_cast<const float4*>(data);
    const uint64_t n4 = n >> 2;
    auto one = [&](float v) {
      const uint64_t key = uint64_t(__float_as_uint(v) & 0x7fffffffu);
      if ((key >> hi) == want) atomicAdd(&sh[(key >> shift) & (nb - 1)], 1u);
    };
    uint64_t j = i;
    for (; j + stride < n4; j += 2 * stride) {
      const float4 a = __ldg(d4 + j), b = __ldg(d4 + j + stride);
      one(a.x); one(a.y); one(a.z); one(a.w);
      one(b.x); one(b.y); one(b.z); one(b.w);
    }
    for (; j < n4; j += stride) {
      const float4 a = __ldg(d4 + j);
      one(a.x); one(a.y); one(a.z); one(a.w);
    }
    i = 4 * n4 + i;  // tail: keys [4*n4, n)
    if (i < n) one(static_cast<const float*>(data)[i]);
    i = n;
  }
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint64_t k0 = mag_key<SRC>(data, i), k1 = mag_key<SRC>(data, i + stride);
    uint64_t k2 = mag_key<SRC>(data, i + 2 * stride), k3 = mag_key<SRC>(data, i + 3 * stride);
    if ((k0 >> hi) == want) atomicAdd(&sh[(k0 >> shift) & (nb - 1)], 1u);
    if ((k1 >> hi) == want) atomicAdd(&sh[(k1 >> shift) & (nb - 1)], 1u);
    if ((k2 >> hi) == want) atomicAdd(&sh[(k2 >> shift) & (nb - 1)], 1u);
    if ((k3 >> hi) == want) atomicAdd(&sh[(k3 >> shift) & (nb - 1)], 1u);
  }
  for (; i < n; i += stride) {
    const uint64_t k0 = mag_key<SRC>(data, i);
    if ((k0 >> hi) == want) atomicAdd(&sh[(k0 >> shift) & (nb - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kThreads)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// One CTA of 1024 threads: find the bin holding the kk-th largest key, update
// the prefix, clear the histogram for the next pass.
__global__ void __launch_bounds__(1024)
    radix_pick_kernel(RadixState* rs, uint32_t* hist, int shift, int bits, int last, int f64,
                      double* th_out) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t s_bin, s_above;
  const int nb = 1 << bits;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const bool active = rs->active != 0;
  // Bins in descending order: position q holds bin nb-1-q.
  const int q0 = 2 * t, q1 = 2 * t + 1;
  const uint32_t c0 = (active && q0 < nb) ? hist[nb - 1 - q0] : 0u;
  const uint32_t c1 = (active && q1 < nb) ? hist[nb - 1 - q1] : 0u;
  uint32_t v = c0 + c1, incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) warp_sums[w] = incl;
  if (t == 0) { s_bin = 0xffffffffu; s_above = 0; }
  __syncthreads();
  if (w == 0) {
    uint32_t ws = warp_sums[lane], wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += x;
    }
    warp_sums[lane] = wi - ws;
  }
  __syncthreads();
  const uint32_t excl = warp_sums[w] + incl - v;
  if (active) {
    const uint64_t kk = rs->kk;
    if (excl < kk && uint64_t(excl) + c0 >= kk) {
      s_bin = uint32_t(nb - 1 - q0);
      s_above = excl;
    } else if (uint64_t(excl) + c0 < kk && uint64_t(excl) + c0 + c1 >= kk) {
      s_bin = uint32_t(nb - 1 - q1);
      s_above = excl + c0;
    }
  }
  __syncthreads();
  for (int b = t; b < nb; b += 1024) hist[b] = 0;
  if (t == 0 && active && s_bin != 0xffffffffu) {
    const uint64_t prefix = rs->prefix | (uint64_t(s_bin) << shift);
    rs->prefix = prefix;
    rs->kk = rs->kk - s_above;
    if (last) {
      *th_out = f64 ? __longlong_as_double(static_cast<long long>(prefix))
                    : double(__uint_as_float(uint32_t(prefix)));
    }
  }
}

// After pass 0's histogram of dense f32 magnitudes: pick the top-11-bit bin
// holding the kk-th largest and write the bin's smallest magnitude to *d_floor
// (every value at or above it is a candidate; at least kk of them exist).
__global__ void radix_floor_kernel(const RadixState* rs, double* d_floor) {
  *d_floor = rs->active ? double(__uint_as_float(uint32_t(rs->prefix))) : 0.0;
}

cudaError_t launch_radix_pass0_floor(Launch& L, RadixState* d_rs, uint32_t* d_hist, double* d_floor) {
  radix_pick_kernel<<<1, 1024, 0, L.s>>>(d_rs, d_hist, 20, 11, 0, 0, nullptr);
  radix_floor_kernel<<<1, 1, 0, L.s>>>(d_rs, d_floor);
  L.launches += 2;
  return cudaGetLastError();
}

// Sampled pass-0 histogram for the cold refresh's candidate threshold: the
// same accumulate arithmetic as K1 (fmaf(alpha, g, eps)), the same 2048 bins
// of the top 11 magnitude bits, over one coordinate per 2^s_log2 block.
__global__ void __launch_bounds__(kThreads)
    sample_hist_kernel(const float* __restrict__ g, const float* __restrict__ eps, float alpha, uint64_t n,
                       uint32_t s_log2, uint64_t m, uint32_t* d_hist) {
  __shared__ uint32_t s_hist[2048];
  for (int i = threadIdx.x; i < 2048; i += kThreads) s_hist[i] = 0;
  __syncthreads();
  const uint64_t mask = (uint64_t(1) << s_log2) - 1;
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  constexpr int U = 4;
  for (uint64_t j0 = uint64_t(blockIdx.x) * kThreads + threadIdx.x; j0 < m; j0 += U * stride) {
    float gv[U], ev[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = j0 + uint64_t(u) * stride;
      const uint64_t i = (j << s_log2) + ((j * 40503u) & mask);
      ok[u] = j < m && i < n;
      gv[u] = ok[u] ? __ldcs(g + i) : 0.f;
      ev[u] = ok[u] ? __ldcs(eps + i) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) atomicAdd(&s_hist[(__float_as_uint(fmaf(alpha, gv[u], ev[u])) & 0x7fffffffu) >> 20], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += kThreads)
    if (s_hist[i]) atomicAdd(&d_hist[i], s_hist[i]);
}

cudaError_t launch_sample_floor(Launch& L, const float* g, const float* eps, float alpha, uint64_t n,
                                uint32_t s_log2, uint64_t q, RadixState* d_rs, uint32_t* d_hist, double* d_floor) {
  const uint64_t m = (n + (uint64_t(1) << s_log2) - 1) >> s_log2;
  cudaError_t e = cudaMemsetAsync(d_hist, 0, 2048 * sizeof(uint32_t), L.s);
  if (e != cudaSuccess) return e;
  if ((e = launch_radix_init(L, d_rs, q, m, nullptr)) != cudaSuccess) return e;
  const uint64_t want = (m + 4 * kThreads - 1) / (4 * kThreads);
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(L.sms) * 4)));
  sample_hist_kernel<<<grid, kThreads, 0, L.s>>>(g, eps, alpha, n, s_log2, m, d_hist);
  ++L.launches;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return launch_radix_pass0_floor(L, d_rs, d_hist, d_floor);
}

cudaError_t launch_radix_init(Launch& L, RadixState* d_rs, uint64_t k, uint64_t n_host,
                              const uint64_t* d_n) {
  radix_init_kernel<<<1, 1, 0, L.s>>>(d_rs, k, n_host, d_n);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_radix_select(Launch& L, RadixSrc src, const void* data, uint64_t n_host,
                                const uint64_t* d_n, uint64_t n_bound, uint64_t k,
                                RadixState* d_rs, uint32_t* d_hist, double* d_th_out,
                                bool hist0_done) {
  static const int f32_pass[3][2] = {{20, 11}, {10, 10}, {0, 10}};
  static const int f64_pass[6][2] = {{52, 11}, {41, 11}, {30, 11}, {19, 11}, {8, 11}, {0, 8}};
  const bool f64 = src == RadixSrc::kF64;
  const int npass = f64 ? 6 : 3;
  cudaError_t e;
  if (!hist0_done) {
    if ((e = launch_radix_init(L, d_rs, k, n_host, d_n)) != cudaSuccess) return e;
  }
  const uint64_t bound = d_n ? n_bound : n_host;
  const int grid = int(std::max<uint64_t>(
      1, std::min<uint64_t>((bound + kThreads * 8 - 1) / (kThreads * 8), uint64_t(L.sms) * 8)));
  for (int p = 0; p < npass; ++p) {
    const int shift = f64 ? f64_pass[p][0] : f32_pass[p][0];
    const int bits = f64 ? f64_pass[p][1] : f32_pass[p][1];
    if (!(p == 0 && hist0_done)) {
      switch (src) {
        case RadixSrc::kDenseF32:
          radix_hist_kernel<0><<<grid, kThreads, 0, L.s>>>(data, n_host, d_n, d_rs, shift, bits, d_hist);
          break;
        case RadixSrc::kAosF32:
          radix_hist_kernel<1><<<grid, kThreads, 0, L.s>>>(data, n_host, d_n, d_rs, shift, bits, d_hist);
          break;
        case RadixSrc::kF64:
          radix_hist_kernel<2><<<grid, kThreads, 0, L.s>>>(data, n_host, d_n, d_rs, shift, bits, d_hist);
          break;
      }
      ++L.launches;
    }
    radix_pick_kernel<<<1, 1024, 0, L.s>>>(d_rs, d_hist, shift, bits, p == npass - 1, f64 ? 1 : 0,
                                           d_th_out);
    ++L.launches;
  }
  return cudaGetLastError();
}

// =============================================================================
// Control kernels
// =============================================================================
__global__ void slice_offsets_kernel(const uint64_t* coo, const uint64_t* d_m, const uint64_t* cuts,
                                     int P, uint64_t* off, uint32_t* cnt_out, const uint32_t* d_flags) {
  __shared__ uint64_t s_off[kMaxP + 1];
  const int d = threadIdx.x;
  const uint64_t m = *d_m;
  if (d <= P) {
    // lower_bound of cuts[d] over the ascending indices of the local selection
    const uint64_t key = cuts[d];
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (uint64_t(coo_idx(coo[mid])) < key) lo = mid + 1;
      else hi = mid;
    }
    s_off[d] = (d == P) ? m : lo;
    off[d] = s_off[d];
  }
  __syncthreads();
  if (d < P) cnt_out[d] = uint32_t(s_off[d + 1] - s_off[d]);
  if (d == 0) cnt_out[P] = *d_flags;
}

cudaError_t launch_slice_offsets(Launch& L, const uint64_t* coo, const uint64_t* d_m,
                                 const uint64_t* d_cuts, int P, uint64_t* d_off, uint32_t* d_cnt_out,
                                 const uint32_t* d_flags) {
  slice_offsets_kernel<<<1, 32, 0, L.s>>>(coo, d_m, d_cuts, P, d_off, d_cnt_out, d_flags);
  ++L.launches;
  return cudaGetLastError();
}

// space_repartition proposal (oktopk.cpp:39-49): cut_r = sel[floor(r*m/P)], or
// r*n/P when nothing was selected.
__global__ void proposals_kernel(const uint32_t* idx, int stride, const uint64_t* d_m, uint64_t m_host,
                                 uint64_t n, int P, uint64_t* prop) {
  const int r = threadIdx.x;
  if (r > P) return;
  const uint64_t m = d_m ? *d_m : m_host;
  uint64_t cut;
  if (r == 0) cut = 0;
  else if (r == P) cut = n;
  else if (m == 0) cut = uint64_t(r) * n / uint64_t(P);
  else {
    const uint64_t pos = uint64_t(r) * m / uint64_t(P);
    cut = pos < m ? uint64_t(idx[pos * uint64_t(stride)]) : n;
  }
  prop[r] = cut;
}

cudaError_t launch_proposals(Launch& L, const uint32_t* idx, int stride, const uint64_t* d_m,
                             uint64_t m_host, uint64_t n, int P, uint64_t* d_prop) {
  proposals_kernel<<<1, 32, 0, L.s>>>(idx, stride, d_m, m_host, n, P, d_prop);
  ++L.launches;
  return cudaGetLastError();
}

// Consensus cuts (oktopk.cpp:51-61): the element-wise mean of P integer
// proposals is exact in fp64 (sums < 2^53, P a power of two), so
// llround(max(0, S/P)) == floor((2S + P) / 2P) in integers.
__global__ void cuts_kernel(const uint64_t* allprop, int P, uint64_t n, uint64_t* cuts) {
  if (threadIdx.x != 0) return;
  cuts[0] = 0;
  uint64_t prev = 0;
  for (int r = 1; r < P; ++r) {
    uint64_t S = 0;
    for (int q = 0; q < P; ++q) S += allprop[uint64_t(q) * (P + 1) + r];
    uint64_t rounded = (2 * S + uint64_t(P)) / (2 * uint64_t(P));
    if (rounded > n) rounded = n;
    if (rounded < prev) rounded = prev;
    cuts[r] = rounded;
    prev = rounded;
  }
  cuts[P] = n;
}

cudaError_t launch_cuts(Launch& L, const uint64_t* d_allprop, int P, uint64_t n, uint64_t* d_cuts) {
  cuts_kernel<<<1, 32, 0, L.s>>>(d_allprop, P, n, d_cuts);
  ++L.launches;
  return cudaGetLastError();
}

__global__ void extract_kernel(const uint64_t* coo, const uint64_t* d_m, uint32_t* idx, double* val) {
  const uint64_t m = *d_m;
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = coo[e];
    idx[e] = coo_idx(x);
    val[e] = double(coo_val(x));
  }
}

cudaError_t launch_extract(Launch& L, const uint64_t* coo, const uint64_t* d_m, uint64_t bound,
                           uint32_t* idx, double* val) {
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>((bound + kThreads - 1) / kThreads,
                                                              uint64_t(L.sms) * 8)));
  extract_kernel<<<grid, kThreads, 0, L.s>>>(coo, d_m, idx, val);
  ++L.launches;
  return cudaGetLastError();
}

__global__ void widen_kernel(const float* in, uint64_t n, double* out) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += uint64_t(gridDim.x) * blockDim.x)
    out[e] = double(in[e]);
}

cudaError_t launch_widen_f32(Launch& L, const float* in, uint64_t n, double* out) {
  if (!n) return cudaSuccess;
  const int grid = int(std::min<uint64_t>((n + kThreads - 1) / kThreads, uint64_t(L.sms) * 8));
  widen_kernel<<<grid, kThreads, 0, L.s>>>(in, n, out);
  ++L.launches;
  return cudaGetLastError();
}

// =============================================================================
// Generators: SplitMix64 streams of proj/core/include/oklab/rng.hpp
// =============================================================================
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t d_mix64(uint64_t a, uint64_t b) {
  return d_splitmix64(a ^ (0x9e3779b97f4a7c15ull + b + (a << 6) + (a >> 2)));
}
__device__ __forceinline__ double d_unit(uint64_t bits) {
  return double(bits >> 11) * 0x1.0p-53;
}

// The i-th draw of SplitMix64(seed) is splitmix64(seed + i*gamma), so the
// sequential stream parallelises exactly.
__global__ void gen_random_dense_kernel(float* out, uint64_t n, uint64_t seed) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double u = d_unit(d_splitmix64(seed + i * 0x9e3779b97f4a7c15ull));
    out[i] = float(__dsub_rn(__dmul_rn(2.0, u), 1.0));
  }
}

__global__ void gen_noise_kernel(float* out, uint64_t n, uint64_t noise_key, double coef) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double u = d_unit(d_mix64(noise_key, i));
    out[i] = float(__dmul_rn(coef, __dsub_rn(__dmul_rn(2.0, u), 1.0)));
  }
}

__global__ void scatter_heavy_kernel(const uint32_t* pos, const float* val, uint64_t count, float* out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[pos[i]] = val[i];
}

cudaError_t launch_gen_random_dense(Launch& L, float* out, uint64_t n, uint64_t seed) {
  if (!n) return cudaSuccess;
  const int grid = int(std::min<uint64_t>((n + kThreads - 1) / kThreads, uint64_t(L.sms) * 16));
  gen_random_dense_kernel<<<grid, kThreads, 0, L.s>>>(out, n, seed);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_gen_noise(Launch& L, float* out, uint64_t n, uint64_t noise_key, double coef) {
  if (!n) return cudaSuccess;
  const int grid = int(std::min<uint64_t>((n + kThreads - 1) / kThreads, uint64_t(L.sms) * 16));
  gen_noise_kernel<<<grid, kThreads, 0, L.s>>>(out, n, noise_key, coef);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_scatter_heavy(Launch& L, const uint32_t* pos, const float* val, uint64_t count,
                                 float* out) {
  if (!count) return cudaSuccess;
  const int grid = int(std::min<uint64_t>((count + kThreads - 1) / kThreads, uint64_t(L.sms) * 8));
  scatter_heavy_kernel<<<grid, kThreads, 0, L.s>>>(pos, val, count, out);
  ++L.launches;
  return cudaGetLastError();
}

// Loads every kernel of the step's paths up front.  With CUDA's lazy module
// loading a kernel is loaded at its first launch: the first warm refresh of a
// run (the candidate path, t = tau' + 1) paid 13.6 ms for it at n = 1M
// (round-2 sweep).  cudaFuncGetAttributes loads a function without running it.
int carveout_pref() {
  static const int v = [] {
    const char* e = std::getenv("OKT_CARVEOUT");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

void preload_kernels() {
  static std::atomic<bool> done[64];  // per device: a module is loaded per context
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev & 63].exchange(true)) return;
  cudaFuncAttributes a;
  const int co = carveout_pref();
  auto touch = [&](const void* f) {
    cudaFuncGetAttributes(&a, f);
    if (co >= 0) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, co);
  };
#define OKT_K1(A, S, H, D, AP)                                                   \
  touch(reinterpret_cast<const void*>(k1_kernel<A, S, H, true, D, AP>));         \
  touch(reinterpret_cast<const void*>(k1_kernel<A, S, H, false, D, AP>))
  OKT_K1(false, true, false, false, false);
  OKT_K1(false, true, false, true, false);
  OKT_K1(false, true, false, true, true);
  OKT_K1(true, true, false, false, false);
  OKT_K1(true, true, false, true, false);
  OKT_K1(true, true, false, true, true);
  OKT_K1(true, false, true, false, false);
  OKT_K1(true, true, true, false, false);
#undef OKT_K1
  touch(reinterpret_cast<const void*>(compact_kernel<0, false>));
  touch(reinterpret_cast<const void*>(compact_kernel<1, false>));
  touch(reinterpret_cast<const void*>(compact_kernel<1, true>));
  touch(reinterpret_cast<const void*>(compact_kernel<2, false>));
  touch(reinterpret_cast<const void*>(compact_kernel<3, false>));
  touch(reinterpret_cast<const void*>(compact_kernel<4, false>));
  touch(reinterpret_cast<const void*>(filter_kernel<true>));
  touch(reinterpret_cast<const void*>(filter_kernel<false>));
  touch(reinterpret_cast<const void*>(apply_kernel));
  touch(reinterpret_cast<const void*>(apply_u_kernel));
  touch(reinterpret_cast<const void*>(select_flags_kernel));
  touch(reinterpret_cast<const void*>(scatter_kernel));
  touch(reinterpret_cast<const void*>(radix_init_kernel));
  touch(reinterpret_cast<const void*>(radix_hist_kernel<0>));
  touch(reinterpret_cast<const void*>(radix_hist_kernel<1>));
  touch(reinterpret_cast<const void*>(radix_hist_kernel<2>));
  touch(reinterpret_cast<const void*>(radix_pick_kernel));
  touch(reinterpret_cast<const void*>(radix_floor_kernel));
  touch(reinterpret_cast<const void*>(sample_hist_kernel));
  touch(reinterpret_cast<const void*>(slice_offsets_kernel));
  touch(reinterpret_cast<const void*>(proposals_kernel));
  touch(reinterpret_cast<const void*>(cuts_kernel));
  touch(reinterpret_cast<const void*>(region_scan_kernel<1, false>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<1, true>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<2, false>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<2, true>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<4, false>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<4, true>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<8, false>));
  touch(reinterpret_cast<const void*>(region_scan_kernel<8, true>));
  preload_p2p_kernels();
  cudaGetLastError();
}

}  // namespace okt
