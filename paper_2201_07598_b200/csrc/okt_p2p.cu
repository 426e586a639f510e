// okt_p2p.cu — kernels of the device-driven multi-GPU exchange (okt_p2p.cuh).
//
// Steady Ok-Topk iteration on P ranks, no host round trip and no compaction
// pass between a producer and its consumers:
//   K1 phase A (chunked staging + per-chunk cut counts in the window;
//     its last CTA publishes L-ready)
//   wait(L ready) -> scatter reads my slice of every chunk of every rank in
//     place over NVLink -> bracket scan / survivor filter, chunked into the
//     window (its last CTA writes the chunk prefix and publishes survivors)
//   wait(survivors) -> plan (offsets, balance) -> pull every chunk to its
//     position in u, applying K7 on the way
//     [balanced: pull my block, publish(block), wait, pull the other blocks]
//   -> indexes.
#include "okt_device.cuh"
#include "okt_kernels.hpp"
#include "okt_p2p.cuh"

#include <algorithm>

namespace okt {

namespace {
constexpr uint32_t kAbortBits = 1u | 8u | 16u;  // local non-finite, peer timeout, peer failure
}

// K3 (M1) fused with the split exchange.  Work items are (source, tile,
// part): only the K1 tiles overlapping my region carry entries for me, and
// each is split into `parts` when there are more warps than tiles.  A warp reads its part of the chunk's slice for my region,
// [lt[c][me], lt[c][me+1]), straight out of the source's HBM (NVLink for a
// peer) and scatters it into the presence mask / coordinate-major staging.
// My own chunks need no hand-off, so they are scattered first, while the
// peers' L-ready flags are in flight.  Order does not matter here: the
// bracket scan re-derives it from coordinates.
__global__ void __launch_bounds__(kThreads)
    p2p_scatter_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, P2PPlan* plan, uint64_t lo, uint64_t W,
                       uint32_t k1_tiles, uint32_t* mask, float* stage, uint32_t* d_flags, uint64_t timeout_ns) {
  __shared__ uint64_t s_seg[kP2PMaxP];
  __shared__ int s_abort;
  const uint64_t epoch = sp->epoch;
  const int par = sp->par;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* const trace = tab->trace;
  const uint32_t G = k1_tiles, cap = kK1Tile;  // same geometry on every rank (same n)
  if (q == 0) {
    s_abort = (*d_flags & 1u) ? 1 : 0;
    trace_stamp(trace, kTrScatter, 0);
  }
  if (q < P) s_seg[q] = 0;
  if (blockIdx.x == 0 && q == 0) {
    // Publish this rank's K1 output (every K1 CTA finished before this kernel
    // started): status, then L-ready at every rank (myself included).
    tab->hdr[me]->pub[par].status = (*d_flags & 1u) ? 1 : 0;
    __threadfence_system();
    for (int r = 0; r < P; ++r) st_relaxed_sys(&tab->hdr[r]->flag[kFlagLReady][me], epoch);
  }
  // K1 chunks are its tiles: the ones overlapping [lo, lo + W).
  uint32_t c_lo = 0, nch = 0;
  if (W > 0 && G > 0) {
    c_lo = uint32_t(lo / kK1Tile);
    nch = uint32_t((lo + W - 1) / kK1Tile) - c_lo + 1;
  }
  const uint32_t warps_total = gridDim.x * kWarps;
  const uint32_t parts = max(1u, min(8u, warps_total / max(1u, uint32_t(P) * nch)));
  const uint32_t per_src = nch * parts;
  const uint32_t gw = blockIdx.x * kWarps + warp;
  __syncthreads();
  auto run = [&](int r, uint32_t it) {
    const uint32_t c = c_lo + it / parts, part = it % parts;
    const uint32_t* lt = tab->klt[r][par] + uint64_t(c) * kP2PMaxP;
    const uint32_t a0 = lt[me];
    const uint32_t b0 = (me + 1 < P) ? lt[me + 1] : tab->kcnt[r][par][c];
    const uint32_t len = b0 > a0 ? b0 - a0 : 0;
    const uint32_t a = a0 + uint32_t(uint64_t(len) * part / parts), b = a0 + uint32_t(uint64_t(len) * (part + 1) / parts);
    const uint64_t* src = tab->kstg[r][par] + uint64_t(c) * cap;
    // Every lane issues its (remote) loads for a 128-entry round before any
    // store, so a round costs one NVLink round trip.
    constexpr int R = 4;
    for (uint32_t j0 = a; j0 < b; j0 += 32 * R) {
      uint64_t e[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const uint32_t j = j0 + lane + 32 * k;
        e[k] = j < b ? src[j] : ~0ull;
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (j0 + lane + 32 * k >= b) continue;
        const uint64_t idx = coo_idx(e[k]);
        if (idx < lo || idx - lo >= W) {
          atomicOr(d_flags, 2u);
          continue;
        }
        const uint64_t i = idx - lo;
        stage[i * uint64_t(P) + r] = coo_val(e[k]);
        atomicOr(&mask[i >> 2], 1u << (unsigned(i & 3u) * 8u + unsigned(r)));
      }
    }
    if (lane == 0 && b > a) atomicAdd(reinterpret_cast<unsigned long long*>(&s_seg[r]), (unsigned long long)(b - a));
  };
  // 1. my own chunks (local HBM, no wait)
  if (!s_abort)
    for (uint32_t it = gw; it < per_src; it += warps_total) run(me, it);
  // 2. wait for every peer's L-ready, then their chunks (NVLink)
  if (q < P && q != me) {
    if (!wait_flag(&tab->hdr[me]->flag[kFlagLReady][q], epoch, timeout_ns)) {
      atomicOr(d_flags, 8u);
      s_abort = 1;
    } else {
      const volatile P2PPub* pub = &tab->hdr[q]->pub[par];
      const uint64_t st = pub->status;
      if (st || pub->k1_G != G || pub->k1_cap != cap) {
        atomicOr(d_flags, 16u);
        s_abort = 1;
      }
      if (blockIdx.x == 0) plan->peer_status[q] = st;
    }
  }
  __syncthreads();
  if (q == 0) trace_stamp(trace, kTrScatter, 1);
  if (!s_abort) {
    const uint32_t remote = uint32_t(P - 1) * per_src;
    for (uint32_t it = gw; it < remote; it += warps_total) {
      const uint32_t k = it / per_src;
      run((me + 1 + int(k)) % P, it % per_src);
    }
  }
  __syncthreads();
  if (q < P && s_seg[q]) atomicAdd(reinterpret_cast<unsigned long long*>(&plan->seg_cnt[q]), (unsigned long long)s_seg[q]);
  if (lane == 0) trace_stamp(trace, kTrScatter, 2);
}

// Allgatherv by pulling.  round 0 waits for every rank's survivors and
// derives the plan of balance_and_allgatherv (oktopk.cpp:172-231; identical on
// all ranks), then one warp per (rank, chunk) copies that chunk's survivors
// from the owner's window to their stream position in my u (unbalanced: all
// of u; balanced: my block).  round 1 (balanced only) pulls the other blocks
// from their block owners' u.  K7 runs on each entry as it lands.
__global__ void __launch_bounds__(kThreads)
    p2p_pull_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, uint64_t* d_S, P2PPlan* plan,
                    uint64_t* d_U, int round, uint32_t* d_flags, uint64_t timeout_ns, P2PApply ap, K1Totals lt) {
  __shared__ uint64_t s_size[kP2PMaxP], s_off[kP2PMaxP + 1], s_blk[kP2PMaxP + 1];
  __shared__ uint32_t s_G[kP2PMaxP], s_cap[kP2PMaxP], s_start[kP2PMaxP + 1];
  __shared__ int s_bal, s_abort;
  const uint64_t epoch = sp->epoch;
  const int par = sp->par;
  float* acc = ap.on ? (ap.sgd ? sp->eps_out : const_cast<float*>(sp->g)) : nullptr;
  float* wm = (ap.on && ap.sgd) ? sp->w : nullptr;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* const trace = tab->trace;
  const int trk = round == 0 ? kTrPull0 : kTrPull1;
  if (q == 0) {
    s_abort = (*d_flags & (1u | 8u | 16u)) ? 1 : 0;
    trace_stamp(trace, trk, 0);
  }
  __syncthreads();
  if (round == 0 && blockIdx.x == 0) {
    // Publish this rank's survivors (every region-scan CTA finished before
    // this kernel started): exclusive prefix of the chunk counts (where each
    // chunk lands in my part of u), S, status, then survivors-ready at every
    // peer and at myself.
    P2PPub* mine = &tab->hdr[me]->pub[par];
    const int G = int(mine->sur_G);
    const uint32_t* cnt = tab->scnt[me][par];
    uint64_t* pre = tab->spre[me][par];
    const int per = (G + kThreads - 1) / kThreads;
    uint64_t own = 0;
    for (int c = q * per; c < min(G, (q + 1) * per); ++c) own += cnt[c];
    uint64_t incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    __shared__ uint64_t wsum[kWarps];
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint64_t wpre = 0, tot = 0;
    for (int w = 0; w < kWarps; ++w) {
      wpre += (w < warp) ? wsum[w] : 0;
      tot += wsum[w];
    }
    uint64_t run = wpre + incl - own;
    for (int c = q * per; c < min(G, (q + 1) * per); ++c) {
      pre[c] = run;
      run += cnt[c];
    }
    __syncthreads();
    if (q == 0) {
      pre[G] = tot;
      *d_S = tot;
      mine->S = tot;
      mine->status = (*d_flags & (1u | 8u | 16u)) ? 1 : 0;
      __threadfence_system();
      for (int r = 0; r < P; ++r) st_relaxed_sys(&tab->hdr[r]->flag[kFlagSurReady][me], epoch);
    }
  }
  if (round == 0) {
    if (q < P) {
      uint64_t sz = 0;
      uint32_t G = 0, cap = 0;
      if (!wait_flag(&tab->hdr[me]->flag[kFlagSurReady][q], epoch, timeout_ns)) {
        atomicOr(d_flags, 8u);
        s_abort = 1;
      } else {
        const volatile P2PPub* pub = &tab->hdr[q]->pub[par];
        sz = pub->S;
        G = pub->sur_G;
        cap = pub->sur_cap;
        if (q != me && pub->status) {
          atomicOr(d_flags, 16u);
          s_abort = 1;
        }
      }
      s_size[q] = sz;
      s_G[q] = G;
      s_cap[q] = cap;
    }
    __syncthreads();
    if (q == 0) {
      uint64_t total = 0, maxs = 0;
      uint32_t items = 0;
      s_off[0] = 0;
      for (int r = 0; r < P; ++r) {
        total += s_size[r];
        maxs = max(maxs, s_size[r]);
        s_off[r + 1] = total;
        s_start[r] = items;
        items += s_G[r];
      }
      s_start[P] = items;
      s_bal = (total > 0 && maxs * uint64_t(P) >= 4 * total) ? 1 : 0;
      // equal_slice_ends (collectives.cpp:79-87): ceil-sized blocks first
      const uint64_t base = total / uint64_t(P), rem = total % uint64_t(P);
      s_blk[0] = 0;
      for (int r = 0; r < P; ++r) s_blk[r + 1] = s_blk[r] + base + (uint64_t(r) < rem ? 1 : 0);
      if (blockIdx.x == 0) {
        for (int r = 0; r < P; ++r) plan->sizes[r] = s_size[r];
        for (int r = 0; r <= P; ++r) {
          plan->off[r] = s_off[r];
          plan->block[r] = s_blk[r];
        }
        plan->total = total;
        plan->balanced = uint32_t(s_bal);
        *d_U = s_abort ? 0 : total;
      }
    }
  } else {
    if (q <= P) {
      s_off[q] = plan->off[q];
      s_blk[q] = plan->block[q];
    }
    if (q == 0) s_bal = int(plan->balanced);
  }
  __syncthreads();
  if (round == 1 && lt.d_m && int(blockIdx.x) <= P) {
    // Off the critical path: this rank's selection size and slice offsets
    // (from K1's chunk counts), one CTA per offset, for the result and the
    // ledger.
    const int d = blockIdx.x;
    const uint32_t G = tab->hdr[me]->pub[par].k1_G;
    const uint32_t* cnt = tab->kcnt[me][par];
    const uint32_t* klt = tab->klt[me][par];
    uint64_t o = 0;
    o = (d == P) ? strided_sum(cnt, G) : strided_sum(klt + d, G, kP2PMaxP);
    __shared__ uint64_t red[kWarps];
    o = block_sum(o, red);
    if (threadIdx.x == 0) {
      lt.d_off[d] = o;
      if (d == P) *lt.d_m = o;
    }
  }
  if (q == 0) trace_stamp(trace, trk, 1);
  if (s_abort) return;
  const bool bal = s_bal != 0;
  if (round == 1 && !bal) return;
  uint32_t* ui = tab->u_idx[me][par];
  double* uv = tab->u_val[me][par];
  const float tf = acc ? ceil_to_float(*ap.d_local_th) : 0.f;
  const double dP = double(P);
  bool bad = false;
  // Lands up to R entries per lane: all (remote) loads first, then the local
  // gathers of acc / w, then the stores — three round trips per batch.
  constexpr int R = 4;
  auto land_batch = [&](const uint64_t (&pos)[R], const bool (&ok)[R], const uint32_t (&i)[R],
                        const double (&v)[R]) {
    float av[R], wv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      av[k] = (acc && ok[k]) ? acc[i[k]] : 0.f;
      wv[k] = (wm && ok[k]) ? wm[i[k]] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (!ok[k]) continue;
      ui[pos[k]] = i[k];
      uv[pos[k]] = v[k];
      if (acc) {
        // K7 (oktopk.cpp:299-302, trainer.cpp:437-442, 478-479) on the entry.
        const bool sel = fabsf(av[k]) >= tf;
        if (wm) {
          const float nw = float(double(wv[k]) - v[k] / dP);
          wm[i[k]] = nw;
          bad |= (__float_as_uint(nw) & 0x7f800000u) == 0x7f800000u;
          if (sel) acc[i[k]] = 0.f;
        }
        if (ap.sel) ap.sel[pos[k]] = sel ? 1 : 0;
      }
    }
  };
  if (round == 0) {
    const uint64_t a = bal ? s_blk[me] : 0, b = bal ? s_blk[me + 1] : s_off[P];
    // (rank, chunk, part) work items: every chunk split so all warps get a share
    const uint32_t items = s_start[P];
    const uint32_t warps_total = gridDim.x * kWarps;
    const uint32_t parts = max(1u, min(8u, warps_total / max(1u, items)));
    for (uint32_t it = blockIdx.x * kWarps + warp; it < items * parts; it += warps_total) {
      const uint32_t item = it / parts, part = it % parts;
      int r = 0;
      while (r + 1 < P && item >= s_start[r + 1]) ++r;
      const uint32_t c = item - s_start[r];
      const uint64_t base = s_off[r] + tab->spre[r][par][c];
      const uint64_t end = base + tab->scnt[r][par][c];
      const uint64_t len = end - base;
      const uint64_t lo = max(base + len * part / parts, a), hi = min(base + len * (part + 1) / parts, b);
      const uint32_t* si = tab->sidx[r][par] + uint64_t(c) * s_cap[r];
      const double* sv = tab->sval[r][par] + uint64_t(c) * s_cap[r];
      for (uint64_t p0 = lo; p0 < hi; p0 += 32 * R) {
        uint64_t pos[R];
        bool ok[R];
        uint32_t i[R];
        double v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
          pos[k] = p0 + lane + 32 * k;
          ok[k] = pos[k] < hi;
          i[k] = ok[k] ? si[pos[k] - base] : 0u;
          v[k] = ok[k] ? sv[pos[k] - base] : 0.0;
        }
        land_batch(pos, ok, i, v);
      }
    }
  } else {
    const uint64_t total = s_off[P];
    const uint64_t stride = uint64_t(gridDim.x) * kThreads;
    for (uint64_t pos = uint64_t(blockIdx.x) * kThreads + threadIdx.x; pos < total; pos += stride) {
      int r = 0;
      while (r + 1 < P && pos >= s_blk[r + 1]) ++r;
      uint64_t pa[R] = {pos, 0, 0, 0};
      bool ok[R] = {!(pos >= s_blk[me] && pos < s_blk[me + 1]), false, false, false};  // not my own block
      uint32_t i[R] = {ok[0] ? tab->u_idx[r][par][pos] : 0u, 0, 0, 0};
      double v[R] = {ok[0] ? tab->u_val[r][par][pos] : 0.0, 0.0, 0.0, 0.0};
      land_batch(pa, ok, i, v);
    }
  }
  if (acc && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(d_flags, 4u);
  if (lane == 0) trace_stamp(trace, trk, 2);
}

// Balanced case only: publish "my block is in u", wait for every other block.
__global__ void p2p_block_sync_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, const P2PPlan* plan,
                                      uint32_t* d_flags, uint64_t timeout_ns) {
  const uint64_t epoch = sp->epoch;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  if (!plan->balanced || (*d_flags & (1u | 8u | 16u))) return;
  __syncthreads();
  if (q < P && q != me) {
    __threadfence_system();
    st_relaxed_sys(&tab->hdr[q]->flag[kFlagBlockReady][me], epoch);
  }
  if (q < P && q != me && !wait_flag(&tab->hdr[me]->flag[kFlagBlockReady][q], epoch, timeout_ns))
    atomicOr(d_flags, 8u);
}

// ---- launchers ----------------------------------------------------------------------------
cudaError_t launch_p2p_scatter(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, P2PPlan* plan, uint64_t lo,
                               uint64_t W, uint64_t n, uint32_t* mask, float* stage, uint32_t* d_flags,
                               uint64_t timeout_ns) {
  const uint32_t k1_tiles = uint32_t((n + kK1Tile - 1) / kK1Tile);
  p2p_scatter_kernel<<<L.sms * 2, kThreads, 0, L.s>>>(d_tab, sp, plan, lo, W, k1_tiles, mask, stage, d_flags,
                                                      timeout_ns);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_p2p_allgatherv(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, const uint64_t* d_S,
                                  P2PPlan* plan, uint64_t* d_U, uint32_t* d_flags, uint64_t timeout_ns,
                                  const P2PApply& ap, const K1Totals& totals) {
  const int grid = L.sms * 2;
  p2p_pull_kernel<<<grid, kThreads, 0, L.s>>>(d_tab, sp, const_cast<uint64_t*>(d_S), plan, d_U, 0, d_flags, timeout_ns, ap,
                                              K1Totals{});
  p2p_block_sync_kernel<<<1, 32, 0, L.s>>>(d_tab, sp, plan, d_flags, timeout_ns);
  p2p_pull_kernel<<<grid, kThreads, 0, L.s>>>(d_tab, sp, const_cast<uint64_t*>(d_S), plan, d_U, 1, d_flags, timeout_ns, ap,
                                              totals);
  L.launches += 3;
  return cudaGetLastError();
}

}  // namespace okt
