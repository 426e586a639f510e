// okt_p2p.cu — kernels of the device-driven multi-GPU exchange (okt_p2p.cuh).
//
// Steady Ok-Topk iteration on P ranks, no host round trip:
//   K1 -> slice offsets -> publish(L ready)
//   wait(L ready) -> scatter reads my slices from every peer's L over NVLink
//   -> bracket scan / survivor filter into my window -> publish(survivors)
//   wait(survivors) -> plan (offsets, balance) -> pull every part into u
//   [balanced: pull my block, publish(block), wait, pull the other blocks]
//   -> apply.
#include "okt_device.cuh"
#include "okt_kernels.hpp"
#include "okt_p2p.cuh"

#include <algorithm>

namespace okt {

namespace {
constexpr uint32_t kAbortBits = 1u | 8u | 16u;  // local non-finite, peer timeout, peer failure
}

// K1 phase B on the P2P path: copy each chunk to its final position in the
// window's L.  K1's phase A already counted, per chunk, the entries below
// every cut; the last CTA to finish turns those counts into the slice
// offsets, publishes them with this rank's status, and raises L-ready at every
// peer.
__global__ void __launch_bounds__(kThreads)
    p2p_compact_L_kernel(const uint64_t* __restrict__ s64, const uint32_t* __restrict__ counts, uint64_t cap,
                         uint64_t* d_m, PubL pb) {
  __shared__ uint64_t red[kWarps];
  __shared__ int s_last;
  const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x, P = pb.P;
  const int par = pb.sp->par;
  uint64_t* __restrict__ out = pb.tab->L[pb.tab->rank][par];
  const uint64_t cnt = counts[c];
  const uint64_t src = uint64_t(c) * cap;
  uint64_t pre = 0;
  for (int q = tid; q < c; q += kThreads) pre += counts[q];
  pre = block_sum(pre, red);
  for (uint64_t j = tid; j < cnt; j += kThreads) out[pre + j] = s64[src + j];
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(pb.done, 1u) == unsigned(G - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  uint64_t tot = 0;
  for (int q = tid; q < G; q += kThreads) tot += counts[q];
  tot = block_sum(tot, red);
  const PeerTab* tab = pb.tab;
  const int me = tab->rank;
  P2PPub* mine = &tab->hdr[me]->pub[par];
  for (int d = 0; d < P; ++d) {
    uint64_t o = 0;
    for (int q = tid; q < G; q += kThreads) o += pb.lt[uint64_t(q) * kP2PMaxP + d];
    o = block_sum(o, red);
    if (tid == 0) {
      pb.d_off[d] = o;
      mine->off[d] = o;
    }
  }
  if (tid == 0) {
    pb.d_off[P] = tot;
    mine->off[P] = tot;
    mine->status = (*pb.flags & 1u) ? 1 : 0;
    *d_m = tot;
    *pb.done = 0;
  }
  __threadfence_system();
  __syncthreads();
  if (tid < P && tid != me) st_release_sys(&tab->hdr[tid]->flag[kFlagLReady][me], pb.sp->epoch);
}

// K3 (M1) fused with the split exchange.  Each CTA waits until every peer's
// L is published, then scatters my region's entries read straight out of the
// peers' HBM (NVLink) into the presence mask / coordinate-major staging.
__global__ void __launch_bounds__(kThreads)
    p2p_scatter_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, const uint64_t* d_off,
                       P2PPlan* plan, uint64_t lo, uint64_t W, uint32_t* mask, float* stage, uint32_t* d_flags,
                       uint64_t timeout_ns) {
  const uint64_t epoch = sp->epoch;
  const int par = sp->par;
  __shared__ uint64_t s_start[kP2PMaxP + 1];
  __shared__ const uint64_t* s_ptr[kP2PMaxP];
  __shared__ uint64_t s_cnt[kP2PMaxP];
  __shared__ int s_abort;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  if (q == 0) s_abort = (*d_flags & 1u) ? 1 : 0;
  __syncthreads();
  if (q < P) {
    uint64_t o0 = 0, c = 0, st = 0;
    if (q == me) {
      o0 = d_off[me];
      c = d_off[me + 1] - o0;
    } else if (!wait_flag(&tab->hdr[me]->flag[kFlagLReady][q], epoch, timeout_ns)) {
      atomicOr(d_flags, 8u);
      s_abort = 1;
    } else {
      const volatile P2PPub* pub = &tab->hdr[q]->pub[par];
      o0 = pub->off[me];
      c = pub->off[me + 1] - o0;
      st = pub->status;
      if (st) {
        atomicOr(d_flags, 16u);
        s_abort = 1;
      }
    }
    s_ptr[q] = tab->L[q][par] + o0;
    s_cnt[q] = c;
    if (blockIdx.x == 0) {
      plan->seg_off[q] = o0;
      plan->seg_cnt[q] = c;
      plan->peer_status[q] = st;
    }
  }
  __syncthreads();
  if (s_abort) return;
  if (q == 0) {
    uint64_t acc = 0;
    for (int r = 0; r < P; ++r) {
      s_start[r] = acc;
      acc += s_cnt[r];
    }
    s_start[P] = acc;
  }
  __syncthreads();
  const uint64_t total = s_start[P];
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  for (uint64_t e = uint64_t(blockIdx.x) * kThreads + threadIdx.x; e < total; e += stride) {
    int r = 0;
    while (r + 1 < P && e >= s_start[r + 1]) ++r;
    const uint64_t entry = s_ptr[r][e - s_start[r]];
    const uint64_t idx = coo_idx(entry);
    if (idx < lo || idx - lo >= W) {
      atomicOr(d_flags, 2u);
      continue;
    }
    const uint64_t i = idx - lo;
    stage[i * uint64_t(P) + r] = coo_val(entry);
    atomicOr(&mask[i >> 2], 1u << (unsigned(i & 3u) * 8u + unsigned(r)));
  }
}

// Allgatherv by pulling.  round 0 waits for every rank's survivor count and
// derives the plan of balance_and_allgatherv (oktopk.cpp:172-231; identical on
// all ranks), then pulls: unbalanced -> every part from its owner's
// survivors; balanced -> my block from the owners' survivors.  round 1
// (balanced only) pulls the other blocks from their block owners' u.
__global__ void __launch_bounds__(kThreads)
    p2p_pull_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, const uint64_t* d_S, P2PPlan* plan,
                    uint64_t* d_U, int round, uint32_t* d_flags, uint64_t timeout_ns, P2PApply ap) {
  const uint64_t epoch = sp->epoch;
  const int par = sp->par;
  float* acc = ap.on ? (ap.sgd ? sp->eps_out : const_cast<float*>(sp->g)) : nullptr;
  float* wm = (ap.on && ap.sgd) ? sp->w : nullptr;
  __shared__ uint64_t s_size[kP2PMaxP], s_off[kP2PMaxP + 1], s_blk[kP2PMaxP + 1];
  __shared__ int s_bal, s_abort;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  if (q == 0) s_abort = (*d_flags & (1u | 8u | 16u)) ? 1 : 0;
  __syncthreads();
  if (round == 0) {
    if (q < P) {
      uint64_t sz = 0;
      if (q == me) {
        sz = *d_S;
      } else if (!wait_flag(&tab->hdr[me]->flag[kFlagSurReady][q], epoch, timeout_ns)) {
        atomicOr(d_flags, 8u);
        s_abort = 1;
      } else {
        const volatile P2PPub* pub = &tab->hdr[q]->pub[par];
        sz = pub->S;
        if (pub->status) {
          atomicOr(d_flags, 16u);
          s_abort = 1;
        }
      }
      s_size[q] = sz;
    }
    __syncthreads();
    if (q == 0) {
      uint64_t total = 0, maxs = 0;
      s_off[0] = 0;
      for (int r = 0; r < P; ++r) {
        total += s_size[r];
        maxs = max(maxs, s_size[r]);
        s_off[r + 1] = total;
      }
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
  if (s_abort) return;
  const bool bal = s_bal != 0;
  if (round == 1 && !bal) return;
  uint32_t* ui = tab->u_idx[me][par];
  double* uv = tab->u_val[me][par];
  const uint64_t total = s_off[P];
  uint64_t a = 0, b = total;
  if (round == 0 && bal) {
    a = s_blk[me];
    b = s_blk[me + 1];
  }
  const uint64_t span = b - a;
  const uint64_t stride = uint64_t(gridDim.x) * kThreads;
  const float tf = acc ? ceil_to_float(*ap.d_local_th) : 0.f;
  const double dP = double(P);
  bool bad = false;
  for (uint64_t x = uint64_t(blockIdx.x) * kThreads + threadIdx.x; x < span; x += stride) {
    const uint64_t pos = a + x;
    if (round == 1 && pos >= s_blk[me] && pos < s_blk[me + 1]) continue;  // my own block
    int r = 0;
    uint32_t i;
    double v;
    if (round == 0) {
      while (r + 1 < P && pos >= s_off[r + 1]) ++r;
      const uint64_t j = pos - s_off[r];
      i = tab->sur_idx[r][par][j];
      v = tab->sur_val[r][par][j];
    } else {
      while (r + 1 < P && pos >= s_blk[r + 1]) ++r;
      i = tab->u_idx[r][par][pos];
      v = tab->u_val[r][par][pos];
    }
    ui[pos] = i;
    uv[pos] = v;
    if (acc) {
      // K7 (oktopk.cpp:299-302, trainer.cpp:437-442, 478-479) on the entry.
      const float av = acc[i];
      const bool sel = fabsf(av) >= tf;
      if (wm) {
        const float nw = float(double(wm[i]) - v / dP);
        wm[i] = nw;
        bad |= (__float_as_uint(nw) & 0x7f800000u) == 0x7f800000u;
      }
      if (wm && sel) acc[i] = 0.f;
      ap.sel[pos] = sel ? 1 : 0;
    }
  }
  if (acc && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(d_flags, 4u);
}

// Balanced case only: publish "my block is in u", wait for every other block.
__global__ void p2p_block_sync_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, const P2PPlan* plan,
                                      uint32_t* d_flags, uint64_t timeout_ns) {
  const uint64_t epoch = sp->epoch;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  if (!plan->balanced || (*d_flags & (1u | 8u | 16u))) return;
  __threadfence_system();
  __syncthreads();
  if (q < P && q != me) st_release_sys(&tab->hdr[q]->flag[kFlagBlockReady][me], epoch);
  if (q < P && q != me && !wait_flag(&tab->hdr[me]->flag[kFlagBlockReady][q], epoch, timeout_ns))
    atomicOr(d_flags, 8u);
}

// ---- launchers ----------------------------------------------------------------------------
cudaError_t launch_p2p_compact_L(Launch& L, const Stage& S, uint32_t G, uint64_t chunk_cap, uint64_t* out,
                                 uint64_t* d_m, const PubL& pub) {
  (void)out;  // the window slot of this step's parity, chosen on the device
  p2p_compact_L_kernel<<<G, kThreads, 0, L.s>>>(S.s64, S.counts, chunk_cap, d_m, pub);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_p2p_scatter(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, const uint64_t* d_off,
                               P2PPlan* plan, uint64_t lo, uint64_t W, uint32_t* mask, float* stage,
                               uint32_t* d_flags, uint64_t timeout_ns) {
  p2p_scatter_kernel<<<L.sms * 2, kThreads, 0, L.s>>>(d_tab, sp, d_off, plan, lo, W, mask, stage, d_flags,
                                                      timeout_ns);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_p2p_allgatherv(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, const uint64_t* d_S,
                                  P2PPlan* plan, uint64_t* d_U, uint32_t* d_flags, uint64_t timeout_ns,
                                  const P2PApply& ap) {
  const int grid = L.sms * 2;
  p2p_pull_kernel<<<grid, kThreads, 0, L.s>>>(d_tab, sp, d_S, plan, d_U, 0, d_flags, timeout_ns, ap);
  p2p_block_sync_kernel<<<1, 32, 0, L.s>>>(d_tab, sp, plan, d_flags, timeout_ns);
  p2p_pull_kernel<<<grid, kThreads, 0, L.s>>>(d_tab, sp, d_S, plan, d_U, 1, d_flags, timeout_ns, ap);
  L.launches += 3;
  return cudaGetLastError();
}

}  // namespace okt
