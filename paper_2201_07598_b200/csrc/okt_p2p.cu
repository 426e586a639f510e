// okt_p2p.cu — kernels of the device-driven multi-GPU exchange (okt_p2p.cuh).
//
// Steady Ok-Topk iteration on P ranks, no host round trip and no compaction
// pass between a producer and its consumers (one CUDA graph):
//   K1 (per-tile staging + per-tile cut counts in the window; its last CTA
//     publishes the selection size and slice offsets)
//   merge: CTA 0 publishes L-ready; every CTA waits on its own flag copy, reads
//     every source's K1 tiles of its region in place (NVLink) and runs the
//     bracket scan / survivor filter in shared memory; survivors chunked into
//     the window
//   pull: CTA 0 publishes the survivor prefix and count; every CTA waits, plans
//     (offsets, balance) and pulls every chunk to its position in u, applying
//     K7 on the way [balanced: my block, an in-grid hand-off, the others]
// Every publish is issued at a kernel start, while the rest of the grid only
// polls: a system fence issued while the grid streams random stores waits for
// that traffic to drain (tools/fence_lat.cu, tools/p2p_noise.cu).
#include "okt_device.cuh"
#include "okt_kernels.hpp"
#include "okt_p2p.cuh"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace okt {

namespace {
constexpr uint32_t kAbortBits = 1u | 8u | 16u;  // local non-finite, peer timeout, peer failure
}

// K3 on the device-driven path: the split exchange and the region merge fused
// into one kernel, with no random global traffic.  A CTA owns one K1 tile t
// (4096 coordinates) of my region: after every source's L-ready, it reads
// each source's compacted entries of tile t (in place: NVLink for a peer —
// the entries of a tile are contiguous and coordinate-sorted), scatters them
// into a shared-memory mask / stage, and runs the bracket scan + global
// threshold filter over the tile from shared memory, writing the tile's
// survivors as one chunk (capacity 4096) of the survivor staging.  (Random
// 4-byte global stores — a global-memory scatter — stall every system fence
// on the GPU for tens of microseconds; tools/p2p_noise.cu.)
constexpr int kMergeTile = kK1Tile;              // coordinates per CTA tile
constexpr int kMergePer = kMergeTile / kThreads;  // 16 coordinates per thread in the scan
template <int P>
// tiles of entries in flight per CTA (OKT_MERGE_STAGES_* at build time, A/B)
#ifndef OKT_MERGE_STAGES_SMALL
#define OKT_MERGE_STAGES_SMALL 12
#endif
#ifndef OKT_MERGE_STAGES_P8
#define OKT_MERGE_STAGES_P8 6
#endif
__host__ __device__ constexpr int merge_stages() { return P <= 4 ? OKT_MERGE_STAGES_SMALL : OKT_MERGE_STAGES_P8; }
#ifndef OKT_MERGE_RING
#define OKT_MERGE_RING 96
#endif
constexpr int kMergeRing = OKT_MERGE_RING;        // entries per source per ring stage (a denser tile's rest: direct)
constexpr int kMergeCntCap = 256;
#ifndef OKT_MERGE_SPLIT_DEFAULT
#define OKT_MERGE_SPLIT_DEFAULT 0
#endif
constexpr int kMergeBalD = 2;  // merge span weights by SM round: 16 - 2 r (16 : 14 : 12 at 3 CTAs per SM)
constexpr int kMergeSplit = OKT_MERGE_SPLIT_DEFAULT;  // survivor spans per merge CTA, ticketed (0: one, static)                 // tiles whose counts are staged at once

template <int P>
__host__ __device__ constexpr size_t merge_smem() {  // mask bytes, values [P][tile], ring [S][P][kMergeRing], counts
  return size_t(kMergeTile) + size_t(P) * kMergeTile * sizeof(float) +
         size_t(merge_stages<P>()) * P * kMergeRing * sizeof(uint64_t) + size_t(kMergeCntCap) * P * sizeof(uint32_t);
}

// First tile of span c when `tiles` tiles are split evenly over G spans.
// (floor(c * tiles / G) without the 64-bit division subroutine: the product
// is < 2^53, so the double quotient is within one of the answer; fix it up.)
__device__ __forceinline__ uint32_t span_at(uint32_t c, uint32_t tiles, uint32_t G) {
  const uint64_t m = uint64_t(c) * tiles;
  uint64_t qv = uint64_t(double(m) / double(G));
  if (qv * G > m) --qv;
  else if ((qv + 1) * G <= m) ++qv;
  return uint32_t(qv);
}

// floor(len * p / q) for q <= 64 (no 64-bit division subroutine).
__device__ __forceinline__ uint64_t frac_at(uint64_t len, uint32_t p, uint32_t q) {
  if (len < (1ull << 26)) return uint32_t(len) * p / q;
  const uint64_t m = len * p;
  uint64_t v = uint64_t(double(m) / double(q));
  if (v * q > m) --v;
  else if ((v + 1) * q <= m) ++v;
  return v;
}

// TMA bulk copies into the ring, completion tracked by one mbarrier per stage.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n"
      "}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16-byte async copy, L2 only (.cg: no L1 line of a peer's buffer survives
// into a later step that reuses the same parity slot).
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// P = 2 is capped at 48 registers: 5 CTAs per SM instead of 4 (shared memory
// allows 6), so more of the region's tiles are in flight at once (interleaved
// A/B on one box, tools/ab_lib.sh: steady N = 2 0.0812 -> 0.0799 ms).
template <int P, bool TMA>
__global__ void __launch_bounds__(kThreads, P == 2 ? 4 : 2)
    p2p_merge_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, P2PPlan* plan, uint64_t lo, uint64_t W,
                     uint32_t k1_tiles, const double* d_gth, uint32_t* d_flags, uint64_t timeout_ns,
                     uint32_t split, uint32_t* ctr) {
  extern __shared__ uint32_t sm[];
  uint32_t* s_mask = sm;                                             // [kMergeTile / 4]: byte per coordinate, bit per source
  float* s_val = reinterpret_cast<float*>(sm + kMergeTile / 4);      // [P][kMergeTile]
  __shared__ uint32_t s_wt[kWarps];
  __shared__ uint32_t s_seg[P];
  __shared__ int s_abort;
  const uint64_t epoch = sp->epoch;
  const int par = sp->par;
  const int me = tab->rank, q = threadIdx.x, lane = q & 31, warp = q >> 5;
  uint64_t* const trace = tab->trace;
  if (q == 0) {
    s_abort = (*d_flags & 1u) ? 1 : 0;
    trace_stamp(trace, kTrMerge, 0);
  }
  if (q < P) s_seg[q] = 0;
  __syncthreads();  // s_abort / s_seg initialised before any thread may set them
  const uint64_t hi = lo + W;
  const uint32_t t_lo = uint32_t(lo / kMergeTile);
  const uint32_t ntiles = W ? uint32_t((hi - 1) / kMergeTile) - t_lo + 1 : 0;
  // survivor chunks: `split` per CTA, handed out by a ticket counter
  // (split 0: one span per CTA, span = blockIdx.x, no tickets; bits 8+ of the
  // argument: a diagnostic permutation of that static assignment)
  const uint32_t perm = (split >> 8) & 0xffu;
  const uint32_t bal_d = (split >> 16) & 0xffu, bal_cps = split >> 24;  // static span weights by SM round, see below
  split &= 0xffu;
  const uint32_t Gc = split ? max(1u, min(ntiles, gridDim.x * split)) : gridDim.x;
  uint32_t span0 = blockIdx.x;
  if (perm == 1) span0 = gridDim.x - 1 - blockIdx.x;  // reversed
  else if (perm == 2 && gridDim.x % 148 == 0)         // the CTAs of one SM (b, b + 148, ...) on adjacent spans
    span0 = (blockIdx.x % 148) * (gridDim.x / 148) + blockIdx.x / 148;
  else if (perm == 3) span0 = uint32_t((uint64_t(blockIdx.x) * 7919u) % gridDim.x);  // scattered (7919 prime)
  if (blockIdx.x == 0) {
    // this rank's K1 output: status, then L-ready at every rank (the GPU is
    // quiet: K1 finished and nobody streams yet)
    if (q == 0) {
      P2PPub* pub = &tab->hdr[me]->pub[par];  // (read by this rank's pull)
      pub->sur_G = Gc;
      pub->sur_tiles = ntiles;
      trace_stamp(trace, kTrPubL, 0);
    }
    const uint64_t pay[3] = {(*d_flags & 1u) ? 1ull : 0ull, k1_tiles, uint64_t(kK1Tile)};
    publish_flag(tab->hdr, P, me, kFlagLReady, epoch, pay);
    if (q == 0) trace_stamp(trace, kTrPubL, 3);
  }
  // every source's L-ready (each CTA polls its own flag copy)
  if (q < P && q != me) {
    const FlagSlot* f = my_flag(tab->hdr[me], kFlagLReady, q);
    if (!wait_flag(&f->epoch, epoch, timeout_ns)) {
      atomicOr(d_flags, 8u);
      s_abort = 1;
    } else {
      const uint64_t st = flag_word(f, 0);
      if (st || flag_word(f, 1) != k1_tiles || flag_word(f, 2) != uint64_t(kK1Tile)) {
        atomicOr(d_flags, 16u);
        s_abort = 1;
      }
      if (blockIdx.x == 0) plan->peer_status[q] = st;
    }
  }
  __syncthreads();
  if (q == 0) trace_stamp(trace, kTrMerge, 1);
  const double gth = *d_gth;
  uint32_t* const out_idx = tab->sidx[me][par];
  double* const out_val = tab->sval[me][par];
  uint32_t* const out_cnt = tab->scnt[me][par];
  // The region's tiles in Gc contiguous spans: one per CTA (default; sized
  // by the CTA's round on its SM, below), or `split` per CTA taken by ticket
  // (OKT_MERGE_SPLIT; slower, DESIGN 7.5).  Span c's survivors: one
  // contiguous chunk at j0 * kMergeTile (the span's capacity), count in
  // out_cnt[c], start j0 in sbeg[c] — a few hundred large chunks per rank for
  // the pull instead of one small chunk per tile.  The span's
  // per-source counts are staged in shared memory first (all loads in flight
  // at once), then a kS-deep ring of TMA bulk copies (cp.async.bulk, one per
  // source and tile, issued by one thread, completion counted in bytes on the
  // stage's mbarrier) keeps the entries of the next tiles of every source in
  // flight over NVLink while a tile is merged (the first kMergeRing entries of
  // a tile per source; a denser tile's rest is read directly).  Round 1 kept
  // one tile in flight: 6.8 us per tile at n = 340M, P = 4, almost all of it
  // NVLink latency.
  uint64_t* const ring = reinterpret_cast<uint64_t*>(s_val + P * kMergeTile);    // [S][P][kMergeRing]
  constexpr int kS = merge_stages<P>();
  uint32_t* const s_cnt = reinterpret_cast<uint32_t*>(ring + kS * P * kMergeRing);  // [kMergeCntCap][P]
  // Static spans sized by the CTA's round on its SM: the merge CTAs of one SM
  // (blocks b, b + R, b + 2R, ... with R = grid / CTAs per SM) do not progress
  // equally — the SM's warp scheduler favours the older CTA, so with equal
  // spans at BERT-L N = 2 the first CTA of every SM finished at 135 us and
  // the third at 174 us, whatever data the spans held (reversed / permuted
  // span orders moved the slow CTAs with the block index, not with the
  // span), and the SM ran short-handed meanwhile.  CTA b in round r gets a
  // span weighted 16 - d r (d = bal_d), so an SM's CTAs finish together.
  __shared__ uint32_t s_bnd[2];
  bool wbal = false;
  // (Only at >= 3 CTAs per SM, P = 2: at P = 4, two per SM, the rounds differed
  // by 4 %, within the spread of the spans' own costs.)
  if (!split && perm == 0 && bal_d && bal_cps >= 3 && gridDim.x % bal_cps == 0 && ntiles) {
    const uint32_t R = gridDim.x / bal_cps;
    auto f = [&](uint32_t r) -> uint64_t { return uint64_t(max(1, 16 - int(bal_d) * int(r))); };
    auto C = [&](uint32_t b) -> uint64_t {  // summed weights of blocks < b
      const uint32_t r = b / R, rem = b % R;
      uint64_t c = 0;
      for (uint32_t i = 0; i < r; ++i) c += uint64_t(R) * f(i);
      return c + uint64_t(rem) * (r < bal_cps ? f(r) : 0);
    };
    if (q < 2) {
      const uint64_t Ct = C(gridDim.x);
      s_bnd[q] = uint32_t(uint64_t(ntiles) * C(blockIdx.x + uint32_t(q)) / Ct);
    }
    wbal = true;
    __syncthreads();
  }
  __shared__ uint32_t s_tk[2];
  if (q == 0) s_tk[0] = split ? atomicAdd(&ctr[0], 1u) : span0;
  // entries received from each source (the ledger's split words), per thread:
  // reduced once at the end instead of a warp reduce + shared atomic per
  // source and tile
  uint32_t seg_mine[P];
#pragma unroll
  for (int r = 0; r < P; ++r) seg_mine[r] = 0;
  uint64_t ph_acc[4] = {0, 0, 0, 0};  // diagnostics (trace on): ns in wait / scatter / scan / emit, thread 0
  for (int w = q; w < kMergeTile / 16; w += kThreads) reinterpret_cast<uint4*>(s_mask)[w] = make_uint4(0, 0, 0, 0);
  __shared__ __align__(8) uint64_t s_mbar[32];  // one per ring stage
  if (q == 0) {
    for (int st = 0; st < kS; ++st) mbar_init(&s_mbar[st], 1);
    fence_proxy_async_smem();  // (the initialised barriers, visible to the copy engine)
  }
  uint32_t ph_bits = 0;  // the parity each stage's barrier completes next (every thread tracks it)
  __syncthreads();
  for (int tpar = 0;; tpar ^= 1) {
  const uint32_t cidx = s_tk[tpar];
  if (cidx >= Gc) break;
  if (trace && q == 0 && tpar == 0 && blockIdx.x < kTraceCtas) {  // diagnostics: SM and first span of the CTA
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trace[(uint64_t(kTrMerge) * kTraceCtas + blockIdx.x) * 4 + 3] = (uint64_t(smid) << 32) | cidx;
  }
  if (q == 0) s_tk[tpar ^ 1] = split ? atomicAdd(&ctr[0], 1u) : Gc;  // (read after this span's barriers)
  const uint32_t j0 = wbal ? s_bnd[0] : span_at(cidx, ntiles, Gc);
  const uint32_t my_n = (wbal ? s_bnd[1] : span_at(cidx + 1, ntiles, Gc)) - j0;
  if (q == 0) tab->sbeg[me][par][cidx] = j0;  // (the pull finds the chunk's survivors there)
  const uint64_t out_base = uint64_t(j0) * kMergeTile;
  uint32_t running = 0;  // survivors of this span so far (block-uniform)
  for (uint32_t i0 = 0; i0 < my_n; i0 += kMergeCntCap) {
    const uint32_t ni = min(my_n - i0, uint32_t(kMergeCntCap));
    for (uint32_t x = q; x < ni * P; x += kThreads) {
      const uint32_t i = x / P;
      const int r = int(x % P);
      s_cnt[x] = s_abort ? 0u : tab->kcnt[r][par][t_lo + j0 + i0 + i];
    }
    __syncthreads();
    auto issue = [&](uint32_t i) {  // ring stage i % S <- tile i's first entries, every source
      if constexpr (!TMA) {
        // cp.async (LDGSTS) by every thread: 16-byte pairs of entries
        if (i < ni) {
          const uint64_t base = uint64_t(t_lo + j0 + i0 + i) * kMergeTile;
          uint64_t* slot = ring + (i % kS) * (P * kMergeRing);
          for (int x = q; x < P * kMergeRing / 2; x += kThreads) {
            const int r = x / (kMergeRing / 2), e = 2 * (x % (kMergeRing / 2));
            if (uint32_t(e) < s_cnt[i * P + r]) cp_async16(slot + r * kMergeRing + e, tab->kstg[r][par] + base + e);
          }
        }
        cp_async_commit();  // (empty groups keep the group count uniform)
      } else if (i < ni && q == 0) {
        // TMA bulk copies issued by thread 0, completion on the stage's mbarrier
        const uint64_t base = uint64_t(t_lo + j0 + i0 + i) * kMergeTile;
        uint64_t* slot = ring + (i % kS) * (P * kMergeRing);
        uint64_t* mb = &s_mbar[i % kS];
        // whole 16-byte pairs of entries (a tile's staging slot starts 16-byte
        // aligned and holds kMergeTile entries, so an odd count's partner is in bounds)
        uint32_t bytes[P], total = 0;
#pragma unroll
        for (int r = 0; r < P; ++r) {
          const uint32_t c = min(s_cnt[i * P + r], uint32_t(kMergeRing));
          bytes[r] = ((c + 1u) & ~1u) * 8u;
          total += bytes[r];
        }
        fence_proxy_async_smem();  // the slot's earlier generic reads before the copy engine's writes
        mbar_expect_tx(mb, total);
#pragma unroll
        for (int r = 0; r < P; ++r)
          if (bytes[r]) bulk_g2s(slot + r * kMergeRing, tab->kstg[r][par] + base, bytes[r], mb);
      }
    };
#pragma unroll
    for (int st = 0; st < kS - 1; ++st) issue(uint32_t(st));
    for (uint32_t i = 0; i < ni; ++i) {
      uint64_t ph0 = 0;
      if (trace && q == 0) ph0 = globaltimer_ns();
      if constexpr (TMA) {
        mbar_wait(&s_mbar[i % kS], (ph_bits >> (i % kS)) & 1u);  // stage i landed
        ph_bits ^= 1u << (i % kS);
      } else {
        cp_async_wait<kS - 2>();
      }
      __syncthreads();  // the slot of tile i - 1 is free; tile i - 1 is emitted
      issue(i + kS - 1);
      if (trace && q == 0) ph_acc[0] += globaltimer_ns() - ph0, ph0 = globaltimer_ns();  // (wait + issue)
      const uint32_t t = t_lo + j0 + i0 + i;
      const uint64_t base = uint64_t(t) * kMergeTile;
      const uint64_t* slot = ring + (i % kS) * (P * kMergeRing);
#pragma unroll
      for (int r = 0; r < P; ++r) {
        auto land = [&](uint64_t ent) {
          const uint64_t idx = coo_idx(ent);
          OKT_DCHECK(idx >= base && idx < base + kMergeTile, "merge: a source's tile entry outside its tile", idx, base);
          if (idx < lo || idx >= hi) return;  // the region's edge tiles
          const uint32_t c = uint32_t(idx - base);
          s_val[r * kMergeTile + c] = coo_val(ent);
          atomicOr(&s_mask[c >> 2], 1u << ((c & 3u) * 8u + uint32_t(r)));
          ++seg_mine[r];
        };
        const uint32_t cr = s_cnt[i * P + r];
        OKT_DCHECK(cr <= uint32_t(kMergeTile), "merge: tile count above the tile", cr, r);
        for (uint32_t e = q; e < cr; e += kThreads)
          land(e < uint32_t(kMergeRing) ? slot[r * kMergeRing + e] : tab->kstg[r][par][base + e]);
      }
      __syncthreads();
      if (trace && q == 0) ph_acc[1] += globaltimer_ns() - ph0, ph0 = globaltimer_ns();
      // bracket scan + filter over the tile: thread q owns coordinates
      // [16 q, 16 q + 16) (four mask words)
      const uint4 mw4 = reinterpret_cast<const uint4*>(s_mask)[q];
      reinterpret_cast<uint4*>(s_mask)[q] = make_uint4(0, 0, 0, 0);  // (this thread's words: clear for the next tile)
      auto bits_of = [&](int k) {  // source bits of coordinate k (select tree: no local memory)
        const int jj = k >> 2;
        const uint32_t w = (jj & 2) ? ((jj & 1) ? mw4.w : mw4.z) : ((jj & 1) ? mw4.y : mw4.x);
        return (w >> (8 * (k & 3))) & 0xffu;
      };
      auto nib = [](uint32_t w) { return ((__vcmpne4(w, 0u) & 0x01010101u) * 0x01020408u) >> 24; };
      const uint32_t present = nib(mw4.x) | (nib(mw4.y) << 4) | (nib(mw4.z) << 8) | (nib(mw4.w) << 12);
      uint32_t sel = 0;
      for (uint32_t rest = present; rest; rest &= rest - 1) {
        const int k = __ffs(rest) - 1;
        const uint32_t c = uint32_t(q) * kMergePer + uint32_t(k);
        float v[P];
#pragma unroll
        for (int r = 0; r < P; ++r) v[r] = s_val[r * kMergeTile + c];
        if (fabs(bracket_regs<P>(v, bits_of(k))) >= gth) sel |= 1u << k;
      }
      const uint32_t n_sel = __popc(sel);
      uint32_t incl = n_sel;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane == 31) s_wt[warp] = incl;
      __syncthreads();
      if (trace && q == 0) ph_acc[2] += globaltimer_ns() - ph0, ph0 = globaltimer_ns();
      uint32_t wpre = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        wpre += (w < warp) ? s_wt[w] : 0u;
        total += s_wt[w];
      }
      uint64_t pos = out_base + running + wpre + incl - n_sel;
      for (uint32_t rest = sel; rest; rest &= rest - 1, ++pos) {
        const int k = __ffs(rest) - 1;
        const uint32_t c = uint32_t(q) * kMergePer + uint32_t(k);
        float v[P];
#pragma unroll
        for (int r = 0; r < P; ++r) v[r] = s_val[r * kMergeTile + c];
        OKT_DCHECK(pos < out_base + uint64_t(my_n) * kMergeTile, "merge: survivor beyond the CTA's chunk", pos, out_base);
        out_idx[pos] = uint32_t(base + c);
        out_val[pos] = bracket_regs<P>(v, bits_of(k));
      }
      running += total;
      if (trace && q == 0) ph_acc[3] += globaltimer_ns() - ph0;
      // (no barrier here: the next tile's first barrier separates this emit
      // from its scatter; s_wt is rewritten only after its second one)
    }
    if constexpr (!TMA) cp_async_wait<0>();
    __syncthreads();
  }
  if (q == 0) out_cnt[cidx] = running;
  __syncthreads();  // (an empty span has no barrier of its own)
  }
  if (split && q == 0) {
    // the last CTA out re-arms the ticket counter for the next launch
    __threadfence();
    if (atomicAdd(&ctr[1], 1u) == gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
  if (trace && q == 0 && blockIdx.x < kTraceCtas) {  // (the balanced pull's slots: free on merge-traced steps)
    uint64_t* tp = trace + (uint64_t(kTrPull1) * kTraceCtas + blockIdx.x) * 4;
    for (int x = 0; x < 4; ++x) tp[x] = ph_acc[x];
  }
#pragma unroll
  for (int r = 0; r < P; ++r) {
    const uint32_t g = __reduce_add_sync(0xffffffffu, seg_mine[r]);
    if (lane == 0 && g) atomicAdd(&s_seg[r], g);
  }
  __syncthreads();
  if (q < P && s_seg[q]) atomicAdd(reinterpret_cast<unsigned long long*>(&plan->seg_cnt[q]), (unsigned long long)s_seg[q]);
  if (lane == 0) trace_stamp(trace, kTrMerge, 2);
}

// Allgatherv by pulling.  Every CTA waits for every rank's survivors and
// derives the plan of balance_and_allgatherv (oktopk.cpp:172-231; identical on
// all ranks), then one warp per (rank, chunk, part) copies survivors from the
// owner's window to their stream position in my u (unbalanced: all of u;
// balanced: my block, then — after every owner's block is complete — the
// other blocks from their owners' u).  K7 runs on each entry as it lands.
__global__ void __launch_bounds__(kThreads, 3)
    p2p_pull_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, uint64_t* d_S, P2PPlan* plan,
                    uint64_t* d_U, uint32_t* d_flags, uint64_t timeout_ns, P2PApply ap, P2PHostOut* hout,
                    uint32_t* done) {
  __shared__ int s_last;
  __shared__ uint64_t s_size[kP2PMaxP], s_off[kP2PMaxP + 1], s_blk[kP2PMaxP + 1];
  __shared__ uint32_t s_G[kP2PMaxP], s_tiles[kP2PMaxP], s_start[kP2PMaxP + 1];
  __shared__ int s_bal, s_abort;
  const uint64_t epoch = sp->epoch;
  const int par = sp->par;
  float* acc = ap.on ? (ap.sgd ? sp->eps_out : const_cast<float*>(sp->g)) : nullptr;
  float* wm = (ap.on && ap.sgd) ? sp->w : nullptr;
  uint32_t* const ubits = (ap.on && ap.sgd) ? (sp->par ? ap.ubits[1] : ap.ubits[0]) : nullptr;
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* const trace = tab->trace;
  if (q == 0) {
    s_abort = (*d_flags & (1u | 8u | 16u)) ? 1 : 0;
    trace_stamp(trace, kTrPull0, 0);
    // done[par] counts this step's CTAs through the balanced hand-off; the
    // previous step cleared it, this one clears the next step's
    if (blockIdx.x == 0) {
      done[par ^ 1] = 0;
      if (ap.flags2) ap.flags2[par ^ 1] = 0;  // the next argument-fed step's flag word
    }
  }
  __syncthreads();
  {
    // CTA 0 publishes this rank's survivors (every region-scan CTA finished
    // before this kernel started; the other CTAs only poll, so the system
    // fence is cheap): the exclusive prefix of the chunk counts (where each
    // chunk lands in my part of u), S, status, then survivors-ready at every
    // rank.
    if (blockIdx.x == 0) {
      P2PPub* mine = &tab->hdr[me]->pub[par];
      const int G = int(mine->sur_G);
      const uint32_t* cnt = tab->scnt[me][par];
      uint64_t* pre = tab->spre[me][par];
      const int per = (G + kThreads - 1) / kThreads;
      const int c0 = q * per, c1 = min(G, (q + 1) * per);
      uint64_t own = 0;
      for (int cb = c0; cb < c1; cb += 8) {  // 8 loads in flight per round
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = cb + u < c1 ? cnt[cb + u] : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) own += v[u];
      }
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
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        wpre += (w < warp) ? wsum[w] : 0;
        tot += wsum[w];
      }
      uint64_t run = wpre + incl - own;
      for (int c = c0; c < c1; ++c) {
        pre[c] = run;
        run += cnt[c];
      }
      __syncthreads();
      if (q == 0) {
        pre[G] = tot;
        *d_S = tot;
        trace_stamp(trace, kTrPubSur, 0);
      }
      __syncthreads();
      const uint64_t pay[4] = {(*d_flags & kAbortBits) ? 1ull : 0ull, tot, uint64_t(G), uint64_t(mine->sur_tiles)};
      publish_flag(tab->hdr, P, me, kFlagSurReady, epoch, pay);
      if (q == 0) trace_stamp(trace, kTrPubSur, 3);
    }
    // every CTA: wait on its own flag copies, read the ranks' survivor counts
    // and geometry, derive the plan (CTA 0 also stores it for the host).  A
    // step that already failed (its merge timed out on a dead peer) does not
    // wait again: its own abort status went out with the publication above.
    if (q < P) {
      uint64_t sz = 0;
      uint32_t G = 0, cap = 0;
      const FlagSlot* f = my_flag(tab->hdr[me], kFlagSurReady, q);
      if (!wait_flag(&f->epoch, epoch, s_abort ? 0 : timeout_ns)) {
        atomicOr(d_flags, 8u);
        if (hout) hout->err_timeout = 1;
        s_abort = 1;
      } else {
        sz = flag_word(f, 1);
        G = uint32_t(flag_word(f, 2));
        cap = uint32_t(flag_word(f, 3));
        if (q != me && flag_word(f, 0)) {
          atomicOr(d_flags, 16u);
          if (hout) hout->err_peer = 1;
          s_abort = 1;
        }
      }
      s_size[q] = sz;
      s_G[q] = G;
      s_tiles[q] = cap;
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
        for (int r = 0; r < P; ++r) {
          plan->sizes[r] = s_size[r];
          plan->sur_G[r] = s_G[r];
          plan->sur_tiles[r] = s_tiles[r];
        }
        for (int r = 0; r <= P; ++r) {
          plan->off[r] = s_off[r];
          plan->block[r] = s_blk[r];
        }
        plan->total = total;
        plan->balanced = uint32_t(s_bal);
        *d_U = s_abort ? 0 : total;
        if (hout) {  // the step's plan for the host's commit and ledger (mapped memory)
          hout->U = s_abort ? 0 : total;
          for (int r = 0; r < P; ++r) {
            hout->sizes[r] = s_size[r];
            hout->seg_cnt[r] = *reinterpret_cast<volatile uint64_t*>(&plan->seg_cnt[r]);  // (merge finished)
          }
          hout->flags_early = *reinterpret_cast<volatile uint32_t*>(d_flags);
          hout->seq_pull = epoch;
        }
      }
    }
  }
  __syncthreads();
  if (q == 0) trace_stamp(trace, kTrPull0, 1);
  if (s_abort) return;
  const bool bal = s_bal != 0;
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
      av[k] = (acc && !ubits && ok[k]) ? acc[i[k]] : 0.f;
      wv[k] = (wm && ok[k]) ? ld_rand(wm + i[k]) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (!ok[k]) continue;
      ui[pos[k]] = i[k];
      uv[pos[k]] = v[k];
      if (ubits) {
        // EF step: the residual was settled by K1 (local selection stored as
        // 0) and is fixed up by the restore kernel; mark u's entry
        atomicOr(&ubits[i[k] >> 5], 1u << (i[k] & 31u));
        const float nw = float(double(wv[k]) - v[k] / dP);
        wm[i[k]] = nw;
        bad |= (__float_as_uint(nw) & 0x7f800000u) == 0x7f800000u;
      } else if (acc) {
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
  {
    const uint64_t a = bal ? s_blk[me] : 0, b = bal ? s_blk[me + 1] : s_off[P];
    // (rank, chunk, part) work items: every chunk split so all warps get a share
    const uint32_t items = s_start[P];
    const uint32_t warps_total = gridDim.x * kWarps;
    // (a chunk is one merge CTA's span: thousands of entries at large n)
    const uint32_t parts = max(1u, min(64u, warps_total / max(1u, items)));
    for (uint32_t it = blockIdx.x * kWarps + warp; it < items * parts; it += warps_total) {
      const uint32_t item = it / parts, part = it % parts;
      int r = 0;
      while (r + 1 < P && item >= s_start[r + 1]) ++r;
      const uint32_t c = item - s_start[r];
      const uint64_t base = s_off[r] + tab->spre[r][par][c];
      const uint64_t end = base + tab->scnt[r][par][c];
      const uint64_t len = end - base;
      OKT_DCHECK(end <= s_off[r + 1], "pull: chunk beyond its rank's survivors", end, s_off[r + 1]);
      const uint64_t lo = max(base + frac_at(len, part, parts), a), hi = min(base + frac_at(len, part + 1, parts), b);
      const uint64_t cbase = uint64_t(tab->sbeg[r][par][c]) * kMergeTile;  // (the merge's span start)
      const uint32_t* si = tab->sidx[r][par] + cbase;
      const double* sv = tab->sval[r][par] + cbase;
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
  }
  if (bal) {
    // Balanced: the other blocks come from their block owners' u once each
    // owner's round 0 is complete.  The last CTA of my grid to finish round 0
    // publishes "my block is complete" (a grid-wide hand-off through a
    // per-parity counter: every CTA is resident, the grid is one wave);
    // every CTA waits for every peer's block on its own flag copy.
    __syncthreads();
    if (q == 0) {
      __threadfence();
      s_last = atomicAdd(&done[par], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      publish_flag(tab->hdr, P, me, kFlagBlockReady, epoch);
    }
    if (q < P && q != me && !wait_flag(&my_flag(tab->hdr[me], kFlagBlockReady, q)->epoch, epoch, timeout_ns)) {
      atomicOr(d_flags, 8u);
      if (hout) hout->err_timeout = 1;
      s_abort = 1;
    }
    __syncthreads();
    if (s_abort) return;
    if (q == 0) trace_stamp(trace, kTrPull1, 0);
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
  if (acc && __syncthreads_or(bad) && threadIdx.x == 0) {
    atomicOr(d_flags, 4u);
    if (hout) hout->err_iter = 1;
  }
  if (lane == 0) trace_stamp(trace, kTrPull0, 2);
}

// EF steps, after the pull: the residual of every locally selected entry
// outside u goes back to acc (K1 stored 0 for the whole local selection), so
// eps ends as acc zeroed at indexes = local selection ∩ u (trainer.cpp:
// 476-480, oktopk.cpp:299-302).  One warp per K1 tile of my staging; the u
// bitmap of the next step is cleared on the way.
__global__ void __launch_bounds__(kThreads)
    p2p_restore_kernel(const PeerTab* __restrict__ tab, const StepPtrs* sp, uint32_t* ub0, uint32_t* ub1,
                       uint64_t nwords, const uint32_t* flags2, const uint32_t* d_flags) {
  const int me = tab->rank, par = sp->par;
  if (threadIdx.x == 0) trace_stamp(tab->trace, kTrCompact, 0);  // (diagnostics: the restore uses the compact slot)
  const uint32_t* ub = par ? ub1 : ub0;
  uint32_t* ub_next = par ? ub0 : ub1;
  const uint64_t gt = uint64_t(blockIdx.x) * kThreads + threadIdx.x, gstride = uint64_t(gridDim.x) * kThreads;
  for (uint64_t w = gt; w < (nwords >> 2); w += gstride) reinterpret_cast<uint4*>(ub_next)[w] = make_uint4(0, 0, 0, 0);
  for (uint64_t w = (nwords & ~uint64_t(3)) + gt; w < nwords; w += gstride) ub_next[w] = 0u;
  const uint32_t fl = flags2 ? flags2[par] : *d_flags;
  if (fl & kAbortBits) return;  // a failed step commits nothing
  float* eps = sp->eps_out;
  const uint32_t G = tab->hdr[me]->pub[par].k1_G;
  const uint32_t* cnt = tab->kcnt[me][par];
  const uint64_t* stg = tab->kstg[me][par];
  // A warp takes kRT tiles per round and keeps their loads in flight together
  // (counts, then two entries per lane and tile, then the bitmap words): three
  // memory round trips per round instead of three per tile.
  constexpr int kRT = 4;
  const int lane = threadIdx.x & 31;
  const uint64_t wid = gt >> 5, wstride = gstride >> 5;
  for (uint64_t t0 = wid * kRT; t0 < G; t0 += wstride * kRT) {
    uint32_t c[kRT];
#pragma unroll
    for (int x = 0; x < kRT; ++x) {
      c[x] = t0 + x < G ? cnt[t0 + x] : 0u;
      OKT_DCHECK(c[x] <= uint32_t(kK1Tile), "restore: tile count above the tile", c[x], t0 + x);
    }
    uint64_t e[kRT][2];
#pragma unroll
    for (int x = 0; x < kRT; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const uint32_t j = lane + 32u * y;
        e[x][y] = j < c[x] ? stg[(t0 + x) * kK1Tile + j] : ~0ull;
      }
    uint32_t bw[kRT][2];
#pragma unroll
    for (int x = 0; x < kRT; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) bw[x][y] = e[x][y] != ~0ull ? ub[coo_idx(e[x][y]) >> 5] : ~0u;
#pragma unroll
    for (int x = 0; x < kRT; ++x) {
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const uint32_t i = coo_idx(e[x][y]);
        if (e[x][y] != ~0ull && !((bw[x][y] >> (i & 31u)) & 1u)) eps[i] = coo_val(e[x][y]);
      }
      for (uint32_t j = 64 + lane; j < c[x]; j += 32) {  // a dense tile's rest
        const uint64_t ee = stg[(t0 + x) * kK1Tile + j];
        const uint32_t i = coo_idx(ee);
        if (!((ub[i >> 5] >> (i & 31u)) & 1u)) eps[i] = coo_val(ee);
      }
    }
  }
  if (lane == 0) trace_stamp(tab->trace, kTrCompact, 2);
}

cudaError_t launch_p2p_restore(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, uint32_t* ub0, uint32_t* ub1,
                               uint64_t n, const uint32_t* flags2, const uint32_t* d_flags) {
  const int grid = L.sms * 8;
  p2p_restore_kernel<<<grid, kThreads, 0, L.s>>>(d_tab, sp, ub0, ub1, (n + 31) / 32, flags2, d_flags);
  ++L.launches;
  return cudaGetLastError();
}

// okt_device_barrier: publish, then wait for every peer (one CTA).
__global__ void p2p_barrier_kernel(const PeerTab* __restrict__ tab, uint64_t epoch, uint32_t* d_flags,
                                   uint64_t timeout_ns) {
  const int P = tab->P, me = tab->rank, q = threadIdx.x;
  publish_flag(tab->hdr, P, me, kFlagBarrier, epoch);
  if (q < P && q != me && !wait_flag(&tab->hdr[me]->flag[kFlagBarrier][0][q].epoch, epoch, timeout_ns))
    atomicOr(d_flags, 8u);
}

// ---- launchers ----------------------------------------------------------------------------
// Test hook (see setup_p2p): shrink the spinning kernels' grids so that
// several ranks sharing one GPU fit side by side.
static int grid_div() {
  static const int d = std::getenv("OKT_P2P_GRID_DIV") ? std::max(1, std::atoi(std::getenv("OKT_P2P_GRID_DIV"))) : 1;
  return d;
}

// The merge ring's copies: cp.async (LDGSTS, default) or TMA bulk copies
// (OKT_MERGE_TMA=1).  Per-tile copies are ~330 bytes per source at 1 %
// density; as TMA bulk copies from the peers they arrived too slowly to keep
// the ring ahead (N = 4, 340M: the merge waited 364 us of 504 on its barriers).
static bool merge_tma() {
  static const bool on = std::getenv("OKT_MERGE_TMA") != nullptr;
  return on;
}

template <int P>
static cudaError_t merge_dispatch(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, P2PPlan* plan, uint64_t lo,
                                  uint64_t W, uint32_t k1_tiles, const double* d_gth, uint32_t* d_flags,
                                  uint64_t timeout_ns, uint32_t* ctr) {
  constexpr size_t smem = merge_smem<P>();
  auto kern = merge_tma() ? p2p_merge_kernel<P, true> : p2p_merge_kernel<P, false>;
  static std::atomic<int> caps[64];  // per device (the dynamic-smem opt-in is per device)
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& cap = caps[dev & 63];
  if (!cap) {
    cudaFuncSetAttribute(p2p_merge_kernel<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(p2p_merge_kernel<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = std::max(1, per_sm * L.sms / grid_div());
  }
  const uint64_t ntiles = W ? (lo + W - 1) / kMergeTile - lo / kMergeTile + 1 : 0;
  const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, uint64_t(cap))));
  static const uint32_t split = [] {  // survivor spans per CTA (OKT_MERGE_SPLIT)
    const char* e = std::getenv("OKT_MERGE_SPLIT");
    const int v = e ? std::atoi(e) : kMergeSplit;
    const char* pe = std::getenv("OKT_MERGE_PERM");  // (diagnostics: permuted static spans)
    const int pm = pe ? std::atoi(pe) : 0;
    // static spans weighted 16 - d r by the CTA's round r on its SM (OKT_MERGE_BAL=d, default kMergeBalD; 0: equal)
    const char* be = std::getenv("OKT_MERGE_BAL");
    const int bd = be ? std::atoi(be) : kMergeBalD;
    return uint32_t(std::max(0, std::min(v, 64))) | (uint32_t(std::max(0, std::min(pm, 3))) << 8) |
           (uint32_t(std::max(0, std::min(bd, 15))) << 16);
  }();
  const uint32_t cps = uint32_t(std::min(15, std::max(1, cap.load() / std::max(1, L.sms)))) << 24;  // CTAs per SM
  kern<<<grid, kThreads, smem, L.s>>>(d_tab, sp, plan, lo, W, k1_tiles, d_gth, d_flags, timeout_ns, split | cps, ctr);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_p2p_merge(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, P2PPlan* plan, int P, uint64_t lo,
                             uint64_t W, uint64_t n, const double* d_gth, uint32_t* d_flags, uint64_t timeout_ns,
                             uint32_t* ctr) {
  const uint32_t k1_tiles = uint32_t((n + kK1Tile - 1) / kK1Tile);
  switch (P) {
    case 2: return merge_dispatch<2>(L, d_tab, sp, plan, lo, W, k1_tiles, d_gth, d_flags, timeout_ns, ctr);
    case 4: return merge_dispatch<4>(L, d_tab, sp, plan, lo, W, k1_tiles, d_gth, d_flags, timeout_ns, ctr);
    case 8: return merge_dispatch<8>(L, d_tab, sp, plan, lo, W, k1_tiles, d_gth, d_flags, timeout_ns, ctr);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_p2p_allgatherv(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, uint64_t* d_S,
                                  P2PPlan* plan, uint64_t* d_U, uint32_t* d_flags, uint64_t timeout_ns,
                                  const P2PApply& ap, P2PHostOut* hout, uint32_t* done) {
  // one wave of as many CTAs as fit (every CTA waits on its own flag copy, so
  // the whole grid must be resident)
  static std::atomic<int> caps[64];  // per device (the dynamic-smem opt-in is per device)
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& cap = caps[dev & 63];
  if (!cap) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p2p_pull_kernel, kThreads, 0) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    cap = std::max(1, std::min(per_sm, 4) * L.sms / grid_div());
  }
  const int grid = cap;
  p2p_pull_kernel<<<grid, kThreads, 0, L.s>>>(d_tab, sp, d_S, plan, d_U, d_flags, timeout_ns, ap, hout, done);
  ++L.launches;
  return cudaGetLastError();
}

cudaError_t launch_p2p_barrier(Launch& L, const PeerTab* d_tab, uint64_t epoch, uint32_t* d_flags,
                               uint64_t timeout_ns) {
  p2p_barrier_kernel<<<1, kThreads, 0, L.s>>>(d_tab, epoch, d_flags, timeout_ns);
  ++L.launches;
  return cudaGetLastError();
}

const void* p2p_merge_func(int P) {
  switch (P) {
    case 2: return merge_tma() ? reinterpret_cast<const void*>(p2p_merge_kernel<2, true>)
                               : reinterpret_cast<const void*>(p2p_merge_kernel<2, false>);
    case 4: return merge_tma() ? reinterpret_cast<const void*>(p2p_merge_kernel<4, true>)
                               : reinterpret_cast<const void*>(p2p_merge_kernel<4, false>);
    case 8: return merge_tma() ? reinterpret_cast<const void*>(p2p_merge_kernel<8, true>)
                               : reinterpret_cast<const void*>(p2p_merge_kernel<8, false>);
  }
  return nullptr;
}
const void* p2p_pull_func() { return reinterpret_cast<const void*>(p2p_pull_kernel); }
const void* p2p_restore_func() { return reinterpret_cast<const void*>(p2p_restore_kernel); }

// (see preload_kernels in okt_kernels.cu)
void preload_p2p_kernels() {
  cudaFuncAttributes a;
  for (const void* f : {reinterpret_cast<const void*>(p2p_merge_kernel<2, false>),
                        reinterpret_cast<const void*>(p2p_merge_kernel<4, false>),
                        reinterpret_cast<const void*>(p2p_merge_kernel<8, false>),
                        reinterpret_cast<const void*>(p2p_merge_kernel<2, true>),
                        reinterpret_cast<const void*>(p2p_merge_kernel<4, true>),
                        reinterpret_cast<const void*>(p2p_merge_kernel<8, true>),
                        reinterpret_cast<const void*>(p2p_pull_kernel),
                        reinterpret_cast<const void*>(p2p_restore_kernel),
                        reinterpret_cast<const void*>(p2p_barrier_kernel)})
  {
    cudaFuncGetAttributes(&a, f);
    if (carveout_pref() >= 0) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pref());
  }
}

}  // namespace okt
