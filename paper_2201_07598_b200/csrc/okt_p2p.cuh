// okt_p2p.cuh — device-driven multi-GPU exchange over NVLink peer memory.
//
// Every rank owns one symmetric window (same layout on all ranks) that its
// peers map: through CUDA IPC across processes, or directly within one
// process.  Phases hand data over with release/acquire flags instead of host
// synchronisation:
//   publish  the producer stores its payload, fences at system scope, then
//            stores flag[kind][copy][me].epoch into every peer's window header;
//   wait     the consumer spins (ld.acquire.sys, bounded by a timeout) on its
//            own header until every peer's flag reached the epoch, then reads
//            the payload that came with it from the same slot.
// Bulk data never moves through a staging copy: the consumer's kernels read
// the producer's buffers in place over NVLink (pull model), e.g. the merge
// reads each source's K1 tiles straight out of that source's HBM.
// Buffers a peer may still read are double-buffered by step parity; a rank can
// only run one step ahead of a peer (each step waits on every peer), so a
// parity slot is never rewritten while someone reads it.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace okt {

constexpr int kP2PMaxP = 8;

// Per-step arguments read from device memory, so one captured CUDA graph
// serves every steady step (the graph refreshes this block from pinned host
// memory as its first node).
struct StepPtrs {
  const float* g;
  const float* eps_in;
  float* eps_out;
  float* w;
  float alpha;
  float pad;
  uint64_t epoch;  // P2P: flag value of this step; P = 1 graph: step sequence number
  int32_t par;     // P2P: parity slot of the window buffers
  int32_t pad2;
  uint64_t* trace;   // diagnostics (OKT_P2P_TRACE): per-CTA stamps, or null
};
enum P2PFlag { kFlagLReady = 0, kFlagSurReady = 1, kFlagBlockReady = 2, kFlagBarrier = 3, kP2PFlagKinds = 4 };

// What a rank publishes for its peers each step (double-buffered by parity).
struct P2PPub {
  uint64_t status;   // non-zero: this rank's step failed (non-finite input)
  uint64_t S;        // survivors of the global threshold
  uint32_t k1_G;     // K1 chunk geometry: chunks and entries per chunk
  uint32_t k1_cap;
  uint32_t sur_G;     // survivor chunks: contiguous spans of the region's tiles (a few per merge CTA)
  uint32_t sur_tiles; // merge tiles of the region (chunk c starts at split(c) * kK1Tile)
  uint64_t pad[4];
};

// Flags are replicated: a publisher stores its epoch into kFlagCopies copies
// (one 128-byte line each) at every rank, and CTA b polls copy b % kFlagCopies
// — a few hundred CTAs polling a single line contend on one L2 slice and see
// the flag microseconds apart, and fanning a flag out inside the grid costs a
// fence that waits for the grid's own traffic.
// A flag slot carries the words its consumers need (status, counts,
// geometry) next to the epoch, so a consumer reads them from its own memory
// instead of every CTA reading the source's header over NVLink.
constexpr int kFlagCopies = 32, kFlagWords = 7;
struct FlagSlot {
  uint64_t epoch;
  uint64_t v[kFlagWords];  // payload, valid once epoch is observed
};
struct P2PHdr {
  FlagSlot flag[kP2PFlagKinds][kFlagCopies][kP2PMaxP];  // [kind][copy][source rank], written by the sources
  P2PPub pub[2];
};

// Peer table: every rank's window pieces (index = rank), both parities.  The
// chunked phase-A outputs are consumed in place: no compaction pass sits
// between a producer and its peers.
struct PeerTab {
  P2PHdr* hdr[kP2PMaxP];
  uint64_t* kstg[kP2PMaxP][2];  // K1 chunk-local staging (AoS u32 idx | f32 val)
  uint32_t* kcnt[kP2PMaxP][2];  // entries per K1 chunk
  uint32_t* klt[kP2PMaxP][2];   // [chunk][kP2PMaxP] entries below each cut
  uint32_t* sidx[kP2PMaxP][2];  // region-scan chunk staging (survivors)
  double* sval[kP2PMaxP][2];
  uint32_t* scnt[kP2PMaxP][2];  // survivors per chunk
  uint64_t* spre[kP2PMaxP][2];  // exclusive prefix of scnt (chunks + 1 entries)
  uint32_t* sbeg[kP2PMaxP][2];  // first region tile of each survivor chunk (the merge's span)
  uint32_t* u_idx[kP2PMaxP][2]; // allgathered u
  double* u_val[kP2PMaxP][2];
  int P;
  int rank;
  uint64_t* trace;  // diagnostics (OKT_P2P_TRACE): [kTraceKinds][kTraceCtas][4] globaltimer stamps, or null
};
// Per-CTA timestamps of the last P2P step (diagnostics only):
// slot 0 = CTA start, 1 = after its flag waits / prologue, 2 = last warp done.
enum TraceKind {
  kTrK1 = 0, kTrMerge = 1, kTrCompact = 2, kTrPull0 = 3, kTrPull1 = 4,
  kTrPubL = 5, kTrPubSur = 6,  // CTA 0's publish: [before fence, after fence, after the flag stores]
  kTraceKinds = 7
};
constexpr int kTraceCtas = 2048;

// Device-side plan of the balance + allgatherv phase (local memory).
struct P2PPlan {
  uint64_t sizes[kP2PMaxP];
  uint64_t off[kP2PMaxP + 1];    // stream offsets of each rank's survivors
  uint64_t block[kP2PMaxP + 1];  // equal blocks when balanced
  uint64_t total;
  uint32_t balanced;
  uint32_t pad;
  uint64_t seg_off[kP2PMaxP];    // my split slices inside each source's L
  uint64_t seg_cnt[kP2PMaxP];
  uint64_t peer_status[kP2PMaxP];
  uint32_t sur_G[kP2PMaxP];      // every rank's survivor chunk geometry (chunks, region tiles)
  uint32_t sur_tiles[kP2PMaxP];
};

// K7 fused into the allgatherv pull: every u entry is touched once.
struct P2PApply {
  int on = 0;
  uint32_t* flags2 = nullptr;   // argument-fed step: the per-parity flag words; CTA 0 clears flags2[par ^ 1]
  int sgd = 0;                  // acc = sp->eps_out and w = sp->w; else acc = sp->g
  const double* d_local_th = nullptr;
  uint8_t* sel = nullptr;       // per u entry: 1 if in the local selection
  // EF steps: u membership bitmaps (1 bit per coordinate, one per parity).
  // The pull sets u's bits and leaves the residual alone (K1 already zeroed
  // the local selection); the restore kernel then puts acc back at the local
  // entries outside u — indexes = local selection ∩ u (oktopk.cpp:299-302)
  // without a random gather of acc per entry of u.
  uint32_t* ubits[2] = {nullptr, nullptr};
};

// What the host reads after a steady device-driven EF step, written by the
// kernels straight into mapped pinned memory (no D2H node).  The error words
// are written (never cleared) by whichever CTA hits the error; the host clears
// them before each launch.
struct P2PHostOut {
  uint64_t seq_pull, seq_tot;   // the step (epoch) that wrote each part
  uint64_t U, m;
  uint64_t sizes[kP2PMaxP];     // every rank's survivors (the balance plan's input)
  uint64_t seg_cnt[kP2PMaxP];   // entries received from each source
  uint64_t off[kP2PMaxP + 1];   // my selection's slice offsets per destination
  uint32_t flags_early;         // K1 / merge error bits, as the pull saw them
  uint32_t err_timeout, err_peer, err_iter;
};

// P2P mode of K1: its per-tile staging, counts and cut counts go straight into
// this rank's window, where the peers' merge kernels read them in place.
struct K1P2P {
  const PeerTab* tab = nullptr;  // device copy
  const StepPtrs* sp = nullptr;  // epoch / parity of the step
  const uint64_t* cuts = nullptr;
  // Argument-fed step (EF steps; no H2D node): the step block travels here by
  // value, K1's CTA 0 stores it at sp_out for the later kernels and zeroes the
  // plan; par_v replaces sp->par inside K1.
  int par_v = -1;
  StepPtrs* sp_out = nullptr;
  P2PPlan* plan_zero = nullptr;
  StepPtrs spv{};
  // EF steps: store the residual of every locally selected entry as 0 (the
  // restore kernel puts acc back where the entry did not make it into u).
  int zero_sel = 0;
  // This rank's selection size and slice offsets (the entries below cut d, d <
  // P; all, d = P), for the result and the ledger: every CTA adds its tiles'
  // counts into tot_acc (kP2PMaxP + 1 words, zero before the first launch),
  // and the last CTA out publishes them to d_off / d_m (and hout) and re-arms.
  uint64_t* tot_acc = nullptr;
  uint64_t* d_off = nullptr;
  uint64_t* d_m = nullptr;
  struct P2PHostOut* hout = nullptr;
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Publishing to P ranks: one __threadfence_system() (fence.sc.sys), then a
// relaxed system-scope store per rank — the fence-based release pattern.  A
// st.release.sys per rank would pay one system fence each (~1.8 us apiece on
// B200; tools/p2p_lat.cu measures it).
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void trace_stamp(uint64_t* tr, int kind, int slot, bool max = false) {
  if (tr && blockIdx.x < kTraceCtas) {
    uint64_t* p = tr + (uint64_t(kind) * kTraceCtas + blockIdx.x) * 4 + slot;
    if (slot == 2 || max)
      atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)globaltimer_ns());
    else
      *p = globaltimer_ns();
  }
}

// Spin until *p >= epoch; false after `timeout_ns` (a peer died or diverged).
__device__ __forceinline__ bool wait_flag(const uint64_t* p, uint64_t epoch, uint64_t timeout_ns) {
  if (ld_acquire_sys(p) >= epoch) return true;
  const uint64_t t0 = globaltimer_ns();
  while (true) {
    __nanosleep(64);
    if (ld_acquire_sys(p) >= epoch) return true;
    if (globaltimer_ns() - t0 > timeout_ns) return false;
  }
}

// Every thread of the publishing CTA, after a __syncthreads: the payload,
// then the epoch, into every copy of this rank's slot of flag `kind` at every
// rank.  Each storing thread fences between its payload and its epoch stores
// (the fence-based release pattern; the fences run in parallel).
template <int NPAY>
__device__ __forceinline__ void publish_flag(P2PHdr* const* hdr, int P, int me, int kind, uint64_t epoch,
                                             const uint64_t (&pay)[NPAY]) {
  static_assert(NPAY <= kFlagWords, "flag payload");
  const int total = P * kFlagCopies;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    FlagSlot* slot = &hdr[i / kFlagCopies]->flag[kind][i % kFlagCopies][me];
#pragma unroll
    for (int k = 0; k < NPAY; ++k) st_relaxed_sys(&slot->v[k], pay[k]);
    __threadfence_system();
    st_relaxed_sys(&slot->epoch, epoch);
  }
}
// This CTA's copy of source q's slot of flag `kind` in my header.
__device__ __forceinline__ const FlagSlot* my_flag(const P2PHdr* mine, int kind, int q) {
  return &mine->flag[kind][blockIdx.x % kFlagCopies][q];
}
// Payload word k of a slot whose epoch this thread has acquired.
__device__ __forceinline__ uint64_t flag_word(const FlagSlot* f, int k) {
  return *reinterpret_cast<const volatile uint64_t*>(&f->v[k]);
}
// Same, without payload.
__device__ __forceinline__ void publish_flag(P2PHdr* const* hdr, int P, int me, int kind, uint64_t epoch) {
  const int total = P * kFlagCopies;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    __threadfence_system();
    st_relaxed_sys(&hdr[i / kFlagCopies]->flag[kind][i % kFlagCopies][me].epoch, epoch);
  }
}
}  // namespace okt
