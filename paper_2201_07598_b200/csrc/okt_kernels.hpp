// okt_kernels.hpp — host launchers for the sm_100a Ok-Topk kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "okt_p2p.cuh"

namespace okt {

// Per-comm launch context: stream and launch accounting.
struct Launch {
  cudaStream_t s = nullptr;
  uint64_t launches = 0;        // kernels launched through this context
  int sms = 148;
  // Profiling: when set, the K1 streaming kernel (phase A) is bracketed by a
  // pair of events from this pool (also captured into CUDA graphs).
  cudaEvent_t (*k1_event)(void* ctx) = nullptr;
  void* k1_ctx = nullptr;
};

struct RadixState {
  uint64_t prefix;
  uint64_t kk;
  uint32_t active;
  uint32_t pad;
};

enum class K1Mode { kSelect, kAccumSelect, kAccumHist, kAccumSelectHist };
enum class RadixSrc { kDenseF32, kAosF32, kF64 };

// Phase-A staging of the two-phase compactions (okt_device.cuh).
struct Stage {
  uint64_t* s64 = nullptr;      // AoS staging (u32 idx | f32 val << 32)
  uint32_t* sidx = nullptr;     // SoA staging indices
  double* sval = nullptr;       // SoA staging values
  uint32_t* counts = nullptr;   // per-chunk emitted counts
  uint32_t* counts2 = nullptr;  // per-chunk secondary counts (K1 dual threshold)
  uint64_t* chunk_cap = nullptr;  // device-computed chunk capacity (entries)
  uint32_t* tile_ctr = nullptr;   // K1 tile tickets [next, CTAs done]; zero between launches
  int max_chunks = 0;
  uint64_t max_tiles = 0;         // counts[] capacity for K1's per-tile counts
  uint64_t* agg = nullptr;        // phase B: per-CTA group totals (tag << 32 | count), >= max_chunks words
  uint32_t* tag_ctr = nullptr;    // host counter tagging phase-B launches (never 0)
};
// Staging entries needed for a pass over `count` elements in tiles of `tile`.
size_t stage_entries(uint64_t count, int tile, int max_chunks);
constexpr int kK1Tile = 4096;   // K1 / region-scan tile (elements)
constexpr int kCooTile = 1024;  // O(k) passes tile (entries)
constexpr int kRegionTileHost = 8192;  // region scan tile (coordinates)

// Output of a compaction: AoS u64 entries or SoA (u32 idx, f64 val).
struct OutCoo {
  uint64_t* aos = nullptr;
  uint32_t* idx = nullptr;
  double* val = nullptr;
};

// Fused K7 for the single-rank path (every entry of u is locally selected).
// What the host reads after a steady single-rank graph step, written by the
// kernels straight into mapped pinned memory (no D2H node): phase B's CTA 0
// writes the counts, and any CTA that detects an error ORs its bit into
// flags (the host clears flags before each launch).
struct HostOut {
  uint64_t seq;  // the step that wrote it (ApplyArgs::seq)
  uint64_t m, S;
  uint32_t flags;     // K1's error bits of the step
  uint32_t bad_iter;  // set by phase B on a non-finite model update (the host clears it)
};

struct ApplyArgs {
  bool k7 = false;        // apply K7 at u's entries (P = 1 EF step; fused into K1)
  float* acc = nullptr;   // residual buffer holding acc; zeroed at u's indices
  float* w = nullptr;     // model; w[i] -= u_i
  uint32_t* d_flags = nullptr;
  const StepPtrs* ind = nullptr;  // when set, acc / w come from here
  HostOut* hout = nullptr;        // when set: the step's scalars go there
  uint64_t seq = 0;               // ... tagged with this step number
  uint32_t* d_flags_next = nullptr;  // when set: CTA 0 clears the next graph step's flag word
  uint64_t* trace = nullptr;      // diagnostics (OKT_P2P_TRACE): per-CTA stamps, kind kTrCompact
  uint32_t tag = 0;               // phase-B launch tag (0: the launcher takes the next from Stage::tag_ctr)
};
// K1's fused single-rank residual zeroing (K1 argument 16).
struct K1Apply {
  float* zero = nullptr;  // select-only pass: the acc buffer, zeroed at every emitted i
};
// The single-rank graph's phase-B kernel, for per-step parameter updates.
const void* compact_graph_kernel(bool apply);

// Split-phase receive segments for the region scatter (M1): one per source.
struct Segs {
  const uint64_t* ptr[8];
  uint64_t start[9];
  int src[8];
  int nseg;
};

// K1: fused residual accumulate + threshold select + order-preserving COO
// compaction over n fp32 elements.  Modes:
//   kSelect       acc = g,                       emit {|acc| >= th}
//   kAccumSelect  acc = fma(alpha, g, eps_in) -> eps_out, emit {|acc| >= th}
//   kAccumHist    acc = fma(alpha, g, eps_in) -> eps_out, radix pass-0 histogram
//   kAccumSelectHist  both: emit {|acc| >= th} (refresh candidates) + the histogram
// With d_th2 (dual threshold) the emitted set is {|acc| >= max(th, th2)} and
// *d_m2 receives |{|acc| >= th}| (P = 1 steady state: u straight from K1).
// Sets bit 0 of *d_flags on any non-finite accumulator.
cudaError_t launch_k1(Launch& L, const Stage& S, K1Mode mode, const float* g, const float* eps_in,
                      float* eps_out, float alpha, uint64_t n, const double* d_th, const double* d_th2,
                      const OutCoo& out, uint64_t* d_m, uint64_t* d_m2, uint32_t* d_flags,
                      uint32_t* d_hist, const ApplyArgs* ap = nullptr, const K1P2P* p2p = nullptr,
                      const StepPtrs* ind = nullptr);

// K2/K4: exact k-th largest magnitude (k clamped to the element count) by MSD
// radix select on the IEEE bit patterns; writes the threshold to *d_th_out
// unless the input is empty.  `hist0_done`: pass 0's histogram was already
// accumulated into d_hist (fused into K1).
cudaError_t launch_radix_select(Launch& L, RadixSrc src, const void* data,
                                uint64_t n_host, const uint64_t* d_n, uint64_t n_bound,
                                uint64_t k, RadixState* d_rs, uint32_t* d_hist,
                                double* d_th_out, bool hist0_done);
// After a fused pass-0 histogram: the pass-0 pick, then the smallest magnitude
// of the chosen bin into *d_floor (the cold refresh's candidate threshold).
cudaError_t launch_radix_pass0_floor(Launch& L, RadixState* d_rs, uint32_t* d_hist, double* d_floor);
// Cold refresh candidates: the pass-0 bin floor of a strided sample of
// |eps + alpha * g| (1 in 2^s_log2 coordinates, one pseudo-random pick per
// block) at sample rank q (from the top), into *d_floor.  d_hist: 2048 words,
// zeroed here; d_rs: a RadixState of its own.
cudaError_t launch_sample_floor(Launch& L, const float* g, const float* eps, float alpha, uint64_t n,
                                uint32_t s_log2, uint64_t q, RadixState* d_rs, uint32_t* d_hist, double* d_floor);
// Zero-initialises the radix state before a fused pass-0 histogram.
cudaError_t launch_radix_init(Launch& L, RadixState* d_rs, uint64_t k, uint64_t n_host,
                              const uint64_t* d_n);

// Survivor filter: {(i, v) : |v| >= *d_th} of a COO list whose length lives in
// device memory.  Input is AoS (u32 idx, f32 val) or SoA (u32, f64); output SoA, or AoS when out_aos
// (f32 values only).
cudaError_t launch_filter(Launch& L, const Stage& S, bool aos, const uint64_t* in_aos,
                          const uint32_t* in_idx, const double* in_val,
                          const uint64_t* d_cnt_in, uint64_t bound, const double* d_th,
                          uint32_t* out_idx, double* out_val, uint64_t* d_cnt_out,
                          const ApplyArgs* ap = nullptr,
                          uint64_t* out_aos = nullptr);

// K7 when indexes = u (one rank): eps[i] = 0, w[i] -= v for every entry of u.
cudaError_t launch_apply_u(Launch& L, const uint32_t* u_idx, const double* u_val, const uint64_t* d_U, uint64_t bound,
                           float* acc, float* w, uint32_t* d_flags);
// K7: for each (i, v) of u: sel = |acc[i]| >= local_th; if w: w[i] -= v / P;
// if zero_eps && sel: acc[i] = 0; emit i into indexes when sel.
cudaError_t launch_apply(Launch& L, const Stage& S, const uint32_t* u_idx, const double* u_val,
                         const uint64_t* d_U, uint64_t bound, float* acc, bool zero_eps,
                         float* w, int P, const double* d_local_th, uint32_t* out_indexes,
                         uint64_t* d_nidx, uint32_t* d_flags);

// K3 (M1): scatter split-phase entries into the owner's presence mask and
// coordinate-major staging [W][P]; out-of-region entries set bit 1 of flags.
cudaError_t launch_scatter(Launch& L, const Segs& segs, uint64_t lo, uint64_t W, int P,
                           uint32_t* mask, float* stage, uint32_t* d_flags);
// K3 (M2): ordered scan of the owned region: bracket-sum the present sources in
// fp64, keep explicit zeros, optionally filter by |sum| >= *d_gth, clear mask.
cudaError_t launch_region_scan(Launch& L, const Stage& S, int P, bool filter, uint64_t lo, uint64_t W,
                               uint32_t* mask, const float* stage, const double* d_gth,
                               uint32_t* out_idx, double* out_val, uint64_t* d_count);

// Small control kernels.
cudaError_t launch_slice_offsets(Launch& L, const uint64_t* coo, const uint64_t* d_m,
                                 const uint64_t* d_cuts, int P, uint64_t* d_off,
                                 uint32_t* d_cnt_out, const uint32_t* d_flags);
cudaError_t launch_proposals(Launch& L, const uint32_t* idx, int stride,
                             const uint64_t* d_m, uint64_t m_host, uint64_t n, int P,
                             uint64_t* d_prop);
cudaError_t launch_cuts(Launch& L, const uint64_t* d_allprop, int P, uint64_t n,
                        uint64_t* d_cuts);
cudaError_t launch_extract(Launch& L, const uint64_t* coo, const uint64_t* d_m,
                           uint64_t bound, uint32_t* idx, double* val);
cudaError_t launch_widen_f32(Launch& L, const float* in, uint64_t n, double* out);

// Input generators (bit-exact with proj/core/include/oklab/rng.hpp streams).
cudaError_t launch_gen_random_dense(Launch& L, float* out, uint64_t n, uint64_t seed);
cudaError_t launch_gen_noise(Launch& L, float* out, uint64_t n, uint64_t noise_key,
                             double coef);
cudaError_t launch_scatter_heavy(Launch& L, const uint32_t* pos, const float* val,
                                 uint64_t count, float* out);

// ---- device-driven multi-GPU exchange (okt_p2p.cu) ----------------------------
// Split exchange + region merge of the steady P2P step (K1's per-tile staging
// of every source read in place; survivors chunked into my window).
cudaError_t launch_p2p_merge(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, P2PPlan* plan, int P, uint64_t lo,
                             uint64_t W, uint64_t n, const double* d_gth, uint32_t* d_flags, uint64_t timeout_ns,
                             uint32_t* ctr);  // ctr: 2 words, zero before the first launch (re-armed by the kernel)
// The P2P kernels, for per-step parameter updates of the instantiated step graph.
const void* p2p_merge_func(int P);
const void* p2p_pull_func();
const void* p2p_restore_func();
// Loads the path's kernels now (lazy module loading would load each at its first launch).
// OKT_CARVEOUT=<0..100>: preferred shared-memory carveout for every kernel (-1: the driver default).
int carveout_pref();
void preload_kernels();
void preload_p2p_kernels();
// EF steps after the pull: acc back at the local entries outside u; clears the next step's u bitmap.
cudaError_t launch_p2p_restore(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, uint32_t* ub0, uint32_t* ub1,
                               uint64_t n, const uint32_t* flags2, const uint32_t* d_flags);
// Waits for every rank's survivors, plans (offsets / balance), pulls u.
cudaError_t launch_p2p_allgatherv(Launch& L, const PeerTab* d_tab, const StepPtrs* sp, uint64_t* d_S,
                                  P2PPlan* plan, uint64_t* d_U, uint32_t* d_flags, uint64_t timeout_ns,
                                  const P2PApply& ap, P2PHostOut* hout, uint32_t* done);
// Device barrier over the peer flags (okt_device_barrier).
cudaError_t launch_p2p_barrier(Launch& L, const PeerTab* d_tab, uint64_t epoch, uint32_t* d_flags,
                               uint64_t timeout_ns);
// indexes = {u_idx[j] : sel[j]} in order (the K7 intersection, after a fused apply).
cudaError_t launch_select_flags(Launch& L, const Stage& S, const uint8_t* sel, const PeerTab* d_tab,
                                const StepPtrs* sp, const uint64_t* d_U, uint64_t bound, uint32_t* out,
                                uint64_t* d_count, const uint32_t* d_flags);

// COO wire codec (okt_wire.cu): out / in are the image as u32 words.
cudaError_t launch_wire_encode(Launch& L, const uint32_t* idx, const double* val, uint64_t nnz, uint32_t* out);
cudaError_t launch_wire_decode(Launch& L, const uint32_t* in, uint64_t nnz, uint64_t n, uint32_t* idx, double* val,
                               uint32_t* err);

// ---- Table-1 baselines (okt_baselines.cu) ----------------------------------------------
// Order-preserving compactions run in chunks of kTopkTrimChunk entries: a
// count pass (per-chunk counts), the host's exclusive prefix, a write pass.
constexpr int kTopkTrimChunk = 1024;
// Exact top-k trim over an AoS f32 (aos != null) or SoA f64 (idx, val) list.
cudaError_t launch_topk_count(Launch& L, const uint64_t* aos, const uint32_t* idx, const double* val, uint64_t m,
                              double th, uint32_t* gt_cnt, uint32_t* eq_cnt);
cudaError_t launch_topk_write(Launch& L, const uint64_t* aos_in, const uint32_t* idx, const double* val, uint64_t m,
                              double th, const uint64_t* off, const uint64_t* eq_before, uint64_t need,
                              uint64_t* aos, uint32_t* out_idx, double* out_val);
// merge_two: positions (tmp of na + nb entries), then heads (off == null: counts).
cudaError_t launch_merge_rank(Launch& L, const uint32_t* ai, const double* av, uint64_t na, const uint32_t* bi,
                              const double* bv, uint64_t nb, uint32_t* ti, double* tv);
cudaError_t launch_merge_heads(Launch& L, const uint32_t* ti, const double* tv, uint64_t N, uint32_t* cnt,
                               const uint64_t* off, uint32_t* oi, double* ov);
cudaError_t launch_dense_nonzero(Launch& L, const double* w, uint64_t W, uint64_t lo, uint32_t* cnt,
                                 const uint64_t* off, uint32_t* oi, double* ov);
cudaError_t launch_aos_to_soa(Launch& L, const uint64_t* aos, uint64_t m, const uint64_t* off, uint32_t* oi,
                              double* ov);
cudaError_t launch_slice_bounds(Launch& L, const uint32_t* idx, uint64_t n, uint64_t lo, uint64_t hi,
                                uint64_t* out);
cudaError_t launch_window_scatter(Launch& L, const uint32_t* idx, const double* val, uint64_t nnz, uint64_t lo,
                                  double* win, bool add);
cudaError_t launch_window_add(Launch& L, double* win, const double* in, uint64_t W);
// Gaussiank: mean and unbiased variance (fp64, fixed reduction shape); partial holds 1024 doubles.
cudaError_t launch_moments(Launch& L, const float* g, uint64_t n, double* partial, double* d_mean, double* d_var);
cudaError_t launch_count_ge(Launch& L, const float* g, uint64_t n, double th, unsigned long long* cnt);

}  // namespace okt
