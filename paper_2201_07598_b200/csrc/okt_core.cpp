// okt_core.cpp — host orchestration of the Ok-Topk sparse allreduce and the
// C-ABI entry points declared in include/okt.h.
//
// One okt_comm per rank.  A step (ok_sparse_allreduce, oktopk.cpp:246-307)
// runs these device phases on the comm's stream:
//   K1  fused accumulate + select + compact           (every iteration)
//   K2  radix select of local_th                      (t-1 ≡ 0 mod tau')
//   K8  proposals + cuts consensus                    (t-1 ≡ 0 mod tau)
//       slice offsets; counts allgather    <- host sync #1 (P > 1)
//       rotated slice exchange (split)
//   K3  scatter + ordered bracket scan of the owned region (fused survivor
//       filter on steady iterations)
//   K4  gather + radix select of global_th + filter  (t-1 ≡ 0 mod tau')
//       survivor-count allgather             <- host sync #2 (P > 1)
//   K5/K6 balance moves + allgatherv into u
//   K7  apply: indexes, residual zero, model update  <- host sync #3
// Thresholds live on the device during a step; the host mirror (okt_state)
// is committed only when the step succeeds, so a failing step leaves the
// state, the residual and the model as the reference leaves them.
#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <unistd.h>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/okt.h"
#include "okt_kernels.hpp"
#include "okt_plan.hpp"
#include "okt_transport.hpp"

using okt::Launch;
using okt::Xfer;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// ---- device buffers ---------------------------------------------------------
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  bool zero_init = false;
  ~Buf() {
    if (p) cudaFree(p);
  }
  // Grow-only.  Rare (capacities track the largest n / counts seen).
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    size_t want = std::max<size_t>(bytes, 256);
    if (p) want = std::max(want, cap + cap / 2);
    if (p) {
      cudaError_t e = cudaFree(p);
      if (e != cudaSuccess) return e;
      p = nullptr;
      cap = 0;
    }
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) return e;
    cap = want;
    if (zero_init) return cudaMemset(p, 0, want);
    return cudaSuccess;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Device-resident scalars of one comm; mirrored to pinned host memory at sync
// points with a single D2H copy.
struct DevScalars {
  double local_th;
  double global_th;
  double th_arg;  // threshold argument of the sub-phase entry points
  double pad0;
  uint64_t m, R, S, U, nidx;
  // The P2P steady step refreshes [sp, plan] with one H2D copy per step
  // (flags and plan zeroed), and reads everything back with one D2H.
  okt::StepPtrs sp;
  uint32_t flags;  // bit0 non-finite input, bit1 out-of-region entry, bit2 non-finite iterate,
                   // bit3 peer timeout, bit4 peer failure
  uint32_t pad1;
  uint32_t pflags[2];  // the single-rank graph step's flag words, by step parity
  uint32_t p2pflags[2];  // the argument-fed P2P step's flag words, by step parity
  okt::P2PPlan plan;
  uint64_t cuts[OKT_MAX_WORLD + 1];
  uint64_t off[OKT_MAX_WORLD + 1];
  uint64_t prop[OKT_MAX_WORLD + 1];
  uint64_t prop_all[OKT_MAX_WORLD * (OKT_MAX_WORLD + 1)];
  uint32_t cnt[OKT_MAX_WORLD + 1];
  uint32_t cnt_all[OKT_MAX_WORLD * (OKT_MAX_WORLD + 1)];
  uint32_t small[2];
  uint32_t small_all[2 * OKT_MAX_WORLD];
  okt::RadixState rs;
  uint32_t merge_ctr[2];  // the P2P merge's span tickets (its last CTA re-arms them)
  uint64_t k1_tot[okt::kP2PMaxP + 1];  // P2P K1's totals accumulators (its last CTA publishes and clears them)
  okt::RadixState rs_sample;  // the cold refresh's sampled candidate threshold
};

bool is_pow2(int v) { return v >= 1 && (v & (v - 1)) == 0; }
using okt::plan::equal_slice_ends;

okt_state default_state() {
  okt_state s;
  std::memset(&s, 0, sizeof(s));
  s.local_th = 0.0;
  s.global_th = 0.0;
  s.tau = 64;
  s.tau_prime = 32;
  s.last_local_eval = -1;
  s.last_global_eval = -1;
  s.regions = -1;
  s.bucket_size = 4;
  s.t = 0;
  return s;
}

// Symmetric P2P window layout (identical on every rank for a given n): per
// parity, K1's per-tile staging + tile counts + per-tile cut counts, the
// merge kernel's per-tile survivor chunks + counts + chunk prefix, and u.
struct WinLayout {
  size_t kstg[2], kcnt[2], klt[2], sidx[2], sval[2], scnt[2], spre[2], sbeg[2], uidx[2], uval[2], bytes;
};
WinLayout win_layout(size_t n, int max_chunks) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t kst = okt::stage_entries(n, okt::kK1Tile, max_chunks);
  // survivor chunks: one per K1 tile overlapping the region (capacity kK1Tile)
  const size_t sst = (n + 2 * size_t(okt::kK1Tile) - 1) / okt::kK1Tile * okt::kK1Tile + okt::kK1Tile;
  const size_t mc = size_t(max_chunks);
  const size_t kt = std::max(mc, (n + okt::kK1Tile - 1) / okt::kK1Tile);  // K1 counts are per tile
  WinLayout w;
  size_t o = al(sizeof(okt::P2PHdr));
  for (int p = 0; p < 2; ++p) {
    w.kstg[p] = o; o += al(8 * kst);
    w.kcnt[p] = o; o += al(4 * kt);
    w.klt[p] = o; o += al(4 * okt::kP2PMaxP * kt);
    w.sidx[p] = o; o += al(4 * sst);
    w.sval[p] = o; o += al(8 * sst);
    w.scnt[p] = o; o += al(4 * (kt + 2));  // one survivor chunk per K1 tile of the region
    w.spre[p] = o; o += al(8 * (kt + 3));
    w.sbeg[p] = o; o += al(4 * (kt + 2));  // first region tile of each survivor chunk
    w.uidx[p] = o; o += al(4 * n);
    w.uval[p] = o; o += al(8 * n);
  }
  w.bytes = o;
  return w;
}

// What every rank contributes to the P2P bootstrap allgather.
struct WinInfo {
  uint64_t pid;
  uint64_t base;
  cudaIpcMemHandle_t handle;
  unsigned char uuid[16];
  int32_t device;
  int32_t ok;
  uint64_t layout_bytes;  // peers compute offsets from their own layout: it must match
};

constexpr uint64_t kP2PTimeoutNs = 20ull * 1000 * 1000 * 1000;

}  // namespace

// =============================================================================
// okt_comm
// =============================================================================
struct okt_comm {
  int rank = 0, P = 1, device = 0;
  okt_world* world = nullptr;
  std::unique_ptr<okt::Transport> tr;
  cudaStream_t own = nullptr;
  cudaEvent_t ready_ev = nullptr;
  Launch L;
  okt_state st = default_state();
  bool dev_stale = true;  // device thresholds / cuts must be re-uploaded
  okt_counters ledger[OKT_PHASE_COUNT] = {};

  // buffers
  Buf coo;                 // local selection, AoS (u32 idx | f32 val << 32)
  Buf rbuf;                // split receive windows
  Buf mask, stage;         // region presence bytes / coordinate-major staging
  Buf reg_idx, reg_val;    // reduced region (refresh iterations)
  Buf sur_idx, sur_val;    // survivors of the global threshold
  Buf gval;                // gathered region values (refresh)
  Buf u_idx, u_val;        // allgathered result
  Buf sel_idx, sel_val;    // sub-phase outputs
  Buf tk_aux, tk_parts;    // baselines: chunk counts / offsets, gathered AoS parts
  Buf bl_ai, bl_av, bl_bi, bl_bv, bl_ci, bl_cv;  // baselines: SoA working lists
  Buf bl_ti, bl_tv;        // baselines: merge positions
  Buf bl_win, bl_win_in, bl_small;  // TopkDSA windows; small scratch
  Buf indexes;
  Buf eps[2];
  Buf hgrad;               // staging for the host-buffer entry points
  Buf galign;              // 16-byte aligned copy of a misaligned gradient (P2P step)
  Buf st64, stidx, stval;  // phase-A compaction staging
  Buf counts, counts2, chunkcap, tilectr;
  Buf agg;                 // phase-B look-back: per-CTA group totals
  uint32_t compact_tag = 0;  // phase-B launch tags (Stage::tag_ctr)
  Buf hist, scal;
  Buf shist;  // the cold refresh's sample histogram (2048 words)
  okt::Stage S;
  // device-driven multi-GPU exchange (okt_p2p.cuh)
  bool p2p_checked = false, p2p = false;
  Buf win, boot, tabd, selflags, trbuf;
  Buf ubits[2];  // EF P2P steps: u membership bitmaps by step parity (zero between uses)
  const float* cur_acc = nullptr;  // the step's accumulator / model (P2P fused apply)
  float* cur_w = nullptr;
  size_t win_n = 0;
  okt::PeerTab tab{};
  std::vector<void*> ipc_open;
  uint64_t p2p_epoch = 0;
  uint64_t bar_epoch = 0;  // okt_device_barrier calls (same count on every rank)
  // CUDA graph of the steady single-rank step (step block H2D, K1, fused
  // compaction + apply, scalar readback); per-step pointers are read from the
  // step block (DevScalars::sp) on the device.
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;     // kept: its kernel nodes hold the captured arguments
    cudaGraphNode_t k1 = nullptr, cb = nullptr;  // K1 and phase B, updated every step
    size_t n = 0, k = 0;
    bool sgd = false, prof = false;
    uint64_t gen = 0, kernels = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
  } graph1;
  uint64_t buf_gen = 1;
  DevScalars* h = nullptr;   // pinned download mirror
  okt::HostOut* hfast = nullptr;      // mapped pinned: the steady P = 1 step's scalars
  okt::HostOut* hfast_dev = nullptr;  // its device address
  uint64_t p1_seq = 0;
  okt::P2PHostOut* hp2p = nullptr;      // mapped pinned: the steady P2P EF step's results
  okt::P2PHostOut* hp2p_dev = nullptr;
  bool hp2p_pending = false;
  uint64_t hp2p_epoch = 0;
  bool hfast_pending = false;
  DevScalars* hup = nullptr; // pinned upload staging
  size_t cap_n = 0;
  int eps_cur = 0;
  size_t eps_n = 0;

  // profiling
  bool prof = false;
  bool graphs_on = std::getenv("OKT_DISABLE_GRAPHS") == nullptr;
  // Single-rank refresh candidates (OKT_REFRESH_CANDIDATES=0: the dense radix passes).
  bool cand_on = [] {
    const char* e = std::getenv("OKT_REFRESH_CANDIDATES");
    return !(e && e[0] == '0');
  }();
  bool refresh_dense_select = true;  // (bytes model) this refresh ran a select-only pass over all of acc
  // Cold refresh candidates from a sampled threshold, for n >= 2^25 (below
  // that its five small launches cost more than the select-only pass over acc
  // it saves: +21 us at n = 14.7M, -137 us at 340M); OKT_COLD_SAMPLE=0: never
  // (the pass-0 histogram's bin floor and a select-only pass over acc), =1: for every n.
  int cold_sample_mode = [] {
    const char* e = std::getenv("OKT_COLD_SAMPLE");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  bool cold_sample_for(uint64_t n) const {
    return cold_sample_mode > 0 || (cold_sample_mode < 0 && n >= (uint64_t(1) << 25));
  }
  // Sample geometry of a cold refresh: 1 coordinate in 2^s_log2 so that about
  // E = 1024..2048 samples lie at or above the k-th largest, and the sample
  // rank q = 1.25 E + 4 sqrt(E): the floor of q's bin then has >= k entries
  // above it in the whole vector unless the sample is off by ~8 standard
  // deviations (and then the step falls back to the dense passes).
  static bool sample_plan(uint64_t n, uint64_t k, uint32_t* s_log2, uint64_t* q) {
    if (k < 4096 || k >= n) return false;
    uint32_t s = 0;
    while (s < 10 && (k >> (s + 1)) >= 1024) ++s;
    const uint64_t m = (n + (uint64_t(1) << s) - 1) >> s;
    const double E = double(k) * double(m) / double(n);
    *s_log2 = s;
    *q = uint64_t(std::ceil(1.25 * E + 4.0 * std::sqrt(E)));
    return *q < m;
  }
  // Steady single-rank step: direct launches (default) or the captured graph (OKT_P1_GRAPH=1).
  bool p1_direct = [] {
    const char* e = std::getenv("OKT_P1_GRAPH");
    return !(e && e[0] == '1');
  }();
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Span { int id; cudaEvent_t a, b; };
  std::vector<Span> spans;
  int open_id = -1;
  cudaEvent_t open_ev = nullptr;
  double t_ms[OKT_T_COUNT] = {};
  uint64_t t_calls[OKT_T_COUNT] = {};
  double t_bytes[OKT_T_COUNT] = {};  // algorithmic HBM bytes per phase

  DevScalars* d() const { return scal.as<DevScalars>(); }
  cudaStream_t pick(void* s) const { return s ? static_cast<cudaStream_t>(s) : own; }

  // ---- ledger ---------------------------------------------------------------
  void credit_send(int ph, uint64_t words, uint64_t msgs, uint64_t bytes) {
    ledger[ph].words_sent += words;
    ledger[ph].msgs_sent += msgs;
    ledger[ph].bytes_sent += bytes;
  }
  void credit_recv(int ph, uint64_t words, uint64_t msgs, uint64_t bytes) {
    ledger[ph].words_recv += words;
    ledger[ph].msgs_recv += msgs;
    ledger[ph].bytes_recv += bytes;
  }
  // small_allreduce_avg of P+1 reals (transport.cpp:103-128): log2 P rounds.
  void credit_avg(uint64_t len, uint64_t bytes_moved) {
    okt::plan::ledger_avg(ledger[OKT_PHASE_CONSENSUS], P, len);
    ledger[OKT_PHASE_CONSENSUS].bytes_sent += bytes_moved * (P - 1);
    ledger[OKT_PHASE_CONSENSUS].bytes_recv += bytes_moved * (P - 1);
  }
  // small_allgather_u32 of one word (transport.cpp:130-160).
  void credit_allgather_u32() {
    okt::plan::ledger_allgather_u32(ledger[OKT_PHASE_CONSENSUS], P);
    ledger[OKT_PHASE_CONSENSUS].bytes_sent += 4ull * (P - 1);
    ledger[OKT_PHASE_CONSENSUS].bytes_recv += 4ull * (P - 1);
  }
  // sparse_allgatherv (collectives.cpp:30-77) over part sizes.
  void credit_allgatherv(int ph, const std::vector<uint64_t>& parts, uint64_t bytes_per_entry) {
    okt::plan::ledger_allgatherv(ledger[ph], rank, P, parts.data());
    uint64_t others = 0;
    for (int q = 0; q < P; ++q)
      if (q != rank) others += parts[q];
    ledger[ph].bytes_sent += parts[rank] * bytes_per_entry * (P - 1);
    ledger[ph].bytes_recv += others * bytes_per_entry;
  }

  // ---- profiling --------------------------------------------------------------
  cudaEvent_t ev_get() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  void tmark(int id, cudaStream_t s) {
    if (!prof) return;
    cudaEvent_t e = ev_get();
    cudaEventRecord(e, s);
    if (open_id >= 0) spans.push_back({open_id, open_ev, e});
    open_id = id;
    open_ev = e;
  }
  void tstop(cudaStream_t s) {
    if (!prof || open_id < 0) return;
    cudaEvent_t e = ev_get();
    cudaEventRecord(e, s);
    spans.push_back({open_id, open_ev, e});
    open_id = -1;
  }
  // Called after the stream was synchronised.
  void tcollect() {
    if (!prof) return;
    for (const Span& sp : spans) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, sp.a, sp.b) == cudaSuccess) {
        t_ms[sp.id] += ms;
        t_calls[sp.id] += 1;
      }
    }
    cudaGetLastError();
    spans.clear();
    ev_used = 0;
    open_id = -1;
    collect_k1();
  }

  // ---- capacity -----------------------------------------------------------------
  int reserve(size_t n) {
    if (n <= cap_n) return OKT_OK;
    cudaError_t e = cudaSuccess;
    const size_t k1_stage = okt::stage_entries(n, okt::kK1Tile, S.max_chunks);
    const size_t coo_stage = std::max({okt::stage_entries(n, okt::kCooTile, S.max_chunks), k1_stage,
                                       okt::stage_entries(n, okt::kRegionTileHost, S.max_chunks)});
    const size_t k1_tiles = (n + okt::kK1Tile - 1) / okt::kK1Tile;
    const size_t ncounts = std::max<size_t>(size_t(S.max_chunks), k1_tiles);
    if (e == cudaSuccess) e = counts.ensure(4 * ncounts);
    if (e == cudaSuccess) e = coo.ensure(8 * n);
    if (e == cudaSuccess) e = st64.ensure(8 * k1_stage);
    if (e == cudaSuccess) e = stidx.ensure(4 * coo_stage);
    if (e == cudaSuccess) e = stval.ensure(8 * coo_stage);
    agg.zero_init = true;
    if (e == cudaSuccess) e = agg.ensure(8 * (size_t(S.max_chunks) + k1_tiles / 256 + 2));
    if (e == cudaSuccess && P == 1) {
      // P = 1 runs without host syncs: survivors/indexes sized for the worst case.
      e = sur_idx.ensure(4 * n);
      if (e == cudaSuccess) e = sur_val.ensure(8 * n);
      if (e == cudaSuccess) e = indexes.ensure(4 * n);
    }
    S.counts = counts.as<uint32_t>();
    S.max_tiles = ncounts;
    S.s64 = st64.as<uint64_t>();
    S.sidx = stidx.as<uint32_t>();
    S.sval = stval.as<double>();
    S.agg = agg.as<uint64_t>();
    S.tag_ctr = &compact_tag;
    ++buf_gen;  // captured graphs hold these pointers
    if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, std::string("reserve: ") + cudaGetErrorString(e));
    cap_n = n;
    return OKT_OK;
  }
  int ensure(Buf& b, size_t bytes) {
    const cudaError_t e = b.ensure(bytes);
    if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return OKT_OK;
  }
  // Data-dependent capacities of the step (region, survivor, receive and
  // gather buffers, the region staging): the first allocation takes 2x
  // headroom, so the drift of the counts between refresh iterations does not
  // land a cudaFree / cudaMalloc pair (a device synchronisation) in a later step.
  int ensure_dd(Buf& b, size_t bytes) { return ensure(b, b.p ? bytes : 2 * bytes); }

  int sync(cudaStream_t s) {
    cudaMemcpyAsync(h, d(), sizeof(DevScalars), cudaMemcpyDeviceToHost, s);
    return wait_stream(s);
  }
  // Host wait on a stream that may hold collectives: bounded on the NCCL
  // transport (a dead peer -> TransportError after the deadline, never a hang).
  int wait_stream(cudaStream_t s) {
    std::string err;
    const int rc = tr ? tr->wait(s, err) : ck(cudaStreamSynchronize(s), "device");
    if (rc && tr) return comm_err(rc, err);
    return rc;
  }
  int ck(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return OKT_OK;
    cudaGetLastError();
    return set_err(OKT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }

  // Upload the host mirror's thresholds (and cuts) when the device copy is stale.
  int upload_state(cudaStream_t s) {
    if (!dev_stale) return OKT_OK;
    hup->local_th = st.local_th;
    hup->global_th = st.global_th;
    std::memcpy(hup->cuts, st.cuts, sizeof(st.cuts));
    int rc = ck(cudaMemcpyAsync(&d()->local_th, &hup->local_th, 2 * sizeof(double),
                                cudaMemcpyHostToDevice, s), "upload");
    if (rc) return rc;
    rc = ck(cudaMemcpyAsync(d()->cuts, hup->cuts, sizeof(hup->cuts), cudaMemcpyHostToDevice, s),
            "upload");
    if (rc) return rc;
    dev_stale = false;
    return OKT_OK;
  }
  int upload_u64(uint64_t* dst, uint64_t v, uint64_t* staging, cudaStream_t s) {
    *staging = v;
    return ck(cudaMemcpyAsync(dst, staging, 8, cudaMemcpyHostToDevice, s), "upload");
  }
  int upload_f64(double* dst, double v, double* staging, cudaStream_t s) {
    *staging = v;
    return ck(cudaMemcpyAsync(dst, staging, 8, cudaMemcpyHostToDevice, s), "upload");
  }

  int comm_err(int rc, const std::string& err) {
    if (rc == OKT_ERR_TRANSPORT) dead = true;  // a closed world / aborted communicator stays failed
    if (rc == OKT_ERR_TRANSPORT && world) return set_err(rc, "TransportError: " + err);
    return set_err(rc, err);
  }
  // Set by a transport failure (world closed, NCCL communicator aborted, a
  // peer that timed out): every later collective call fails at once with
  // TransportError, as calls on a closed InprocTransport do (inproc.cpp:54-61).
  bool dead = false;

  // ---- phases -----------------------------------------------------------------------
  // space_repartition from a selected index list (oktopk.cpp:28-61).  Cuts land
  // in d()->cuts; no host sync.
  int repartition_dev(const uint32_t* idx, int stride, const uint64_t* d_m, uint64_t m_host,
                      uint64_t n, cudaStream_t s) {
    int rc = ck(okt::launch_proposals(L, idx, stride, d_m, m_host, n, P, d()->prop), "proposals");
    if (rc) return rc;
    if (P > 1) {
      std::string err;
      rc = tr->allgather(d()->prop, d()->prop_all, sizeof(uint64_t) * (P + 1), s, err);
      if (rc) return comm_err(rc, err);
      credit_avg(uint64_t(P + 1), sizeof(uint64_t) * (P + 1));
      rc = ck(okt::launch_cuts(L, d()->prop_all, P, n, d()->cuts), "cuts");
    } else {
      rc = ck(cudaMemcpyAsync(d()->cuts, d()->prop, 2 * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s),
              "cuts");
    }
    return rc;
  }

  // split_and_reduce (oktopk.cpp:95-163) given the local selection in coo/d->m
  // and cuts in d->cuts.  Region (filter=false) or survivors of *d_gth
  // (filter=true) land in out_idx/out_val with count *d_out_cnt.  Host sync #1.
  // On return h->cnt_all / h->cuts are valid.
  int split_reduce_dev(uint64_t n, uint32_t bucket, bool filter, const double* d_gth, Buf& out_idx,
                       Buf& out_val, uint64_t* d_out_cnt, uint64_t& bound_out, cudaStream_t s) {
    int rc = ck(okt::launch_slice_offsets(L, coo.as<uint64_t>(), &d()->m, d()->cuts, P, d()->off,
                                          d()->cnt, &d()->flags),
                "slice_offsets");
    if (rc) return rc;
    std::string err;
    tmark(OKT_T_SPLIT, s);
    rc = tr->allgather(d()->cnt, d()->cnt_all, sizeof(uint32_t) * (P + 1), s, err);
    if (rc) return comm_err(rc, err);
    if ((rc = sync(s))) return rc;
    // Any rank with a non-finite accumulator aborts the step everywhere.
    for (int q = 0; q < P; ++q) {
      if (h->cnt_all[q * (P + 1) + P] & 1u) {
        if (q == rank) return set_err(OKT_ERR_NUMERIC, "ok_sparse_allreduce: non-finite input");
        return set_err(OKT_ERR_TRANSPORT, "TransportError: rank " + std::to_string(q) +
                                              " failed (non-finite input)");
      }
    }
    const uint64_t lo = h->cuts[rank], hi = h->cuts[rank + 1];
    const uint64_t W = hi > lo ? hi - lo : 0;
    std::vector<uint64_t> scnt(P), rcnt(P), roff(P + 1, 0);
    for (int q = 0; q < P; ++q) {
      scnt[q] = h->cnt_all[rank * (P + 1) + q];
      rcnt[q] = h->cnt_all[q * (P + 1) + rank];
    }
    // Ledger: rotated schedule dst = (r+s)%P, src = (r-s+P)%P (oktopk.cpp:113-157).
    uint64_t in_total = 0;
    {
      std::vector<uint64_t> counts(size_t(P) * P);
      for (int q = 0; q < P; ++q)
        for (int d2 = 0; d2 < P; ++d2) counts[size_t(q) * P + d2] = h->cnt_all[q * (P + 1) + d2];
      okt::plan::ledger_split(ledger[OKT_PHASE_SPLIT], rank, P, counts.data(), bucket);
      for (int q = 0; q < P; ++q)
        if (q != rank) {
          ledger[OKT_PHASE_SPLIT].bytes_sent += 8 * scnt[q];
          ledger[OKT_PHASE_SPLIT].bytes_recv += 8 * rcnt[q];
        }
    }
    for (int q = 0; q < P; ++q) {
      roff[q + 1] = roff[q] + (q == rank ? 0 : rcnt[q]);
      if (q != rank) in_total += rcnt[q];
    }
    if ((rc = ensure_dd(rbuf, 8 * std::max<uint64_t>(in_total, 1)))) return rc;
    std::vector<Xfer> sends, recvs;
    uint64_t* cooP = coo.as<uint64_t>();
    uint64_t* rb = rbuf.as<uint64_t>();
    for (int step = 1; step < P; ++step) {
      const int dst = (rank + step) % P, src = (rank - step + P) % P;
      sends.push_back({dst, cooP + h->off[dst], 8 * scnt[dst]});
      recvs.push_back({src, rb + roff[src], 8 * rcnt[src]});
    }
    rc = tr->exchange(sends, recvs, s, err);
    if (rc) return comm_err(rc, err);

    // K3: region merge.
    tmark(OKT_T_MERGE, s);
    const uint64_t bound = in_total + scnt[rank];
    if ((rc = ensure_dd(mask, ((W + 15) / 16) * 16 + 16))) return rc;
    if ((rc = ensure_dd(stage, 4 * std::max<uint64_t>(W, 1) * P))) return rc;
    if ((rc = ensure_dd(out_idx, 4 * std::max<uint64_t>(bound, 1)))) return rc;
    if ((rc = ensure_dd(out_val, 8 * std::max<uint64_t>(bound, 1)))) return rc;
    okt::Segs segs{};
    segs.nseg = 0;
    segs.start[0] = 0;
    for (int q = 0; q < P; ++q) {
      const uint64_t c = q == rank ? scnt[rank] : rcnt[q];
      segs.ptr[segs.nseg] = q == rank ? cooP + h->off[rank] : rb + roff[q];
      segs.src[segs.nseg] = q;
      segs.start[segs.nseg + 1] = segs.start[segs.nseg] + c;
      ++segs.nseg;
    }
    rc = ck(okt::launch_scatter(L, segs, lo, W, P, mask.as<uint32_t>(), stage.as<float>(), &d()->flags),
            "scatter");
    if (rc) return rc;
    rc = ck(okt::launch_region_scan(L, S, P, filter, lo, W, mask.as<uint32_t>(), stage.as<float>(), d_gth,
                                    out_idx.as<uint32_t>(), out_val.as<double>(), d_out_cnt),
            "region_scan");
    bound_out = bound;
    return rc;
  }

  // Global threshold refresh (oktopk.cpp:277-293): gather all regions, k-th
  // largest fp64 magnitude; unchanged when everything is empty.
  int refresh_global_dev(uint64_t k, uint64_t R_bound, cudaStream_t s) {
    (void)R_bound;
    int rc;
    std::string err;
    if (P == 1) {
      return ck(okt::launch_radix_select(L, okt::RadixSrc::kF64, reg_val.p, 0, &d()->R, R_bound, k,
                                         &d()->rs, hist.as<uint32_t>(), &d()->global_th, false),
                "radix");
    }
    rc = ck(cudaMemcpyAsync(&d()->small[0], &d()->R, 4, cudaMemcpyDeviceToDevice, s), "copy");
    if (rc) return rc;
    rc = tr->allgather(&d()->small[0], d()->small_all, 4, s, err);
    if (rc) return comm_err(rc, err);
    if ((rc = sync(s))) return rc;
    std::vector<uint64_t> parts(P), goff(P + 1, 0);
    for (int q = 0; q < P; ++q) {
      parts[q] = h->small_all[q];
      goff[q + 1] = goff[q] + parts[q];
    }
    const uint64_t total = goff[P];
    if ((rc = ensure_dd(gval, 8 * std::max<uint64_t>(total, 1)))) return rc;
    double* gv = gval.as<double>();
    if (parts[rank]) {
      rc = ck(cudaMemcpyAsync(gv + goff[rank], reg_val.p, 8 * parts[rank], cudaMemcpyDeviceToDevice, s),
              "copy");
      if (rc) return rc;
    }
    std::vector<Xfer> sends, recvs;
    for (int q = 0; q < P; ++q) {
      if (q == rank) continue;
      sends.push_back({q, reg_val.p, 8 * parts[rank]});
      recvs.push_back({q, gv + goff[q], 8 * parts[q]});
    }
    rc = tr->exchange(sends, recvs, s, err);
    if (rc) return comm_err(rc, err);
    credit_allgatherv(OKT_PHASE_GATHER, parts, 8);
    return ck(okt::launch_radix_select(L, okt::RadixSrc::kF64, gv, total, nullptr, total, k, &d()->rs,
                                       hist.as<uint32_t>(), &d()->global_th, false),
              "radix");
  }

  // balance_and_allgatherv (oktopk.cpp:165-244) on survivors already in
  // sur_idx/sur_val with count d->S.  u lands in u_idx/u_val; returns U.
  int balance_allgatherv_dev(cudaStream_t s, uint64_t& U) {
    int rc;
    std::string err;
    rc = ck(cudaMemcpyAsync(&d()->small[0], &d()->S, 4, cudaMemcpyDeviceToDevice, s), "copy");
    if (rc) return rc;
    rc = tr->allgather(&d()->small[0], d()->small_all, 4, s, err);
    if (rc) return comm_err(rc, err);
    if ((rc = sync(s))) return rc;
    credit_allgather_u32();
    std::vector<uint64_t> sizes(P);
    for (int q = 0; q < P; ++q) sizes[q] = h->small_all[q];
    const okt::plan::Balance B = okt::plan::balance(rank, P, sizes);
    const uint64_t total = B.total;
    U = total;
    if ((rc = ensure_dd(u_idx, 4 * std::max<uint64_t>(total, 1)))) return rc;
    if ((rc = ensure_dd(u_val, 8 * std::max<uint64_t>(total, 1)))) return rc;
    uint32_t* ui = u_idx.as<uint32_t>();
    double* uv = u_val.as<double>();
    const uint32_t* si = sur_idx.as<uint32_t>();
    const double* sv = sur_val.as<double>();
    const uint64_t mine = B.off[rank];
    // My own survivors (or the part of my block I hold) land straight at their
    // final position in u: the stream order is the result order.
    if (B.own.b > B.own.a) {
      const uint64_t a = B.own.a, b = B.own.b;
      rc = ck(cudaMemcpyAsync(ui + a, si + (a - mine), 4 * (b - a), cudaMemcpyDeviceToDevice, s), "copy");
      if (!rc) rc = ck(cudaMemcpyAsync(uv + a, sv + (a - mine), 8 * (b - a), cudaMemcpyDeviceToDevice, s), "copy");
      if (rc) return rc;
    }
    if (B.on) {
      std::vector<Xfer> sends, recvs;
      for (const okt::plan::Piece& p : B.sends) {
        sends.push_back({p.peer, const_cast<uint32_t*>(si) + (p.a - mine), 4 * (p.b - p.a)});
        sends.push_back({p.peer, const_cast<double*>(sv) + (p.a - mine), 8 * (p.b - p.a)});
        ledger[OKT_PHASE_BALANCE].bytes_sent += 12 * (p.b - p.a);
      }
      for (const okt::plan::Piece& p : B.recvs) {
        recvs.push_back({p.peer, ui + p.a, 4 * (p.b - p.a)});
        recvs.push_back({p.peer, uv + p.a, 8 * (p.b - p.a)});
        ledger[OKT_PHASE_BALANCE].bytes_recv += 12 * (p.b - p.a);
      }
      okt::plan::ledger_balance(ledger[OKT_PHASE_BALANCE], B);
      rc = tr->exchange(sends, recvs, s, err);
      if (rc) return comm_err(rc, err);
    }
    const std::vector<uint64_t>& part_off = B.part_off;
    const std::vector<uint64_t>& part_sz = B.part_sz;
    // allgatherv: every rank's part to every peer, straight into u.
    std::vector<Xfer> sends, recvs;
    for (int q = 0; q < P; ++q) {
      if (q == rank) continue;
      sends.push_back({q, ui + part_off[rank], 4 * part_sz[rank]});
      sends.push_back({q, uv + part_off[rank], 8 * part_sz[rank]});
      recvs.push_back({q, ui + part_off[q], 4 * part_sz[q]});
      recvs.push_back({q, uv + part_off[q], 8 * part_sz[q]});
    }
    rc = tr->exchange(sends, recvs, s, err);
    if (rc) return comm_err(rc, err);
    credit_allgatherv(OKT_PHASE_ALLGATHERV, part_sz, 12);
    return OKT_OK;
  }

  // ---- P2P window bootstrap (collective) ---------------------------------------------------
  int allgather_host(const void* mine, void* all, size_t bytes, cudaStream_t s) {
    int rc;
    if ((rc = ensure(boot, bytes * (P + 1)))) return rc;
    char* b = boot.as<char>();
    if ((rc = ck(cudaMemcpyAsync(b + bytes * P, mine, bytes, cudaMemcpyHostToDevice, s), "h2d"))) return rc;
    std::string err;
    rc = tr->allgather(b + bytes * P, b, bytes, s, err);
    if (rc) return comm_err(rc, err);
    if ((rc = ck(cudaMemcpyAsync(all, b, bytes * P, cudaMemcpyDeviceToHost, s), "d2h"))) return rc;
    return wait_stream(s);
  }

  void close_peers() {
    for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
    ipc_open.clear();
  }

  // Maps every peer's window when all ranks sit on distinct, peer-accessible
  // GPUs; otherwise the exchanges stay on the host-synchronised transport.
  // Collective: every rank calls it with the same n.
  int setup_p2p(size_t n, cudaStream_t s) {
    if (P == 1 || (p2p_checked && !p2p) || (p2p && win_n >= n)) return OKT_OK;
    if (std::getenv("OKT_DISABLE_P2P")) {
      p2p_checked = true;
      return OKT_OK;
    }
    int rc;
    int one = 1;
    std::vector<int> ones(P);
    close_peers();
    if ((rc = allgather_host(&one, ones.data(), sizeof(int), s))) return rc;  // peers closed my old window
    const WinLayout lay = win_layout(n, S.max_chunks);
    win.zero_init = false;
    if (win.p) {
      cudaFree(win.p);
      win.p = nullptr;
      win.cap = 0;
    }
    if ((rc = ensure(win, lay.bytes))) return rc;
    if ((rc = ck(cudaMemset(win.p, 0, sizeof(okt::P2PHdr)), "memset"))) return rc;
    WinInfo me{};
    me.pid = uint64_t(getpid());
    me.base = reinterpret_cast<uint64_t>(win.p);
    me.device = device;
    me.layout_bytes = lay.bytes;
    me.ok = cudaIpcGetMemHandle(&me.handle, win.p) == cudaSuccess;
    cudaGetLastError();
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) std::memcpy(me.uuid, prop.uuid.bytes, 16);
    std::vector<WinInfo> all(P);
    if ((rc = allgather_host(&me, all.data(), sizeof(WinInfo), s))) return rc;
    bool ok = me.ok != 0;
    std::vector<char*> base(P, nullptr);
    base[rank] = win.as<char>();
    // Test hook: OKT_P2P_ALLOW_SHARED=1 (with OKT_P2P_GRID_DIV >= the ranks per
    // GPU, so the ranks' spinning kernels fit side by side) runs the
    // device-driven path with several ranks of one process on one GPU.
    static const bool allow_shared = std::getenv("OKT_P2P_ALLOW_SHARED") != nullptr;
    for (int q = 0; q < P && ok; ++q) {
      if (q == rank) continue;
      const bool same_gpu = std::memcmp(all[q].uuid, me.uuid, 16) == 0;
      if (all[q].layout_bytes != me.layout_bytes) {
        ok = false;  // asymmetric windows (e.g. GPUs with different SM counts): host-synchronised path
        break;
      }
      if (!all[q].ok || (same_gpu && !(allow_shared && all[q].pid == me.pid))) {
        ok = false;  // a shared GPU: in-kernel cross-rank waits are not safe there
        break;
      }
      if (same_gpu) {
        base[q] = reinterpret_cast<char*>(all[q].base);
      } else if (all[q].pid == me.pid) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, device, all[q].device);
        if (!can) {
          ok = false;
          break;
        }
        const cudaError_t e = cudaDeviceEnablePeerAccess(all[q].device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ok = false;
        cudaGetLastError();
        base[q] = reinterpret_cast<char*>(all[q].base);
      } else {
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, all[q].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          ok = false;
          break;
        }
        ipc_open.push_back(ptr);
        base[q] = static_cast<char*>(ptr);
      }
    }
    int mine_ok = ok ? 1 : 0;
    std::vector<int> oks(P);
    if ((rc = allgather_host(&mine_ok, oks.data(), sizeof(int), s))) return rc;
    p2p_checked = true;
    p2p = true;
    for (int q = 0; q < P; ++q) p2p = p2p && oks[q];
    if (!p2p) {
      close_peers();
      return OKT_OK;
    }
    tab = okt::PeerTab{};
    tab.P = P;
    tab.rank = rank;
    for (int q = 0; q < P; ++q) {
      tab.hdr[q] = reinterpret_cast<okt::P2PHdr*>(base[q]);
      for (int p = 0; p < 2; ++p) {
        tab.kstg[q][p] = reinterpret_cast<uint64_t*>(base[q] + lay.kstg[p]);
        tab.kcnt[q][p] = reinterpret_cast<uint32_t*>(base[q] + lay.kcnt[p]);
        tab.klt[q][p] = reinterpret_cast<uint32_t*>(base[q] + lay.klt[p]);
        tab.sidx[q][p] = reinterpret_cast<uint32_t*>(base[q] + lay.sidx[p]);
        tab.sval[q][p] = reinterpret_cast<double*>(base[q] + lay.sval[p]);
        tab.scnt[q][p] = reinterpret_cast<uint32_t*>(base[q] + lay.scnt[p]);
        tab.spre[q][p] = reinterpret_cast<uint64_t*>(base[q] + lay.spre[p]);
        tab.sbeg[q][p] = reinterpret_cast<uint32_t*>(base[q] + lay.sbeg[p]);
        tab.u_idx[q][p] = reinterpret_cast<uint32_t*>(base[q] + lay.uidx[p]);
        tab.u_val[q][p] = reinterpret_cast<double*>(base[q] + lay.uval[p]);
      }
    }
    tab.trace = trbuf.as<uint64_t>();  // (null unless OKT_P2P_TRACE)
    if ((rc = ensure(tabd, sizeof(okt::PeerTab)))) return rc;
    if ((rc = ck(cudaMemcpy(tabd.p, &tab, sizeof(okt::PeerTab), cudaMemcpyHostToDevice), "tab"))) return rc;
    if ((rc = ensure(indexes, 4 * std::max<size_t>(n, 1)))) return rc;
    if ((rc = ensure(selflags, std::max<size_t>(n, 1)))) return rc;
    for (Buf& b : ubits) {
      b.zero_init = true;
      if (b.p && b.cap < 4 * ((n + 127) / 128 * 4)) {
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
      }
      if ((rc = ensure(b, 4 * ((n + 127) / 128 * 4)))) return rc;  // (whole uint4 words)
    }
    win_n = n;
    return OKT_OK;
  }

  // Argument-fed EF steps (OKT_P2P_ARGFED=0: the H2D step block instead; diagnostics).
  const bool argfed_on = [] {
    const char* e = std::getenv("OKT_P2P_ARGFED");
    return !(e && e[0] == '0');
  }();
  // K1's P2P arguments for this step (hup->sp holds the step block).
  okt::K1P2P k1p2p_args(bool argfed) {
    okt::K1P2P kp;
    kp.tab = tabd.as<okt::PeerTab>();
    kp.sp = &d()->sp;
    kp.cuts = d()->cuts;
    if (argfed) {
      kp.par_v = hup->sp.par;
      kp.sp_out = &d()->sp;
      kp.plan_zero = &d()->plan;
      kp.spv = hup->sp;
    }
    kp.tot_acc = d()->k1_tot;
    kp.d_off = d()->off;
    kp.d_m = &d()->m;
    return kp;
  }

  // Enqueues a whole steady P2P iteration on `s` (no host synchronisation):
  // step block refresh, flag reset, K1 (+ slice offsets + L publication),
  // fused split/scatter, bracket scan (+ survivor publication), allgatherv
  // pull with the fused apply, indexes, scalar readback.  Per-step values
  // (pointers, epoch, parity) are read from the step block on the device, so the same
  // sequence is captured once into a CUDA graph.
  int enqueue_p2p_step(size_t n, size_t k, bool sgd, cudaStream_t s) {
    const okt::StepPtrs* sp = &d()->sp;
    okt::P2PPlan* dp = &d()->plan;
    const okt::PeerTab* dt = tabd.as<okt::PeerTab>();
    const uint64_t lo = st.cuts[rank], hi = st.cuts[rank + 1];
    const uint64_t W = hi > lo ? hi - lo : 0;
    (void)k;
    // EF steps are argument-fed: the step block rides in K1's arguments (K1's
    // CTA 0 stores it and clears the plan; the flag word alternates by parity
    // and the pull clears the next one), so the step starts with K1 — no H2D
    // node.  The plain allreduce keeps one H2D of the step block, zeroed flags
    // and a zeroed plan.
    const bool argfed = sgd && argfed_on;
    const int par = hup->sp.par;
    uint32_t* fl = argfed ? &d()->p2pflags[par] : &d()->flags;
    int rc = OKT_OK;
    if (!argfed) {
      const size_t blk = offsetof(DevScalars, plan) + sizeof(okt::P2PPlan) - offsetof(DevScalars, sp);
      rc = ck(cudaMemcpyAsync(&d()->sp, &hup->sp, blk, cudaMemcpyHostToDevice, s), "h2d");
    }
    tmark(OKT_T_SELECT, s);
    okt::K1P2P kp = k1p2p_args(argfed);
    kp.zero_sel = sgd ? 1 : 0;
    kp.hout = sgd ? hp2p_dev : nullptr;  // (K1's last CTA: selection size and slice offsets)
    if (!rc)
      rc = ck(okt::launch_k1(L, S, sgd ? okt::K1Mode::kAccumSelect : okt::K1Mode::kSelect, hup->sp.g,
                             hup->sp.eps_in, hup->sp.eps_out, hup->sp.alpha, n, &d()->local_th, nullptr,
                             okt::OutCoo{}, &d()->m, nullptr, fl, nullptr, nullptr, &kp, argfed ? nullptr : sp),
              "k1");
    // (K1's totals — selection size, slice offsets — come from K1's last CTA:
    // a side-stream kernel for them held SMs the merge's CTAs then waited for)
    tmark(OKT_T_MERGE, s);
    // split exchange + region merge in one kernel (reads every source's K1
    // tiles of my region in place)
    if (!rc) rc = ck(okt::launch_p2p_merge(L, dt, sp, dp, P, lo, W, n, &d()->global_th, fl, kP2PTimeoutNs,
                                                  d()->merge_ctr), "p2p");
    tmark(OKT_T_ALLGATHER, s);
    okt::P2PApply pa;
    pa.on = 1;
    pa.flags2 = argfed ? d()->p2pflags : nullptr;
    pa.sgd = sgd ? 1 : 0;
    pa.d_local_th = &d()->local_th;
    // oktopk_sgd_step reports no index list (trainer.hpp:123-127): only the
    // plain allreduce needs the sel flags and the indexes compaction.
    pa.sel = sgd ? nullptr : selflags.as<uint8_t>();
    if (sgd) {
      pa.ubits[0] = ubits[0].as<uint32_t>();
      pa.ubits[1] = ubits[1].as<uint32_t>();
    }
    if (!rc) rc = ck(okt::launch_p2p_allgatherv(L, dt, sp, &d()->S, dp, &d()->U, fl, kP2PTimeoutNs, pa,
                                                sgd ? hp2p_dev : nullptr, S.tile_ctr + 4),
                     "p2p");
    if (sgd) {
      tmark(OKT_T_APPLY, s);
      if (!rc) rc = ck(okt::launch_p2p_restore(L, dt, sp, ubits[0].as<uint32_t>(), ubits[1].as<uint32_t>(), n,
                                               argfed ? d()->p2pflags : nullptr, fl), "restore");
    } else {
      tmark(OKT_T_APPLY, s);
      if (!rc) rc = ck(okt::launch_select_flags(L, S, selflags.as<uint8_t>(), dt, sp, &d()->U, win_n,
                                                indexes.as<uint32_t>(), &d()->nidx, &d()->flags), "indexes");
    }
    tstop(s);
    // EF steps hand their results back through mapped host memory (hp2p); the
    // plain allreduce (indexes, ...) reads the scalars back with one D2H
    if (!rc && !sgd) rc = ck(cudaMemcpyAsync(h, d(), sizeof(DevScalars), cudaMemcpyDeviceToHost, s), "d2h");
    return rc;
  }

  struct P2PGraph {
    cudaGraphExec_t exec = nullptr;
    size_t n = 0, k = 0;
    bool sgd = false;
    uint64_t lo = 0, W = 0, gen = 0, win = 0, kernels = 0;
    cudaGraph_t graph = nullptr;  // kept: its kernel nodes are patched per launch (argument-fed steps)
    cudaGraphNode_t k1 = nullptr, merge = nullptr, pull = nullptr;
  } graph2;

  // The steady P2P iteration through one graph launch (captured on first use
  // and whenever the buffers or the owned region change).
  int launch_p2p_step(size_t n, size_t k, bool sgd, cudaStream_t s) {
    int rc;
    const uint64_t lo = st.cuts[rank], hi = st.cuts[rank + 1];
    const uint64_t W = hi > lo ? hi - lo : 0;
    if ((rc = ensure_dd(mask, ((W + 15) / 16) * 16 + 16)) || (rc = ensure_dd(stage, 4 * std::max<uint64_t>(W, 1) * P)))
      return rc;
    if (prof || !graphs_on) return enqueue_p2p_step(n, k, sgd, s);
    P2PGraph& G = graph2;
    const uint64_t gen = buf_gen + reinterpret_cast<uintptr_t>(mask.p) + reinterpret_cast<uintptr_t>(stage.p);
    if (!G.exec || G.n != n || G.k != k || G.sgd != sgd || G.lo != lo || G.W != W || G.gen != gen || G.win != win_n) {
      if (G.exec) {
        cudaGraphExecDestroy(G.exec);
        G.exec = nullptr;
      }
      const uint64_t l0 = L.launches;
      if ((rc = ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture"))) return rc;
      rc = enqueue_p2p_step(n, k, sgd, s);
      cudaGraph_t graph = nullptr;
      const cudaError_t e2 = cudaStreamEndCapture(s, &graph);
      if (rc || e2 != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return rc ? rc : ck(e2, "graph capture");
      }
      G.k1 = G.merge = G.pull = nullptr;
      if (sgd && argfed_on) {  // the nodes whose arguments change per step (K1: the kernel that is none of the others)
        size_t nn = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(graph, nodes.data(), &nn);
        const void* fm = okt::p2p_merge_func(P);
        const void* fp = okt::p2p_pull_func();
        const void* fr = okt::p2p_restore_func();
        for (cudaGraphNode_t nd : nodes) {
          cudaGraphNodeType ty;
          cudaGraphNodeGetType(nd, &ty);
          if (ty != cudaGraphNodeTypeKernel) continue;
          cudaKernelNodeParams kp{};
          cudaGraphKernelNodeGetParams(nd, &kp);
          if (kp.func == fm) G.merge = nd;
          else if (kp.func == fp) G.pull = nd;
          else if (kp.func != fr) G.k1 = nd;
        }
      }
      const cudaError_t e = cudaGraphInstantiate(&G.exec, graph, 0);
      if (sgd && argfed_on && (!G.k1 || !G.merge || !G.pull)) {
        if (e == cudaSuccess) cudaGraphExecDestroy(G.exec);
        G.exec = nullptr;
        cudaGraphDestroy(graph);
        return set_err(OKT_ERR_INTERNAL, "P2P step graph: kernel nodes not found");
      }
      // (the node handles stay valid for exec updates while the graph lives)
      if (G.graph) cudaGraphDestroy(G.graph);
      G.graph = graph;
      if ((rc = ck(e, "graph instantiate"))) return rc;
      G.kernels = L.launches - l0;
      L.launches = l0;
      G.n = n;
      G.k = k;
      G.sgd = sgd;
      G.lo = lo;
      G.W = W;
      G.gen = gen;
      G.win = win_n;
    } else if (sgd && argfed_on) {
      // this step's arguments into the instantiated nodes: K1 (g, eps_in,
      // eps_out, alpha, the flag word, K1P2P = arguments 0-3, 12, 15 of 17),
      // the merge's and the pull's flag word (arguments 7 and 5)
      uint32_t* fl = &d()->p2pflags[hup->sp.par];
      okt::K1P2P kp = k1p2p_args(true);
      kp.zero_sel = 1;
      kp.hout = hp2p_dev;
      if ((rc = patch_node(G.exec, G.k1, kK1Args, {{0, &hup->sp.g}, {1, &hup->sp.eps_in}, {2, &hup->sp.eps_out},
                                              {3, &hup->sp.alpha}, {12, &fl}, {15, &kp}})) ||
          (rc = patch_node(G.exec, G.merge, 11, {{7, &fl}})) || (rc = patch_node(G.exec, G.pull, 10, {{5, &fl}})))
        return rc;
    }
    if ((rc = ck(cudaGraphLaunch(G.exec, s), "graph launch"))) return rc;
    L.launches += G.kernels;
    return OKT_OK;
  }

  // Rewrites some arguments of an instantiated kernel node (index -> value).
  // Kernel parameter counts of the patched nodes (okt_kernels.cu: k1_kernel,
  // compact_kernel; okt_p2p.cu: p2p_merge_kernel, p2p_pull_kernel).
  static constexpr int kK1Args = 17, kCompactArgs = 16;
  int patch_node(cudaGraphExec_t exec, cudaGraphNode_t nd, int nargs,
                 std::initializer_list<std::pair<int, void*>> args) {
    cudaKernelNodeParams kp{};
    int rc = ck(cudaGraphKernelNodeGetParams(nd, &kp), "graph params");
    if (rc) return rc;
    void* a[24];
    for (int i = 0; i < nargs && i < 24; ++i) a[i] = kp.kernelParams[i];
    for (const auto& x : args) a[x.first] = x.second;
    kp.kernelParams = a;
    return ck(cudaGraphExecKernelNodeSetParams(exec, nd, &kp), "graph params");
  }

  // Ledger of a P2P step, from the sizes every rank agreed on (h valid).
  void p2p_credit() {
    std::vector<uint64_t> counts(size_t(P) * P, 0);
    for (int q = 0; q < P; ++q) {
      counts[size_t(rank) * P + q] = h->off[q + 1] - h->off[q];
      counts[size_t(q) * P + rank] = h->plan.seg_cnt[q];
    }
    okt::plan::ledger_split(ledger[OKT_PHASE_SPLIT], rank, P, counts.data(), st.bucket_size);
    for (int q = 0; q < P; ++q)
      if (q != rank) {
        ledger[OKT_PHASE_SPLIT].bytes_sent += 8 * counts[size_t(rank) * P + q];
        ledger[OKT_PHASE_SPLIT].bytes_recv += 8 * h->plan.seg_cnt[q];
      }
    credit_allgather_u32();
    const std::vector<uint64_t> sizes(h->plan.sizes, h->plan.sizes + P);
    const okt::plan::Balance B = okt::plan::balance(rank, P, sizes);
    if (B.on) {
      okt::plan::ledger_balance(ledger[OKT_PHASE_BALANCE], B);
      for (const auto& p : B.sends) ledger[OKT_PHASE_BALANCE].bytes_sent += 12 * (p.b - p.a);
      for (const auto& p : B.recvs) ledger[OKT_PHASE_BALANCE].bytes_recv += 12 * (p.b - p.a);
    }
    credit_allgatherv(OKT_PHASE_ALLGATHERV, B.part_sz, 12);
  }

  // Steady single-rank step through one CUDA graph launch.  Returns with the
  // stream synchronised and h valid.
  int run_graph_p1(const float* g, const float* eps_in, float* eps_out, float* w, float alpha, size_t n, size_t k,
                   bool sgd, cudaStream_t s) {
    int rc;
    StepGraph& G = graph1;
    // The step's pointers, α and flag word are kernel arguments, rewritten in
    // the instantiated graph every step (no H2D node); the flag word
    // alternates by step parity and phase B clears the next one.
    const uint64_t seq = ++p1_seq;
    uint32_t* fl = &d()->pflags[seq & 1];
    uint32_t* fl_next = &d()->pflags[(seq + 1) & 1];
    okt::ApplyArgs ap;
    ap.k7 = sgd;
    ap.acc = sgd ? eps_out : nullptr;
    ap.w = sgd ? w : nullptr;
    ap.d_flags = fl;
    ap.hout = hfast_dev;
    ap.seq = seq;
    ap.d_flags_next = fl_next;
    ap.trace = trbuf.as<uint64_t>();
    ap.tag = ++compact_tag;  // (patched into the graph every step: a fresh tag per launch)
    if (ap.tag < 2) ap.tag = compact_tag = 2;
    hfast->bad_iter = 0;
    if (p1_direct) {
      // The same two kernels launched directly, arguments and all (no graph):
      // at n = 340M cudaGraphLaunch of the parameter-patched graph took 34 us
      // of host time (+ 2 x 8 us patching) while the GPU waited (CUPTI trace,
      // round 2); two cudaLaunchKernel calls take a few us and the second one
      // is queued while K1 runs.
      tmark(OKT_T_SELECT, s);
      rc = ck(okt::launch_k1(L, S, sgd ? okt::K1Mode::kAccumSelect : okt::K1Mode::kSelect, g, eps_in, eps_out, alpha,
                             n, &d()->local_th, &d()->global_th,
                             okt::OutCoo{nullptr, sur_idx.as<uint32_t>(), sur_val.as<double>()}, &d()->S, &d()->m, fl,
                             nullptr, &ap, nullptr, nullptr),
              "k1");
      tstop(s);
      if (rc) return rc;
    } else if (!G.exec || G.n != n || G.k != k || G.sgd != sgd || G.gen != buf_gen || G.prof != prof) {
      if (G.exec) {
        cudaGraphExecDestroy(G.exec);
        G.exec = nullptr;
      }
      if (G.graph) {
        cudaGraphDestroy(G.graph);
        G.graph = nullptr;
      }
      if (!G.e0) {
        cudaEventCreate(&G.e0);
        cudaEventCreate(&G.e1);
      }
      const uint64_t l0 = L.launches;
      if ((rc = ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture"))) return rc;
      if (prof) cudaEventRecordWithFlags(G.e0, s, cudaEventRecordExternal);
      cudaError_t e = okt::launch_k1(L, S, sgd ? okt::K1Mode::kAccumSelect : okt::K1Mode::kSelect, g, eps_in,
                                     eps_out, alpha, n, &d()->local_th, &d()->global_th,
                                     okt::OutCoo{nullptr, sur_idx.as<uint32_t>(), sur_val.as<double>()}, &d()->S,
                                     &d()->m, fl, nullptr, &ap, nullptr, nullptr);
      if (prof) cudaEventRecordWithFlags(G.e1, s, cudaEventRecordExternal);
      // (no D2H node: phase B's CTA 0 writes m, S and the flags to hfast)
      const cudaError_t e2 = cudaStreamEndCapture(s, &G.graph);
      if (e != cudaSuccess || e2 != cudaSuccess) {
        if (G.graph) cudaGraphDestroy(G.graph);
        G.graph = nullptr;
        return ck(e != cudaSuccess ? e : e2, "graph capture");
      }
      // the two kernel nodes: phase B by its function, K1 the other one
      size_t nn = 0;
      cudaGraphGetNodes(G.graph, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      cudaGraphGetNodes(G.graph, nodes.data(), &nn);
      G.k1 = G.cb = nullptr;
      const void* cfunc = okt::compact_graph_kernel(sgd);
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType ty;
        cudaGraphNodeGetType(nd, &ty);
        if (ty != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp{};
        cudaGraphKernelNodeGetParams(nd, &kp);
        (kp.func == cfunc ? G.cb : G.k1) = nd;
      }
      if (!G.k1 || !G.cb) return set_err(OKT_ERR_INTERNAL, "single-rank graph: kernel nodes not found");
      e = cudaGraphInstantiate(&G.exec, G.graph, 0);
      if ((rc = ck(e, "graph instantiate"))) return rc;
      G.kernels = L.launches - l0;
      L.launches = l0;
      graph1_k1_pairs = k1_used / 2;
      k1_used = 0;
      G.n = n;
      G.k = k;
      G.sgd = sgd;
      G.gen = buf_gen;
      G.prof = prof;
    } else {
      // this step's arguments into the instantiated nodes: K1 (g, eps_in,
      // eps_out, alpha, d_flags = arguments 0-3 and 12) and phase B
      // (ApplyArgs = argument 15: model pointer, flag words, tag)
      if ((rc = patch_node(G.exec, G.k1, kK1Args, {{0, &g}, {1, &eps_in}, {2, &eps_out}, {3, &alpha}, {12, &fl}})) ||
          (rc = patch_node(G.exec, G.cb, kCompactArgs, {{15, &ap}})))
        return rc;
    }
    if (!p1_direct) {
      if ((rc = ck(cudaGraphLaunch(G.exec, s), "graph launch"))) return rc;
      L.launches += G.kernels;
      if (prof) k1_used = 2 * graph1_k1_pairs;  // the graph re-recorded its K1 events
      graph_prof_pending = prof;
    }
    if (defer) {
      hfast_pending = true;  // read by wait_pending after its sync
      return OKT_OK;
    }
    if ((rc = ck(cudaStreamSynchronize(s), "device"))) return rc;
    if ((rc = read_hfast())) return rc;
    collect_graph_prof();
    return OKT_OK;
  }
  // The scalars a steady single-rank graph step hands back through mapped
  // host memory (into the DevScalars mirror, where commit_step reads them).
  // The results of a steady device-driven EF step, written by its kernels into
  // mapped host memory (into the DevScalars mirror, where commit_step reads them).
  int read_hp2p() {
    if (!hp2p_pending) return OKT_OK;
    hp2p_pending = false;
    const volatile okt::P2PHostOut* o = hp2p;
    if (o->seq_pull != hp2p_epoch || o->seq_tot != hp2p_epoch)
      return set_err(OKT_ERR_INTERNAL, "device-driven step: no results from the device");
    h->m = o->m;
    h->U = o->U;
    for (int q = 0; q <= P; ++q) h->off[q] = o->off[q];
    for (int q = 0; q < P; ++q) {
      h->plan.sizes[q] = o->sizes[q];
      h->plan.seg_cnt[q] = o->seg_cnt[q];
    }
    h->flags = o->flags_early | (o->err_timeout ? 8u : 0u) | (o->err_peer ? 16u : 0u) | (o->err_iter ? 4u : 0u);
    return OKT_OK;
  }
  int read_hfast() {
    const volatile okt::HostOut* o = hfast;
    if (o->seq != p1_seq) return set_err(OKT_ERR_INTERNAL, "single-rank step: no scalars from the device");
    h->m = o->m;
    h->S = o->S;
    h->flags = o->flags | (o->bad_iter ? 4u : 0u);  // (bits 0 and 2: all a single-rank step sets)
    return OKT_OK;
  }
  bool graph_prof_pending = false;
  // K1 phase-A event pairs (profiling); the graph's pairs are reused per launch.
  std::vector<cudaEvent_t> k1_pool;
  size_t k1_used = 0;
  static cudaEvent_t k1_event_cb(void* ctx) {
    okt_comm* c = static_cast<okt_comm*>(ctx);
    if (c->k1_used == c->k1_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->k1_pool.push_back(e);
    }
    return c->k1_pool[c->k1_used++];
  }
  void collect_k1() {
    for (size_t i = 0; i + 1 < k1_used; i += 2) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, k1_pool[i], k1_pool[i + 1]) == cudaSuccess) {
        t_ms[OKT_T_K1] += ms;
        t_calls[OKT_T_K1] += 1;
      }
    }
    cudaGetLastError();
    k1_used = 0;
  }
  size_t graph1_k1_pairs = 0;  // events [0, 2*pairs) belong to the captured graph
  void collect_graph_prof() {
    if (!graph_prof_pending) return;
    graph_prof_pending = false;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, graph1.e0, graph1.e1) == cudaSuccess) {
      t_ms[OKT_T_SELECT] += ms;
      t_calls[OKT_T_SELECT] += 1;
    }
    cudaGetLastError();
  }

  // ---- the step ---------------------------------------------------------------------
  int step(const float* g, float* w, size_t n, double alpha, int64_t t, size_t k, bool sgd,
           okt_result* out, cudaStream_t s) {
    if (pending.on) {
      const int prc = wait_pending(nullptr);
      if (prc) return prc;
    }
    if (n == 0 || k < 1 || t < 1)
      return set_err(OKT_ERR_INVALID_ARGUMENT, "ok_sparse_allreduce: empty input, k < 1, or t < 1");
    if (dead && P > 1) return set_err(OKT_ERR_TRANSPORT, "TransportError: the transport failed earlier (peer lost)");
    if (n > 0xffffffffull) return set_err(OKT_ERR_INVALID_ARGUMENT, "n exceeds the u32 index space");
    if (st.tau == 0 || st.tau_prime == 0)
      return set_err(OKT_ERR_INVALID_ARGUMENT, "tau and tau_prime must be >= 1");
    if (!g) return set_err(OKT_ERR_INVALID_ARGUMENT, "null gradient");
    int rc;
    if ((rc = reserve(n))) return rc;
    if (sgd) {
      if (eps_n == 0) {
        if ((rc = residual_reset(n, nullptr, s))) return rc;
      } else if (eps_n != n) {
        return set_err(OKT_ERR_INVALID_ARGUMENT, "oktopk_sgd_step: residual size does not match problem");
      }
    }
    L.s = s;
    cudaEvent_t step_begin = nullptr;
    if (prof) {
      step_begin = ev_get();
      cudaEventRecord(step_begin, s);
    }
    if ((rc = upload_state(s))) return rc;
    const bool thr = (t - 1) % int64_t(st.tau_prime) == 0;
    const bool bnd = (t - 1) % int64_t(st.tau) == 0;
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    const bool use_graph = P == 1 && !thr && (p1_direct || (graphs_on && al16(g) && (!sgd || al16(w))));
    if (P > 1 && (rc = setup_p2p(n, s))) return rc;
    // The path choice must be the same on every rank, so it may not depend on
    // rank-local pointer alignment: a gradient that is not 16-byte aligned
    // (the vectorised K1 of the device-driven step needs it) is staged into an
    // aligned buffer first.  (The model is only scattered: any alignment.)
    if (P > 1 && p2p && !al16(g)) {
      if ((rc = ensure(galign, 4 * n))) return rc;
      if ((rc = ck(cudaMemcpyAsync(galign.p, g, 4 * n, cudaMemcpyDeviceToDevice, s), "stage"))) return rc;
      g = galign.as<float>();
    }
    // Steady iterations on distinct GPUs run the device-driven exchange; the
    // refresh iterations (1 in tau') keep the host-synchronised protocol.
    const bool use_p2p = p2p && !thr && !bnd && st.regions == P;
    if (!use_graph && !use_p2p && (rc = ck(cudaMemsetAsync(&d()->flags, 0, 4, s), "memset"))) return rc;
    uint64_t epoch = 0;
    int par = 0;
    if (use_p2p) {
      epoch = ++p2p_epoch;
      par = int(epoch & 1);
    }
    const float* acc = g;
    const float* eps_in = nullptr;
    float* eps_out = nullptr;
    if (sgd) {
      eps_in = eps[eps_cur].as<float>();
      eps_out = eps[eps_cur ^ 1].as<float>();
      acc = eps_out;
    }
    uint32_t* hp = hist.as<uint32_t>();
    const float fa = float(alpha);
    if (use_graph) {
      if ((rc = run_graph_p1(g, eps_in, eps_out, w, fa, n, k, sgd, s))) return abort_step(rc);
      if (prof) {
        cudaEvent_t e = ev_get();
        cudaEventRecord(e, s);
        spans.push_back({OKT_T_STEP, step_begin, e});
      }
      if (defer_commit(n, t, thr, sgd, std::vector<uint64_t>{0, uint64_t(n)}, sur_idx.as<uint32_t>(),
                       sur_val.as<double>(), s))
        return OKT_OK;
      cudaStreamSynchronize(s);
      tcollect();
      return commit_step(n, t, thr, sgd, std::vector<uint64_t>{0, uint64_t(n)}, sur_idx.as<uint32_t>(),
                         sur_val.as<double>(), out);
    }
    if (use_p2p) {
      okt::StepPtrs& sp = hup->sp;
      sp.g = g;
      sp.eps_in = eps_in;
      sp.eps_out = eps_out;
      sp.w = sgd ? w : nullptr;
      sp.alpha = fa;
      sp.epoch = epoch;
      sp.par = par;
      if (sgd) {  // the kernels set these on an error (the step's results come through hp2p)
        hp2p->err_timeout = hp2p->err_peer = hp2p->err_iter = 0;
        hp2p_pending = true;
        hp2p_epoch = epoch;
      }
      if ((rc = launch_p2p_step(n, k, sgd, s))) return abort_step(rc);
      if (prof) {
        cudaEvent_t e = ev_get();
        cudaEventRecord(e, s);
        spans.push_back({OKT_T_STEP, step_begin, e});
      }
      const std::vector<uint64_t> cuts(st.cuts, st.cuts + P + 1);
      p2p_credit_pending = true;
      if (defer_commit(n, t, thr, sgd, cuts, tab.u_idx[rank][par], tab.u_val[rank][par], s)) return OKT_OK;
      if ((rc = ck(cudaStreamSynchronize(s), "device"))) return abort_step(rc);
      if ((rc = read_hp2p())) return abort_step(rc);
      tcollect();
      return commit_step(n, t, thr, sgd, cuts, tab.u_idx[rank][par], tab.u_val[rank][par], out);
    }
    // P = 1: u is a subset of the local selection, so K7 (w -= u, eps = 0 at u)
    // is fused into the compaction that writes u, and indexes = u.indices.
    okt::ApplyArgs ap1;
    if (sgd && P == 1) {  // K7 fused: residual zero in K1, model update in phase B
      ap1.k7 = true;
      ap1.acc = eps_out;
      ap1.w = w;
      ap1.d_flags = &d()->flags;
    }

    // ---- K1 / K2 ----
    if (thr) {
      bool sel_done = false;  // the refresh-candidate path produced u already
      if (sgd) {
        tmark(OKT_T_SELECT, s);
        rc = ck(okt::launch_radix_init(L, &d()->rs, k, n, nullptr), "radix_init");
        // Refresh candidates: thresholds drift slowly between refreshes, so a
        // warm refresh's K1 accumulate pass also emits every entry with
        // |acc| >= local_th_old / 2.  When at least k entries qualify, the
        // k-th largest is among them: the exact radix select, the local
        // selection / survivor selection and K7 then run over the candidates,
        // instead of two more radix passes and a second select pass over all n
        // (at n = 340M: 0.39 + 0.43 ms).  Otherwise the dense passes run as
        // before (pass 0's histogram came out of the same K1 pass).
        // Cold refresh (no previous threshold): pass 0's histogram picks the
        // top-11-bit bin holding the k-th largest, and a select-only K1 pass
        // over acc emits everything at or above that bin as the candidates —
        // instead of two more radix passes and a second select pass.
        // Cold refresh with a large k: the candidate threshold from a strided
        // sample of acc (a few MB read) instead of pass 0 over all of acc
        // followed by a second, select-only pass over it (0.40 ms at 340M); the
        // accumulate pass then emits the candidates as in a warm refresh.
        const bool warm = cand_on && st.local_th > 0.0 && std::isfinite(st.local_th);
        uint32_t s_log2 = 0;
        uint64_t s_q = 0;
        const bool sampled = !warm && cand_on && cold_sample_for(n) && sample_plan(n, k, &s_log2, &s_q);
        bool have_cand = false;  // candidates in coo (AoS) with count d()->R, at least k of them
        uint64_t C_bound = n;    // (grid sizing of the candidate kernels)
        refresh_dense_select = !(warm || sampled);
        if (warm || sampled) {
          if (warm) {
            if (!rc) rc = upload_f64(&d()->th_arg, 0.5 * st.local_th, &hup->th_arg, s);
          } else if (!rc) {
            rc = ck(okt::launch_sample_floor(L, g, eps_in, fa, n, s_log2, s_q, &d()->rs_sample, shist.as<uint32_t>(),
                                             &d()->th_arg), "sample");
          }
          if (!rc) rc = ck(okt::launch_k1(L, S, okt::K1Mode::kAccumSelectHist, g, eps_in, eps_out, fa, n,
                                          &d()->th_arg, nullptr, okt::OutCoo{coo.as<uint64_t>()}, &d()->R, nullptr,
                                          &d()->flags, hp), "k1");
          if (!rc) rc = sync(s);
          if (rc) return abort_step(rc);
          if (P == 1 && (h->flags & 1u)) {  // (P > 1: the split's counts exchange tells every rank)
            dev_stale = true;
            return set_err(OKT_ERR_NUMERIC, "ok_sparse_allreduce: non-finite input");
          }
          if (h->R >= k) {
            have_cand = true;
            C_bound = h->R;
          } else {
            tmark(OKT_T_THRESHOLD, s);
            rc = ck(okt::launch_radix_select(L, okt::RadixSrc::kDenseF32, acc, n, nullptr, n, k, &d()->rs, hp,
                                             &d()->local_th, true), "radix");
          }
        } else {
          if (!rc) rc = ck(okt::launch_k1(L, S, okt::K1Mode::kAccumHist, g, eps_in, eps_out, fa, n, nullptr, nullptr,
                                          okt::OutCoo{}, nullptr, nullptr, &d()->flags, hp), "k1");
          tmark(OKT_T_THRESHOLD, s);
          if (cand_on) {
            if (!rc) rc = ck(okt::launch_radix_pass0_floor(L, &d()->rs, hp, &d()->th_arg), "radix");
            tmark(OKT_T_SELECT, s);
            if (!rc) rc = ck(okt::launch_k1(L, S, okt::K1Mode::kSelect, acc, nullptr, nullptr, 0.f, n, &d()->th_arg,
                                            nullptr, okt::OutCoo{coo.as<uint64_t>()}, &d()->R, nullptr, &d()->flags,
                                            nullptr), "k1");
            have_cand = true;
          } else if (!rc) {
            rc = ck(okt::launch_radix_select(L, okt::RadixSrc::kDenseF32, acc, n, nullptr, n, k, &d()->rs, hp,
                                             &d()->local_th, true), "radix");
          }
        }
        if (have_cand) {
          // the exact k-th largest among the candidates, then the local
          // selection (P > 1, AoS for the split) or u with K7 (P = 1)
          tmark(OKT_T_THRESHOLD, s);
          if (!rc) rc = ck(cudaMemsetAsync(hp, 0, 2048 * sizeof(uint32_t), s), "memset");
          if (!rc) rc = ck(okt::launch_radix_select(L, okt::RadixSrc::kAosF32, coo.p, 0, &d()->R, C_bound, k,
                                                    &d()->rs, hp, &d()->local_th, false), "radix");
          tmark(OKT_T_SELECT, s);
          if (P > 1) {
            if (!rc) rc = ck(okt::launch_filter(L, S, true, coo.as<uint64_t>(), nullptr, nullptr, &d()->R, C_bound,
                                                &d()->local_th, nullptr, nullptr, &d()->m, nullptr,
                                                coo.as<uint64_t>()), "filter");
          } else {
            if (!rc) rc = ck(cudaMemcpyAsync(&d()->global_th, &d()->local_th, 8, cudaMemcpyDeviceToDevice, s), "copy");
            if (!rc) rc = ck(okt::launch_filter(L, S, true, coo.as<uint64_t>(), nullptr, nullptr, &d()->R, C_bound,
                                                &d()->local_th, sur_idx.as<uint32_t>(), sur_val.as<double>(),
                                                &d()->S), "filter");
            if (!rc) rc = ck(cudaMemcpyAsync(&d()->m, &d()->S, 8, cudaMemcpyDeviceToDevice, s), "copy");
            tmark(OKT_T_APPLY, s);
            if (!rc) rc = ck(okt::launch_apply_u(L, sur_idx.as<uint32_t>(), sur_val.as<double>(), &d()->S, C_bound,
                                                 eps_out, w, &d()->flags), "apply");
          }
          sel_done = true;
        }
      } else {
        tmark(OKT_T_THRESHOLD, s);
        rc = ck(okt::launch_radix_select(L, okt::RadixSrc::kDenseF32, acc, n, nullptr, n, k, &d()->rs, hp,
                                         &d()->local_th, false), "radix");
      }
      if (!sel_done) tmark(OKT_T_SELECT, s);
      if (sel_done) {
        // (the candidate path produced u (P = 1) or the local selection (P > 1))
      } else if (P == 1) {
        // One rank: the region is the local selection {|acc| >= local_th}, so
        // its k-th largest magnitude (the global refresh, oktopk.cpp:277-293)
        // is local_th itself, and u = the local selection comes straight out
        // of a dual-threshold select over acc, K7 fused as in the steady step.
        if (!rc) rc = ck(cudaMemcpyAsync(&d()->global_th, &d()->local_th, 8, cudaMemcpyDeviceToDevice, s), "copy");
        if (!rc) rc = ck(okt::launch_k1(L, S, okt::K1Mode::kSelect, acc, nullptr, nullptr, 0.f, n, &d()->local_th,
                                        &d()->global_th,
                                        okt::OutCoo{nullptr, sur_idx.as<uint32_t>(), sur_val.as<double>()},
                                        &d()->S, &d()->m, &d()->flags, nullptr, &ap1), "k1");
      } else if (!rc) {
        rc = ck(okt::launch_k1(L, S, okt::K1Mode::kSelect, acc, nullptr, nullptr, 0.f, n, &d()->local_th, nullptr,
                               okt::OutCoo{coo.as<uint64_t>()}, &d()->m, nullptr, &d()->flags, nullptr), "k1");
      }
    } else if (P == 1) {
      // Steady state, one rank: the region is the local selection itself, so
      // u = {|acc| >= max(local_th, global_th)} comes straight out of K1 and
      // the local selection is only counted.
      tmark(OKT_T_SELECT, s);
      rc = ck(okt::launch_k1(L, S, sgd ? okt::K1Mode::kAccumSelect : okt::K1Mode::kSelect, g, eps_in, eps_out, fa,
                             n, &d()->local_th, &d()->global_th,
                             okt::OutCoo{nullptr, sur_idx.as<uint32_t>(), sur_val.as<double>()}, &d()->S, &d()->m,
                             &d()->flags, nullptr, &ap1), "k1");
    } else {
      tmark(OKT_T_SELECT, s);
      rc = ck(okt::launch_k1(L, S, sgd ? okt::K1Mode::kAccumSelect : okt::K1Mode::kSelect, g, eps_in, eps_out, fa,
                             n, &d()->local_th, nullptr, okt::OutCoo{coo.as<uint64_t>()}, &d()->m, nullptr,
                             &d()->flags, nullptr), "k1");
    }
    if (rc) return abort_step(rc);

    uint64_t U_bound = n;
    const uint64_t* d_U = nullptr;
    const uint32_t* ui = nullptr;
    const double* uv = nullptr;
    std::vector<uint64_t> new_cuts(P + 1, 0);

    if (P == 1) {
      ui = sur_idx.as<uint32_t>();
      uv = sur_val.as<double>();
      d_U = &d()->S;
      new_cuts[0] = 0;
      new_cuts[1] = n;
    } else {
      if (!is_pow2(P)) return set_err(OKT_ERR_CONFIG, "world size must be a power of two");
      // ---- boundaries ----
      if (bnd) {
        tmark(OKT_T_SPLIT, s);
        rc = repartition_dev(coo.as<uint32_t>(), 2, &d()->m, 0, n, s);
        if (rc) return abort_step(rc);
      } else if (st.regions != P) {
        const std::vector<uint64_t> eq = equal_slice_ends(n, P);
        std::memcpy(hup->cuts, eq.data(), sizeof(uint64_t) * (P + 1));
        rc = ck(cudaMemcpyAsync(d()->cuts, hup->cuts, sizeof(uint64_t) * (P + 1), cudaMemcpyHostToDevice, s),
                "upload");
        if (rc) return abort_step(rc);
      }
      uint64_t bound = 0;
      Buf& oi = thr ? reg_idx : sur_idx;
      Buf& ov = thr ? reg_val : sur_val;
      rc = split_reduce_dev(n, st.bucket_size, !thr, &d()->global_th, oi, ov, thr ? &d()->R : &d()->S, bound, s);
      if (rc) return abort_step(rc);
      for (int q = 0; q <= P; ++q) new_cuts[q] = h->cuts[q];
      if (thr) {
        tmark(OKT_T_GLOBAL, s);
        rc = refresh_global_dev(k, bound, s);
        if (!rc) {
          if ((rc = ensure_dd(sur_idx, 4 * std::max<uint64_t>(bound, 1))) ||
              (rc = ensure_dd(sur_val, 8 * std::max<uint64_t>(bound, 1))))
            return abort_step(rc);
          rc = ck(okt::launch_filter(L, S, false, nullptr, reg_idx.as<uint32_t>(), reg_val.as<double>(), &d()->R,
                                     bound, &d()->global_th, sur_idx.as<uint32_t>(), sur_val.as<double>(),
                                     &d()->S), "filter");
        }
        if (rc) return abort_step(rc);
      }
      tmark(OKT_T_ALLGATHER, s);
      uint64_t U = 0;
      rc = balance_allgatherv_dev(s, U);
      if (rc) return abort_step(rc);
      if ((rc = ensure_dd(indexes, 4 * std::max<uint64_t>(U, 1)))) return abort_step(rc);
      if ((rc = upload_u64(&d()->U, U, &hup->U, s))) return abort_step(rc);
      U_bound = U;
      d_U = &d()->U;
      ui = u_idx.as<uint32_t>();
      uv = u_val.as<double>();
    }

    // ---- K7 (fused into the compaction for P = 1; the P2P path returned above) ----
    if (P > 1) {
      tmark(OKT_T_APPLY, s);
      rc = ck(okt::launch_apply(L, S, ui, uv, d_U, U_bound, const_cast<float*>(acc), sgd, sgd ? w : nullptr, P,
                                &d()->local_th, indexes.as<uint32_t>(), &d()->nidx, &d()->flags), "apply");
      if (rc) return abort_step(rc);
    }
    tstop(s);
    if (prof) {
      cudaEvent_t e = ev_get();
      cudaEventRecord(e, s);
      spans.push_back({OKT_T_STEP, step_begin, e});
    }
    if ((rc = sync(s))) return abort_step(rc);
    tcollect();
    return commit_step(n, t, thr, sgd, new_cuts, ui, uv, out);
  }

  bool p2p_credit_pending = false;
  // A step enqueued by okt_sgd_step_async / okt_sparse_allreduce_async whose
  // readback has not been waited for yet.
  struct Pending {
    bool on = false;
    size_t n = 0;
    int64_t t = 0;
    bool thr = false, sgd = false;
    std::vector<uint64_t> cuts;
    const uint32_t* ui = nullptr;
    const double* uv = nullptr;
    cudaStream_t s = nullptr;
  } pending;
  bool defer = false;  // set by the async entry points for the current call
  bool has_sync_result = false;  // an async call that completed synchronously
  okt_result last_result{};

  int wait_pending(okt_result* out) {
    if (!pending.on) return OKT_OK;
    pending.on = false;
    int rc = ck(cudaStreamSynchronize(pending.s), "device");
    if (rc) return abort_step(rc);
    if (hfast_pending) {
      hfast_pending = false;
      if ((rc = read_hfast())) return abort_step(rc);
    }
    if ((rc = read_hp2p())) return abort_step(rc);
    tcollect();
    collect_graph_prof();
    return commit_step(pending.n, pending.t, pending.thr, pending.sgd, pending.cuts, pending.ui, pending.uv, out);
  }
  bool defer_commit(size_t n, int64_t t, bool thr, bool sgd, const std::vector<uint64_t>& cuts, const uint32_t* ui,
                    const double* uv, cudaStream_t s) {
    if (!defer) return false;
    pending = Pending{true, n, t, thr, sgd, cuts, ui, uv, s};
    return true;
  }
  // Error checks + commit of a finished step (h valid, stream synchronised).
  int commit_step(size_t n, int64_t t, bool thr, bool sgd, const std::vector<uint64_t>& new_cuts,
                  const uint32_t* ui, const double* uv, okt_result* out) {
    const bool credit = p2p_credit_pending;
    p2p_credit_pending = false;
    // the P2P EF step produces no index list (oktopk_sgd_step reports none)
    const bool no_indexes = credit && sgd;
    if (prof) {
      // Algorithmic bytes: K1 reads g (+ eps), writes eps and
      // emits the COO (8 B per local entry; 12 B per u entry when the
      // single-rank step emits u directly); refresh iterations add the radix
      // passes over acc; K7 reads u, gathers acc, updates w and eps.
      const double nn = double(n), mm = double(h->m);
      const double uu = double(P == 1 ? h->S : h->U);
      double sel = (sgd ? 12.0 : 4.0) * nn;
      // single-rank EF step: the model half of K7 in phase B (w read + write: 8 B per entry of u)
      sel += (P == 1 && sgd) ? 8.0 * uu : 0.0;
      if (P == 1 && !thr) {
        sel += 12.0 * uu;
      } else {
        sel += 8.0 * mm;
        if (thr && sgd && refresh_dense_select) sel += 4.0 * nn;  // the select-only K1 after the accumulate pass
      }
      t_bytes[OKT_T_SELECT] += sel;
      // the streaming kernel alone: reads g (+ eps), writes eps and 8 B per staged entry
      t_bytes[OKT_T_K1] += (sgd ? 12.0 : 4.0) * nn + 8.0 * ((P == 1 && !thr) ? uu : mm) +
                           ((thr && sgd && refresh_dense_select) ? 4.0 * nn : 0.0);
      if (thr) t_bytes[OKT_T_THRESHOLD] += (sgd ? 2.0 : 3.0) * 4.0 * nn;
      if (P > 1) t_bytes[OKT_T_APPLY] += uu * (sgd ? 28.0 : 16.0);
    }
    if (h->flags & 1u) {
      dev_stale = true;
      return set_err(OKT_ERR_NUMERIC, "ok_sparse_allreduce: non-finite input");
    }
    if (h->flags & 8u) {
      dev_stale = true;
      dead = true;
      return set_err(OKT_ERR_TRANSPORT, "TransportError: a peer did not reach the exchange (timeout)");
    }
    if (h->flags & 16u) {
      dev_stale = true;
      return set_err(OKT_ERR_TRANSPORT, "TransportError: a peer failed (non-finite input)");
    }
    if (credit) p2p_credit();
    if (h->flags & 2u) {
      dev_stale = true;
      return set_err(OKT_ERR_PROTOCOL, "split_and_reduce: entries outside my region");
    }
    // Commit.  Thresholds change only on refresh iterations (oktopk.cpp:258-293);
    // a steady step leaves them alone.  (The steady graph / P2P steps refresh
    // only part of the mirror h, so its threshold words may be stale there.)
    if (thr) {
      st.local_th = h->local_th;
      st.global_th = h->global_th;
      st.last_local_eval = t;
      st.last_global_eval = t;
    }
    st.regions = P;
    for (int q = 0; q <= P; ++q) st.cuts[q] = new_cuts[q];
    st.t = t;
    if (sgd) eps_cur ^= 1;
    if (out) {
      out->u.d_idx = ui;
      out->u.d_val = uv;
      out->u.nnz = P == 1 ? h->S : h->U;
      out->u.n = n;
      out->d_indexes = P == 1 ? ui : (no_indexes ? nullptr : indexes.as<uint32_t>());
      out->n_indexes = P == 1 ? h->S : (no_indexes ? 0 : h->nidx);
      out->local_selected = h->m;
    }
    if (h->flags & 4u) return set_err(OKT_ERR_NUMERIC, "oktopk_sgd_step: non-finite iterate");
    return OKT_OK;
  }

  int abort_step(int rc) {
    dev_stale = true;
    hp2p_pending = false;
    hfast_pending = false;
    {
      std::string e2;  // (bounded: an aborted NCCL comm has ended its kernels)
      if (tr) tr->wait(L.s, e2);
      else cudaStreamSynchronize(L.s);
    }
    cudaGetLastError();
    spans.clear();
    ev_used = 0;
    open_id = -1;
    return rc;
  }

  int residual_reset(size_t n, const float* init, cudaStream_t s) {
    int rc;
    if ((rc = ensure(eps[0], 4 * std::max<size_t>(n, 1)))) return rc;
    if ((rc = ensure(eps[1], 4 * std::max<size_t>(n, 1)))) return rc;
    eps_cur = 0;
    eps_n = n;
    if (init)
      rc = ck(cudaMemcpyAsync(eps[0].p, init, 4 * n, cudaMemcpyDeviceToDevice, s), "residual");
    else
      rc = ck(cudaMemsetAsync(eps[0].p, 0, 4 * n, s), "residual");
    if (rc) return rc;
    return ck(cudaStreamSynchronize(s), "residual");
  }
};

// =============================================================================
// C-ABI
// =============================================================================
namespace {

int init_comm(okt_comm* c) {
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
  c->L.sms = dev_sms;
  okt::preload_kernels();
  // L2 fetch granularity (diagnostics A/B, OKT_L2_FETCH_BYTES = 32 / 64 / 128):
  // the scatter kernels' random 4-byte accesses pull ~128 bytes each from DRAM
  // (phase B at 340M reads 446 MB for 3.4M model words, ncu).  Measured: no
  // effect at 32 or 64 (tools/ab_l2fetch.sh, profiles/r02_l2fetch_ab.txt), so
  // it is only set when asked for.
  if (const char* e = std::getenv("OKT_L2_FETCH_BYTES")) {
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, size_t(std::atoi(e)));
    cudaGetLastError();
  }
  if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ready_ev, cudaEventDisableTiming) != cudaSuccess) {
    return set_err(OKT_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(cudaGetLastError()));
  }
  c->L.s = c->own;
  c->hist.zero_init = true;
  c->scal.zero_init = true;
  c->mask.zero_init = true;
  c->S.max_chunks = dev_sms * 8;
  cudaError_t e = c->hist.ensure(2048 * 4);
  if (e == cudaSuccess) e = c->shist.ensure(2048 * 4);
  if (e == cudaSuccess) e = c->scal.ensure(sizeof(DevScalars));
  if (e == cudaSuccess) e = c->counts.ensure(4 * size_t(c->S.max_chunks));
  if (e == cudaSuccess) e = c->counts2.ensure(4 * size_t(c->S.max_chunks));
  if (e == cudaSuccess) e = c->chunkcap.ensure(64);
  c->tilectr.zero_init = true;
  if (e == cudaSuccess) e = c->tilectr.ensure(64);
  if (e == cudaSuccess) e = cudaMallocHost(&c->h, sizeof(DevScalars));
  if (e == cudaSuccess) e = cudaMallocHost(&c->hup, sizeof(DevScalars));
  if (e == cudaSuccess) e = cudaHostAlloc(&c->hfast, sizeof(okt::HostOut), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hfast_dev), c->hfast, 0);
  if (e == cudaSuccess) e = cudaHostAlloc(&c->hp2p, sizeof(okt::P2PHostOut), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hp2p_dev), c->hp2p, 0);
  if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, std::string("init: ") + cudaGetErrorString(e));
  std::memset(c->h, 0, sizeof(DevScalars));
  std::memset(c->hup, 0, sizeof(DevScalars));
  c->S.counts = c->counts.as<uint32_t>();
  c->S.counts2 = c->counts2.as<uint32_t>();
  c->S.chunk_cap = c->chunkcap.as<uint64_t>();
  c->S.tile_ctr = c->tilectr.as<uint32_t>();
  if (std::getenv("OKT_P2P_TRACE")) {  // diagnostics: per-CTA globaltimer stamps
    c->trbuf.zero_init = true;
    if (c->trbuf.ensure(8 * size_t(okt::kTraceKinds) * okt::kTraceCtas * 4) != cudaSuccess)
      return set_err(OKT_ERR_CUDA, "trace buffer");
  }
  return c->reserve(4096);
}

struct DeviceGuard {
  explicit DeviceGuard(int dev) { cudaSetDevice(dev); }
};

#define OKT_COMM_CHECK(c)                                               \
  do {                                                                  \
    if (!(c)) return set_err(OKT_ERR_INVALID_ARGUMENT, "null comm");    \
  } while (0)

}  // namespace

extern "C" {

int okt_abi_version(void) { return OKT_ABI_VERSION; }

const char* okt_status_string(int s) {
  switch (s) {
    case OKT_OK: return "ok";
    case OKT_ERR_INVALID_ARGUMENT: return "invalid_argument";
    case OKT_ERR_NUMERIC: return "NumericError";
    case OKT_ERR_PROTOCOL: return "ProtocolError";
    case OKT_ERR_TRANSPORT: return "TransportError";
    case OKT_ERR_CONFIG: return "ConfigError";
    case OKT_ERR_CUDA: return "cuda";
    case OKT_ERR_NCCL: return "nccl";
    default: return "internal";
  }
}

const char* okt_last_error(void) { return g_err.c_str(); }

int okt_world_create_local(okt_world** out, int P, const int* devices) {
  if (!out) return set_err(OKT_ERR_INVALID_ARGUMENT, "null out");
  if (P < 1) return set_err(OKT_ERR_INVALID_ARGUMENT, "P must be >= 1");
  if (!is_pow2(P) || P > OKT_MAX_WORLD)
    return set_err(OKT_ERR_CONFIG, "world size must be a power of two <= 8");
  auto* w = new okt_world();
  w->P = P;
  int cur = 0;
  cudaGetDevice(&cur);
  for (int r = 0; r < P; ++r) w->devices.push_back(devices ? devices[r] : cur);
  w->sends.assign(P, std::vector<std::vector<Xfer>>(P));
  w->ready.assign(P, nullptr);
  *out = w;
  return OKT_OK;
}

int okt_world_close(okt_world* w) {
  if (!w) return set_err(OKT_ERR_INVALID_ARGUMENT, "null world");
  w->close();
  return OKT_OK;
}

int okt_world_destroy(okt_world* w) {
  delete w;
  return OKT_OK;
}

int okt_comm_init_local(okt_comm** out, okt_world* w, int rank) {
  if (!out || !w) return set_err(OKT_ERR_INVALID_ARGUMENT, "null argument");
  if (rank < 0 || rank >= w->P) return set_err(OKT_ERR_INVALID_ARGUMENT, "rank out of range");
  auto* c = new okt_comm();
  c->rank = rank;
  c->P = w->P;
  c->device = w->devices[rank];
  c->world = w;
  DeviceGuard g(c->device);
  int rc = init_comm(c);
  if (rc) {
    delete c;
    return rc;
  }
  c->tr.reset(new okt::LocalTransport(w, rank, c->device, c->ready_ev));
  *out = c;
  return OKT_OK;
}

int okt_nccl_unique_id(void* out, size_t len) {
  if (!out || len < sizeof(ncclUniqueId)) return set_err(OKT_ERR_INVALID_ARGUMENT, "buffer too small");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(OKT_ERR_NCCL, ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
  return OKT_OK;
}

int okt_comm_init_nccl(okt_comm** out, int rank, int P, int device, const void* uid, size_t len) {
  if (!out || !uid || len < sizeof(ncclUniqueId)) return set_err(OKT_ERR_INVALID_ARGUMENT, "bad argument");
  if (P < 1 || rank < 0 || rank >= P) return set_err(OKT_ERR_INVALID_ARGUMENT, "bad rank/world");
  if (!is_pow2(P) || P > OKT_MAX_WORLD)
    return set_err(OKT_ERR_CONFIG, "world size must be a power of two <= 8");
  auto* c = new okt_comm();
  c->rank = rank;
  c->P = P;
  c->device = device;
  DeviceGuard g(device);
  int rc = init_comm(c);
  if (rc) {
    delete c;
    return rc;
  }
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t nc = nullptr;
  // Non-blocking communicator: every later wait on it is bounded (okt_transport.hpp).
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  // Blocking by default: a non-blocking communicator made every
  // host-synchronised refresh 3-5x slower (VGG N = 2: 1.8-2.7 vs 0.56 ms per
  // refresh; round-2 A/B).  The waits on the stream stay bounded either way
  // (NcclTransport::wait aborts the communicator at the deadline); only a
  // peer dying inside an enqueue call itself (first-use connection setup)
  // needs OKT_NCCL_NONBLOCKING=1.
  cfg.blocking = std::getenv("OKT_NCCL_NONBLOCKING") ? 0 : 1;
  ncclResult_t r = ncclCommInitRankConfig(&nc, P, id, rank, &cfg);
  if (r == ncclInProgress) r = okt::NcclTransport::settle(nc, std::max(120000L, okt::NcclTransport::timeout_from_env()));
  if (r != ncclSuccess) {
    if (nc) ncclCommAbort(nc);
    delete c;
    return set_err(OKT_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  c->tr.reset(new okt::NcclTransport(nc));
  *out = c;
  return OKT_OK;
}

int okt_comm_destroy(okt_comm* c) {
  if (!c) return OKT_OK;
  DeviceGuard g(c->device);
  cudaStreamSynchronize(c->own);
  c->tr.reset();
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->ready_ev) cudaEventDestroy(c->ready_ev);
  if (c->h) cudaFreeHost(c->h);
  if (c->hup) cudaFreeHost(c->hup);
  if (c->hfast) cudaFreeHost(c->hfast);
  if (c->hp2p) cudaFreeHost(c->hp2p);
  if (c->graph1.exec) cudaGraphExecDestroy(c->graph1.exec);
  if (c->graph1.graph) cudaGraphDestroy(c->graph1.graph);
  if (c->graph2.exec) cudaGraphExecDestroy(c->graph2.exec);
  if (c->graph2.graph) cudaGraphDestroy(c->graph2.graph);
  if (c->graph1.e0) {
    cudaEventDestroy(c->graph1.e0);
    cudaEventDestroy(c->graph1.e1);
  }
  c->close_peers();
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return OKT_OK;
}

int okt_comm_info(const okt_comm* c, int* rank, int* P, int* device) {
  OKT_COMM_CHECK(c);
  if (rank) *rank = c->rank;
  if (P) *P = c->P;
  if (device) *device = c->device;
  return OKT_OK;
}

int okt_comm_reserve(okt_comm* c, size_t n) {
  OKT_COMM_CHECK(c);
  DeviceGuard g(c->device);
  const int rc = c->reserve(n);
  return rc;
}

int okt_get_state(const okt_comm* cc, okt_state* out) {
  OKT_COMM_CHECK(cc);
  okt_comm* c = const_cast<okt_comm*>(cc);
  if (c->pending.on) {
    DeviceGuard g(c->device);
    const int rc = c->wait_pending(nullptr);
    if (rc) return rc;
  }
  if (!out) return set_err(OKT_ERR_INVALID_ARGUMENT, "null out");
  *out = c->st;
  return OKT_OK;
}

int okt_set_state(okt_comm* c, const okt_state* in) {
  OKT_COMM_CHECK(c);
  if (c->pending.on) {
    DeviceGuard g(c->device);
    const int rc = c->wait_pending(nullptr);
    if (rc) return rc;
  }
  if (!in) return set_err(OKT_ERR_INVALID_ARGUMENT, "null state");
  c->st = *in;
  c->dev_stale = true;
  return OKT_OK;
}

int okt_set_params(okt_comm* c, uint32_t tau, uint32_t tau_prime, uint32_t bucket) {
  OKT_COMM_CHECK(c);
  if (tau == 0 || tau_prime == 0) return set_err(OKT_ERR_INVALID_ARGUMENT, "tau and tau_prime must be >= 1");
  c->st.tau = tau;
  c->st.tau_prime = tau_prime;
  c->st.bucket_size = bucket;
  return OKT_OK;
}

int okt_ledger(const okt_comm* cc, int phase, okt_counters* out) {
  OKT_COMM_CHECK(cc);
  okt_comm* c = const_cast<okt_comm*>(cc);
  if (c->pending.on) {
    DeviceGuard g(c->device);
    const int rc = c->wait_pending(nullptr);
    if (rc) return rc;
  }
  if (phase < 0 || phase >= OKT_PHASE_COUNT || !out) return set_err(OKT_ERR_INVALID_ARGUMENT, "bad phase");
  *out = c->ledger[phase];
  return OKT_OK;
}

int okt_ledger_reset(okt_comm* c) {
  OKT_COMM_CHECK(c);
  std::memset(c->ledger, 0, sizeof(c->ledger));
  return OKT_OK;
}

int okt_sparse_allreduce(okt_comm* c, const float* d_acc, size_t n, int64_t t, size_t k, okt_result* out,
                         void* stream) {
  OKT_COMM_CHECK(c);
  DeviceGuard g(c->device);
  int rc = c->reserve(n);
  if (rc) return rc;
  return c->step(d_acc, nullptr, n, 0.0, t, k, false, out, c->pick(stream));
}

int okt_sparse_allreduce_async(okt_comm* c, const float* d_acc, size_t n, int64_t t, size_t k, void* stream) {
  OKT_COMM_CHECK(c);
  DeviceGuard g(c->device);
  int rc = c->reserve(n);
  if (rc) return rc;
  c->defer = true;
  c->has_sync_result = false;
  rc = c->step(d_acc, nullptr, n, 0.0, t, k, false, &c->last_result, c->pick(stream));
  c->defer = false;
  c->has_sync_result = rc == OKT_OK && !c->pending.on;
  return rc;
}

int okt_sgd_step_async(okt_comm* c, const float* d_grad, float* d_w, size_t n, double alpha, int64_t t, size_t k,
                       void* stream) {
  OKT_COMM_CHECK(c);
  if (!d_w) return set_err(OKT_ERR_INVALID_ARGUMENT, "null model");
  DeviceGuard g(c->device);
  int rc = c->reserve(n);
  if (rc) return rc;
  c->defer = true;
  c->has_sync_result = false;
  rc = c->step(d_grad, d_w, n, alpha, t, k, true, &c->last_result, c->pick(stream));
  c->defer = false;
  c->has_sync_result = rc == OKT_OK && !c->pending.on;
  return rc;
}

int okt_device_barrier(okt_comm* c, void* stream) {
  OKT_COMM_CHECK(c);
  DeviceGuard g(c->device);
  int rc;
  if ((rc = c->wait_pending(nullptr))) return rc;
  cudaStream_t s = c->pick(stream);
  if (c->P == 1) return OKT_OK;
  if (c->p2p) {
    c->L.s = s;
    return c->ck(okt::launch_p2p_barrier(c->L, c->tabd.as<okt::PeerTab>(), ++c->bar_epoch, &c->d()->flags,
                                         kP2PTimeoutNs), "barrier");
  }
  int one = 1;
  std::vector<int> all(c->P);
  return c->allgather_host(&one, all.data(), sizeof(int), s);
}

int okt_step_wait(okt_comm* c, okt_result* out) {
  OKT_COMM_CHECK(c);
  DeviceGuard g(c->device);
  if (!c->pending.on) {
    if (!c->has_sync_result) return set_err(OKT_ERR_INVALID_ARGUMENT, "no step in flight");
    c->has_sync_result = false;
    if (out) *out = c->last_result;
    return OKT_OK;
  }
  return c->wait_pending(out);
}

int okt_residual_reset(okt_comm* c, size_t n, const float* d_init, void* stream) {
  OKT_COMM_CHECK(c);
  if (c->pending.on && c->wait_pending(nullptr)) return OKT_ERR_INTERNAL;
  DeviceGuard g(c->device);
  return c->residual_reset(n, d_init, c->pick(stream));
}

int okt_residual(okt_comm* c, float** d_eps, size_t* n) {
  OKT_COMM_CHECK(c);
  if (c->pending.on) {
    DeviceGuard g(c->device);
    const int rc = c->wait_pending(nullptr);
    if (rc) return rc;
  }
  if (d_eps) *d_eps = c->eps_n ? c->eps[c->eps_cur].as<float>() : nullptr;
  if (n) *n = c->eps_n;
  return OKT_OK;
}

int okt_sgd_step(okt_comm* c, const float* d_grad, float* d_w, size_t n, double alpha, int64_t t, size_t k,
                 okt_result* out, void* stream) {
  OKT_COMM_CHECK(c);
  if (!d_w) return set_err(OKT_ERR_INVALID_ARGUMENT, "null model");
  DeviceGuard g(c->device);
  int rc = c->reserve(n);
  if (rc) return rc;
  return c->step(d_grad, d_w, n, alpha, t, k, true, out, c->pick(stream));
}

// ---- host-buffer entry points --------------------------------------------------------
static int copy_result_to_host(okt_comm* c, const okt_result& r, uint32_t* h_idx, double* h_val,
                               uint32_t* h_indexes, size_t cap, cudaStream_t s) {
  if (!h_idx && !h_val && !h_indexes) return OKT_OK;  // result stays on the device
  if (r.u.nnz > cap) return set_err(OKT_ERR_INVALID_ARGUMENT, "u does not fit the host buffers");
  cudaError_t e = cudaSuccess;
  if (r.u.nnz && h_idx) e = cudaMemcpyAsync(h_idx, r.u.d_idx, 4 * r.u.nnz, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && r.u.nnz && h_val)
    e = cudaMemcpyAsync(h_val, r.u.d_val, 8 * r.u.nnz, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && r.n_indexes && h_indexes)
    e = cudaMemcpyAsync(h_indexes, r.d_indexes, 4 * r.n_indexes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return c->ck(e, "copy result");
}

// The host gradient is staged into device memory with one H2D copy (copy
// engine).  Reading a pinned gradient in place from K1 over PCIe was measured
// slower end to end (1.27 vs 1.22 ms/iter at the VGG size): the copy engine
// sustains more PCIe read bandwidth than SM-issued loads.
static const float* host_input(okt_comm* c, const float* h, size_t n, cudaStream_t s, int* rc) {
  if ((*rc = c->ensure(c->hgrad, 4 * std::max<size_t>(n, 1)))) return nullptr;
  if (n && (*rc = c->ck(cudaMemcpyAsync(c->hgrad.p, h, 4 * n, cudaMemcpyHostToDevice, s), "h2d"))) return nullptr;
  return c->hgrad.as<float>();
}

int okt_sparse_allreduce_host(okt_comm* c, const float* h_acc, size_t n, int64_t t, size_t k, uint32_t* h_u_idx,
                              double* h_u_val, uint32_t* h_indexes, size_t u_cap, okt_result* out, void* stream) {
  OKT_COMM_CHECK(c);
  if (!h_acc) return set_err(OKT_ERR_INVALID_ARGUMENT, "null gradient");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  int rc;
  const float* gin = host_input(c, h_acc, n, s, &rc);
  if (rc) return rc;
  okt_result r{};
  if ((rc = c->reserve(n))) return rc;
  rc = c->step(gin, nullptr, n, 0.0, t, k, false, &r, s);
  if (rc) return rc;
  if (out) *out = r;
  return copy_result_to_host(c, r, h_u_idx, h_u_val, h_indexes, u_cap, s);
}

int okt_sgd_step_host(okt_comm* c, const float* h_grad, float* d_w, size_t n, double alpha, int64_t t, size_t k,
                      uint32_t* h_u_idx, double* h_u_val, size_t u_cap, okt_result* out, void* stream) {
  OKT_COMM_CHECK(c);
  if (!h_grad || !d_w) return set_err(OKT_ERR_INVALID_ARGUMENT, "null argument");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  int rc;
  const float* gin = host_input(c, h_grad, n, s, &rc);
  if (rc) return rc;
  okt_result r{};
  if ((rc = c->reserve(n))) return rc;
  rc = c->step(gin, d_w, n, alpha, t, k, true, &r, s);
  if (rc) return rc;
  if (out) *out = r;
  return copy_result_to_host(c, r, h_u_idx, h_u_val, nullptr, u_cap, s);
}

int okt_memcpy_h2d(void* d_dst, const void* h_src, size_t bytes, void* stream) {
  cudaError_t e = stream ? cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream))
                         : cudaMemcpy(d_dst, h_src, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, cudaGetErrorString(e));
  return OKT_OK;
}

int okt_memcpy_d2h(void* h_dst, const void* d_src, size_t bytes, void* stream) {
  cudaError_t e = stream ? cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream))
                         : cudaMemcpy(h_dst, d_src, bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && stream) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, cudaGetErrorString(e));
  return OKT_OK;
}

// ---- sub-phases ----------------------------------------------------------------------
int okt_th_re_evaluate_dense(okt_comm* c, const float* d_g, size_t n, size_t k, double* th, void* stream) {
  OKT_COMM_CHECK(c);
  if (n == 0) return set_err(OKT_ERR_INVALID_ARGUMENT, "th_re_evaluate: empty gradient");
  if (k < 1) return set_err(OKT_ERR_INVALID_ARGUMENT, "th_re_evaluate: k must be >= 1");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc = c->ck(okt::launch_radix_select(c->L, okt::RadixSrc::kDenseF32, d_g, n, nullptr, n, k, &c->d()->rs,
                                          c->hist.as<uint32_t>(), &c->d()->th_arg, false), "radix");
  if (rc || (rc = c->sync(s))) return rc;
  *th = c->h->th_arg;
  return OKT_OK;
}

int okt_th_re_evaluate_sparse(okt_comm* c, const double* d_val, size_t nnz, size_t k, double* th, void* stream) {
  OKT_COMM_CHECK(c);
  if (nnz == 0) return set_err(OKT_ERR_INVALID_ARGUMENT, "th_re_evaluate: empty gradient");
  if (k < 1) return set_err(OKT_ERR_INVALID_ARGUMENT, "th_re_evaluate: k must be >= 1");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc = c->ck(okt::launch_radix_select(c->L, okt::RadixSrc::kF64, d_val, nnz, nullptr, nnz, k, &c->d()->rs,
                                          c->hist.as<uint32_t>(), &c->d()->th_arg, false), "radix");
  if (rc || (rc = c->sync(s))) return rc;
  *th = c->h->th_arg;
  return OKT_OK;
}

int okt_select_by_threshold(okt_comm* c, const float* d_g, size_t n, double th, okt_sparse* out, void* stream) {
  OKT_COMM_CHECK(c);
  if (!(th >= 0.0)) return set_err(OKT_ERR_INVALID_ARGUMENT, "select_by_threshold: th must be >= 0");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc = c->reserve(std::max<size_t>(n, 1));
  if (rc) return rc;
  if ((rc = c->ensure(c->sel_idx, 4 * std::max<size_t>(n, 1))) ||
      (rc = c->ensure(c->sel_val, 8 * std::max<size_t>(n, 1))))
    return rc;
  if ((rc = c->upload_f64(&c->d()->th_arg, th, &c->hup->th_arg, s))) return rc;
  if (n) {
    rc = c->ck(okt::launch_k1(c->L, c->S, okt::K1Mode::kSelect, d_g, nullptr, nullptr, 0.f, n, &c->d()->th_arg,
                              nullptr, okt::OutCoo{nullptr, c->sel_idx.as<uint32_t>(), c->sel_val.as<double>()},
                              &c->d()->m, nullptr, &c->d()->flags, nullptr), "k1");
  } else {
    rc = c->ck(cudaMemsetAsync(&c->d()->m, 0, 8, s), "memset");
  }
  if (rc || (rc = c->sync(s))) return rc;
  out->d_idx = c->sel_idx.as<uint32_t>();
  out->d_val = c->sel_val.as<double>();
  out->nnz = c->h->m;
  out->n = n;
  return OKT_OK;
}

int okt_space_repartition(okt_comm* c, const uint32_t* d_sel_idx, size_t m, size_t n, uint64_t* cuts_out,
                          void* stream) {
  OKT_COMM_CHECK(c);
  if (!cuts_out) return set_err(OKT_ERR_INVALID_ARGUMENT, "null cuts");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc = c->repartition_dev(d_sel_idx, 1, nullptr, m, n, s);
  if (rc || (rc = c->sync(s))) return rc;
  for (int q = 0; q <= c->P; ++q) cuts_out[q] = c->h->cuts[q];
  c->dev_stale = true;  // device cuts no longer mirror the state
  return OKT_OK;
}

int okt_split_and_reduce(okt_comm* c, const float* d_g, size_t n, double local_th, const uint64_t* cuts,
                         uint32_t bucket, okt_sparse* region, okt_sparse* local, void* stream) {
  OKT_COMM_CHECK(c);
  if (!cuts) return set_err(OKT_ERR_INVALID_ARGUMENT, "split_and_reduce: boundaries do not match P");
  if (!(local_th >= 0.0)) return set_err(OKT_ERR_INVALID_ARGUMENT, "select_by_threshold: th must be >= 0");
  if (n == 0 || n > 0xffffffffull) return set_err(OKT_ERR_INVALID_ARGUMENT, "bad n");
  for (int q = 0; q < c->P; ++q)
    if (cuts[q] > cuts[q + 1] || cuts[c->P] > n)
      return set_err(OKT_ERR_INVALID_ARGUMENT, "split_and_reduce: bad boundaries");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc = c->reserve(n);
  if (rc) return rc;
  if ((rc = c->ensure(c->sel_idx, 4 * n)) || (rc = c->ensure(c->sel_val, 8 * n))) return rc;
  if ((rc = c->upload_f64(&c->d()->th_arg, local_th, &c->hup->th_arg, s))) return rc;
  std::memcpy(c->hup->cuts, cuts, sizeof(uint64_t) * (c->P + 1));
  if ((rc = c->ck(cudaMemcpyAsync(c->d()->cuts, c->hup->cuts, sizeof(uint64_t) * (c->P + 1),
                                  cudaMemcpyHostToDevice, s), "upload")))
    return rc;
  c->dev_stale = true;
  if ((rc = c->ck(cudaMemsetAsync(&c->d()->flags, 0, 4, s), "memset"))) return rc;
  rc = c->ck(okt::launch_k1(c->L, c->S, okt::K1Mode::kSelect, d_g, nullptr, nullptr, 0.f, n, &c->d()->th_arg,
                            nullptr, okt::OutCoo{c->coo.as<uint64_t>()}, &c->d()->m, nullptr, &c->d()->flags,
                            nullptr), "k1");
  if (rc) return rc;
  // The reference's split_and_reduce does not test finiteness; keep the
  // collective non-finite abort of the full step out of this entry point.
  if ((rc = c->ck(cudaMemsetAsync(&c->d()->flags, 0, 4, s), "memset"))) return rc;
  if (c->P == 1) {
    if ((rc = c->ensure(c->reg_idx, 4 * n)) || (rc = c->ensure(c->reg_val, 8 * n))) return rc;
    rc = c->ck(okt::launch_extract(c->L, c->coo.as<uint64_t>(), &c->d()->m, n, c->reg_idx.as<uint32_t>(),
                                   c->reg_val.as<double>()), "extract");
    if (rc) return rc;
    rc = c->ck(cudaMemcpyAsync(&c->d()->R, &c->d()->m, 8, cudaMemcpyDeviceToDevice, s), "copy");
  } else {
    uint64_t bound = 0;
    rc = c->split_reduce_dev(n, bucket, false, nullptr, c->reg_idx, c->reg_val, &c->d()->R, bound, s);
  }
  if (rc) return c->abort_step(rc);
  rc = c->ck(okt::launch_extract(c->L, c->coo.as<uint64_t>(), &c->d()->m, n, c->sel_idx.as<uint32_t>(),
                                 c->sel_val.as<double>()), "extract");
  if (rc || (rc = c->sync(s))) return rc;
  if (c->h->flags & 2u) return set_err(OKT_ERR_PROTOCOL, "split_and_reduce: entries outside my region");
  region->d_idx = c->reg_idx.as<uint32_t>();
  region->d_val = c->reg_val.as<double>();
  region->nnz = c->h->R;
  region->n = n;
  local->d_idx = c->sel_idx.as<uint32_t>();
  local->d_val = c->sel_val.as<double>();
  local->nnz = c->h->m;
  local->n = n;
  return OKT_OK;
}

int okt_balance_and_allgatherv(okt_comm* c, const uint32_t* d_idx, const double* d_val, size_t nnz, size_t n,
                               double global_th, okt_sparse* u, void* stream) {
  OKT_COMM_CHECK(c);
  if (!(global_th >= 0.0)) return set_err(OKT_ERR_INVALID_ARGUMENT, "select_by_threshold: th must be >= 0");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc;
  if ((rc = c->ensure(c->sur_idx, 4 * std::max<size_t>(nnz, 1))) ||
      (rc = c->ensure(c->sur_val, 8 * std::max<size_t>(nnz, 1))))
    return rc;
  if ((rc = c->upload_f64(&c->d()->th_arg, global_th, &c->hup->th_arg, s))) return rc;
  if ((rc = c->upload_u64(&c->d()->R, nnz, &c->hup->R, s))) return rc;
  rc = c->ck(okt::launch_filter(c->L, c->S, false, nullptr, d_idx, d_val, &c->d()->R, nnz, &c->d()->th_arg,
                                c->sur_idx.as<uint32_t>(), c->sur_val.as<double>(), &c->d()->S), "filter");
  if (rc) return rc;
  if (c->P == 1) {
    if ((rc = c->sync(s))) return rc;
    u->d_idx = c->sur_idx.as<uint32_t>();
    u->d_val = c->sur_val.as<double>();
    u->nnz = c->h->S;
    u->n = n;
    return OKT_OK;
  }
  uint64_t U = 0;
  rc = c->balance_allgatherv_dev(s, U);
  if (rc || (rc = c->sync(s))) return rc;
  u->d_idx = c->u_idx.as<uint32_t>();
  u->d_val = c->u_val.as<double>();
  u->nnz = U;
  u->n = n;
  return OKT_OK;
}

// ---- Table-1 baselines (collectives.cpp:152-354) ---------------------------------------
// TopkA, gTopk, TopkDSA and Gaussiank on the GPU: the comparison collectives
// of the paper's Table 1.  They are host-orchestrated (a sync per exchange
// round, as the reference's blocking send/recv) and exact against the
// reference: the same selections, the same combination trees and the same
// fp64 adds.  Kernels in okt_baselines.cu; exchanges over the comm's
// transport; ledger credited as the reference's Message words (ints + reals).
namespace {

struct SpRef {  // a device SoA sparse list
  uint32_t* idx = nullptr;
  double* val = nullptr;
  uint64_t nnz = 0;
};

// Exclusive prefix of per-chunk counts, uploaded next to them; returns the total.
int bl_prefix(okt_comm* c, const uint32_t* d_cnt, uint64_t chunks, uint64_t* d_off, uint64_t& total,
              cudaStream_t s) {
  std::vector<uint32_t> hc(chunks);
  int rc = c->ck(cudaMemcpyAsync(hc.data(), d_cnt, 4 * chunks, cudaMemcpyDeviceToHost, s), "d2h");
  if (rc || (rc = c->wait_stream(s))) return rc;
  std::vector<uint64_t> ho(chunks);
  uint64_t pos = 0;
  for (uint64_t i = 0; i < chunks; ++i) {
    ho[i] = pos;
    pos += hc[i];
  }
  total = pos;
  rc = c->ck(cudaMemcpyAsync(d_off, ho.data(), 8 * chunks, cudaMemcpyHostToDevice, s), "h2d");
  if (rc || (rc = c->wait_stream(s))) return rc;
  return OKT_OK;
}

uint64_t bl_chunks(uint64_t m) { return (m + okt::kTopkTrimChunk - 1) / okt::kTopkTrimChunk; }

// topk_exact's trim of a selection whose k-th largest magnitude is th: every
// |v| > th, then the first k - #gt ties.  Source: AoS f32 (aos_in) or SoA f64.
int bl_trim(okt_comm* c, const uint64_t* aos_in, const uint32_t* idx_in, const double* val_in, uint64_t m,
            double th, uint64_t k, uint64_t* aos_out, uint32_t* idx_out, double* val_out, cudaStream_t s) {
  const uint64_t chunks = bl_chunks(m);
  int rc = c->ensure(c->tk_aux, 24 * std::max<uint64_t>(chunks, 1));
  if (rc) return rc;
  uint32_t* gt = c->tk_aux.as<uint32_t>();
  uint32_t* eq = gt + chunks;
  uint64_t* off = reinterpret_cast<uint64_t*>(c->tk_aux.as<char>() + 8 * chunks);
  uint64_t* eqb = off + chunks;
  rc = c->ck(okt::launch_topk_count(c->L, aos_in, idx_in, val_in, m, th, gt, eq), "topk_count");
  if (rc) return rc;
  std::vector<uint32_t> hc(2 * chunks);
  if ((rc = c->ck(cudaMemcpyAsync(hc.data(), gt, 8 * chunks, cudaMemcpyDeviceToHost, s), "d2h"))) return rc;
  if ((rc = c->wait_stream(s))) return rc;
  uint64_t n_gt = 0;
  for (uint64_t i = 0; i < chunks; ++i) n_gt += hc[i];
  if (n_gt >= k) return set_err(OKT_ERR_INTERNAL, "topk_exact: threshold above the k-th magnitude");
  const uint64_t need = k > n_gt ? k - n_gt : 0;
  std::vector<uint64_t> ho(2 * chunks);
  uint64_t pos = 0, eq_seen = 0;
  for (uint64_t i = 0; i < chunks; ++i) {
    ho[i] = pos;
    ho[chunks + i] = eq_seen;
    const uint64_t keep_eq = eq_seen >= need ? 0 : std::min<uint64_t>(hc[chunks + i], need - eq_seen);
    pos += hc[i] + keep_eq;
    eq_seen += hc[chunks + i];
  }
  if (pos != k) return set_err(OKT_ERR_INTERNAL, "topk_exact: tie trim miscounted");
  if ((rc = c->ck(cudaMemcpyAsync(off, ho.data(), 16 * chunks, cudaMemcpyHostToDevice, s), "h2d"))) return rc;
  rc = c->ck(okt::launch_topk_write(c->L, aos_in, idx_in, val_in, m, th, off, eqb, need, aos_out, idx_out, val_out),
             "topk_write");
  if (rc || (rc = c->wait_stream(s))) return rc;
  return OKT_OK;
}

// Local exact top-k of a dense fp32 gradient (topk_exact, sparse.cpp:75-80):
// radix select of the k-th magnitude, K1 select {|g| >= th} into coo, trim.
// `bad` reports a non-finite gradient (the trim is then skipped).
int bl_local_topk(okt_comm* c, const float* d_g, uint64_t n, uint64_t k, uint64_t* aos_out, uint32_t* idx_out,
                  double* val_out, bool& bad, cudaStream_t s) {
  int rc = c->reserve(n);
  if (rc) return rc;
  rc = c->ck(cudaMemsetAsync(&c->d()->flags, 0, 4, s), "memset");
  if (!rc)
    rc = c->ck(okt::launch_radix_select(c->L, okt::RadixSrc::kDenseF32, d_g, n, nullptr, n, k, &c->d()->rs,
                                        c->hist.as<uint32_t>(), &c->d()->th_arg, false), "radix");
  if (!rc)
    rc = c->ck(okt::launch_k1(c->L, c->S, okt::K1Mode::kSelect, d_g, nullptr, nullptr, 0.f, n, &c->d()->th_arg,
                              nullptr, okt::OutCoo{c->coo.as<uint64_t>(), nullptr, nullptr}, &c->d()->m, nullptr,
                              &c->d()->flags, nullptr), "k1");
  if (rc || (rc = c->sync(s))) return rc;
  bad = (c->h->flags & 1u) != 0;
  if (bad) return OKT_OK;
  if (c->h->m < k) return set_err(OKT_ERR_INTERNAL, "topk_exact: selection smaller than k");
  return bl_trim(c, c->coo.as<uint64_t>(), nullptr, nullptr, c->h->m, c->h->th_arg, k, aos_out, idx_out, val_out,
                 s);
}

// Every rank's (count, health) before any data moves; a non-finite rank fails
// with NumericError, the others with TransportError (the reference's abort).
int bl_agree(okt_comm* c, const char* who, uint64_t count, bool bad, std::vector<uint64_t>& counts, cudaStream_t s) {
  const int P = c->P;
  counts.assign(P, 0);
  if (P == 1) {
    if (bad) return set_err(OKT_ERR_NUMERIC, std::string(who) + ": non-finite input");
    counts[0] = count;
    return OKT_OK;
  }
  c->hup->small[0] = uint32_t(count);
  c->hup->small[1] = bad ? 1u : 0u;
  int rc = c->ck(cudaMemcpyAsync(&c->d()->small[0], &c->hup->small[0], 8, cudaMemcpyHostToDevice, s), "h2d");
  if (rc) return rc;
  std::string err;
  rc = c->tr->allgather(&c->d()->small[0], c->d()->small_all, 8, s, err);
  if (rc) return c->comm_err(rc, err);
  if ((rc = c->sync(s))) return rc;
  for (int q = 0; q < P; ++q) {
    if (c->h->small_all[2 * q + 1]) {
      if (q == c->rank) return set_err(OKT_ERR_NUMERIC, std::string(who) + ": non-finite input");
      return set_err(OKT_ERR_TRANSPORT, "TransportError: rank " + std::to_string(q) + " failed (non-finite input)");
    }
    counts[q] = c->h->small_all[2 * q];
  }
  return OKT_OK;
}

// sparse_allgatherv of AoS f32 parts (counts[q] entries each, parts laid out
// back to back by rank) + sparse_sum (stride-doubling bracket) via the region
// merge over [0, n).  Result in sel_idx/sel_val.
int bl_allgather_sum_aos(okt_comm* c, uint64_t n, const std::vector<uint64_t>& counts, okt_sparse* out,
                         cudaStream_t s) {
  const int P = c->P, rank = c->rank;
  std::vector<uint64_t> off(P + 1, 0);
  for (int q = 0; q < P; ++q) off[q + 1] = off[q] + counts[q];
  uint64_t* parts = c->tk_parts.as<uint64_t>();
  std::vector<Xfer> sends, recvs;
  for (int q = 0; q < P; ++q) {
    if (q == rank) continue;
    sends.push_back({q, parts + off[rank], 8 * counts[rank]});
    recvs.push_back({q, parts + off[q], 8 * counts[q]});
  }
  std::string err;
  int rc = c->tr->exchange(sends, recvs, s, err);
  if (rc) return c->comm_err(rc, err);
  c->credit_allgatherv(OKT_PHASE_ALLGATHERV, counts, 12);
  const uint64_t bound = std::max<uint64_t>(off[P], 1);
  if ((rc = c->ensure(c->mask, ((n + 15) / 16) * 16 + 16)) || (rc = c->ensure(c->stage, 4 * n * size_t(P))) ||
      (rc = c->ensure(c->sel_idx, 4 * bound)) || (rc = c->ensure(c->sel_val, 8 * bound)))
    return rc;
  okt::Segs segs{};
  segs.nseg = P;
  segs.start[0] = 0;
  for (int q = 0; q < P; ++q) {
    segs.ptr[q] = parts + off[q];
    segs.src[q] = q;
    segs.start[q + 1] = off[q + 1];
  }
  rc = c->ck(okt::launch_scatter(c->L, segs, 0, n, P, c->mask.as<uint32_t>(), c->stage.as<float>(), &c->d()->flags),
             "scatter");
  if (!rc)
    rc = c->ck(okt::launch_region_scan(c->L, c->S, P, false, 0, n, c->mask.as<uint32_t>(), c->stage.as<float>(),
                                       nullptr, c->sel_idx.as<uint32_t>(), c->sel_val.as<double>(), &c->d()->R),
               "region_scan");
  if (rc || (rc = c->sync(s))) return rc;
  out->d_idx = c->sel_idx.as<uint32_t>();
  out->d_val = c->sel_val.as<double>();
  out->nnz = c->h->R;
  out->n = n;
  return OKT_OK;
}

// merge_two (sparse.cpp:206-237) of two sorted SoA lists into `o` (capacity
// a.nnz + b.nnz); returns o.nnz.
int bl_merge(okt_comm* c, const SpRef& a, const SpRef& b, SpRef& o, cudaStream_t s) {
  const uint64_t N = a.nnz + b.nnz;
  int rc;
  if ((rc = c->ensure(c->bl_ti, 4 * std::max<uint64_t>(N, 1))) || (rc = c->ensure(c->bl_tv, 8 * std::max<uint64_t>(N, 1))))
    return rc;
  const uint64_t chunks = bl_chunks(N);
  if ((rc = c->ensure(c->tk_aux, 24 * std::max<uint64_t>(chunks, 1)))) return rc;
  uint32_t* cnt = c->tk_aux.as<uint32_t>();
  uint64_t* off = reinterpret_cast<uint64_t*>(c->tk_aux.as<char>() + 8 * chunks);
  uint32_t* ti = c->bl_ti.as<uint32_t>();
  double* tv = c->bl_tv.as<double>();
  rc = c->ck(okt::launch_merge_rank(c->L, a.idx, a.val, a.nnz, b.idx, b.val, b.nnz, ti, tv), "merge_rank");
  if (!rc) rc = c->ck(okt::launch_merge_heads(c->L, ti, tv, N, cnt, nullptr, nullptr, nullptr), "merge_count");
  uint64_t total = 0;
  if (rc || (rc = bl_prefix(c, cnt, chunks, off, total, s))) return rc;
  rc = c->ck(okt::launch_merge_heads(c->L, ti, tv, N, nullptr, off, o.idx, o.val), "merge_write");
  o.nnz = total;
  return rc;
}

// One send and one receive with `partner` (the reference's paired send/recv).
int bl_swap(okt_comm* c, int partner, const std::vector<std::pair<const void*, size_t>>& out,
            const std::vector<std::pair<void*, size_t>>& in, cudaStream_t s) {
  std::vector<Xfer> sends, recvs;
  for (auto& x : out) sends.push_back({partner, const_cast<void*>(x.first), x.second});
  for (auto& x : in) recvs.push_back({partner, x.first, x.second});
  std::string err;
  int rc = c->tr->exchange(sends, recvs, s, err);
  if (rc) return c->comm_err(rc, err);
  return OKT_OK;
}

int bl_check(okt_comm* c, const char* who, const float* d_g, size_t n, size_t k, okt_sparse* out) {
  (void)c;
  if (!out || (!d_g && n)) return set_err(OKT_ERR_INVALID_ARGUMENT, std::string(who) + ": null argument");
  if (k < 1 || k > n) return set_err(OKT_ERR_INVALID_ARGUMENT, "topk_exact: k must be in [1, n]");
  if (n > 0xffffffffull) return set_err(OKT_ERR_INVALID_ARGUMENT, std::string(who) + ": n exceeds 32-bit indices");
  return OKT_OK;
}

void bl_credit_pair(okt_comm* c, int ph, uint64_t sent_words, uint64_t recv_words) {
  okt::plan::credit(c->ledger[ph], true, sent_words, 1);
  okt::plan::credit(c->ledger[ph], false, recv_words, 1);
}

// Acklam's rational approximation of the standard normal quantile, refined by
// two Halley steps on the erfc-based CDF (the reference's inverse_normal_cdf,
// sparse.cpp:122-165).
double inverse_normal_cdf(double p) {
  static const double A[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
  static const double B[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01,  -1.328068155288572e+01};
  static const double C[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
  static const double D[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  const double plow = 0.02425;
  auto tail = [&](double q) {
    return (((((C[0] * q + C[1]) * q + C[2]) * q + C[3]) * q + C[4]) * q + C[5]) /
           ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
  };
  double x;
  if (p < plow) {
    x = tail(std::sqrt(-2.0 * std::log(p)));
  } else if (p <= 1.0 - plow) {
    const double q = p - 0.5, r = q * q;
    x = (((((A[0] * r + A[1]) * r + A[2]) * r + A[3]) * r + A[4]) * r + A[5]) * q /
        (((((B[0] * r + B[1]) * r + B[2]) * r + B[3]) * r + B[4]) * r + 1.0);
  } else {
    x = -tail(std::sqrt(-2.0 * std::log(1.0 - p)));
  }
  const double sqrt2pi = 2.5066282746310005;
  for (int it = 0; it < 2; ++it) {
    const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
    const double u = e * sqrt2pi * std::exp(x * x / 2.0);
    x = x - u / (1.0 + x * u / 2.0);
  }
  return x;
}

}  // namespace

// dense_allreduce (collectives.cpp:89-150): the fp32 gradient widened to fp64,
// recursive-halving reduce-scatter over equal_slice_ends (own + partner's half,
// the reference's adds), recursive-doubling allgather of the reduced slices.
int okt_dense_allreduce(okt_comm* c, const float* d_g, size_t n, double** d_out, void* stream) {
  OKT_COMM_CHECK(c);
  if (!d_out || (!d_g && n)) return set_err(OKT_ERR_INVALID_ARGUMENT, "dense_allreduce: null argument");
  if (n > 0xffffffffull) return set_err(OKT_ERR_INVALID_ARGUMENT, "dense_allreduce: n exceeds 32-bit sizes");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  const int P = c->P, rank = c->rank;
  int rc;
  if ((rc = c->ensure(c->bl_win, 8 * std::max<size_t>(n, 1))) || (rc = c->ensure(c->bl_win_in, 8 * std::max<size_t>(n, 1))))
    return rc;
  double* buf = c->bl_win.as<double>();
  double* in = c->bl_win_in.as<double>();
  if ((rc = c->ck(okt::launch_widen_f32(c->L, d_g, n, buf), "widen"))) return rc;
  std::vector<uint64_t> sizes;
  if ((rc = bl_agree(c, "dense_allreduce", n, false, sizes, s))) return rc;
  for (int q = 0; q < P; ++q)
    if (sizes[q] != n) return set_err(OKT_ERR_PROTOCOL, "ProtocolError: dense_allreduce: length mismatch");
  if (P > 1) {
    const std::vector<uint64_t> ends = equal_slice_ends(n, P);
    int lo = 0, hi = P;
    for (int mask = P >> 1; mask > 0; mask >>= 1) {
      const int partner = rank ^ mask, mid = lo + mask;
      const bool low = (rank & mask) == 0;
      const int keep_lo = low ? lo : mid, keep_hi = low ? mid : hi, send_lo = low ? mid : lo, send_hi = low ? hi : mid;
      const uint64_t sc = ends[send_hi] - ends[send_lo], kc = ends[keep_hi] - ends[keep_lo];
      rc = bl_swap(c, partner, {{buf + ends[send_lo], 8 * sc}}, {{in, 8 * kc}}, s);
      if (rc) return rc;
      bl_credit_pair(c, OKT_PHASE_DENSE, sc, kc);
      if ((rc = c->ck(okt::launch_window_add(c->L, buf + ends[keep_lo], in, kc), "window_add"))) return rc;
      lo = keep_lo;
      hi = keep_hi;
    }
    for (int mask = 1; mask < P; mask <<= 1) {
      const int partner = rank ^ mask, base = rank & ~(2 * mask - 1);
      const int my_lo = (rank & mask) ? base + mask : base, their_lo = (rank & mask) ? base : base + mask;
      const uint64_t mc = ends[my_lo + mask] - ends[my_lo], tc = ends[their_lo + mask] - ends[their_lo];
      rc = bl_swap(c, partner, {{buf + ends[my_lo], 8 * mc}}, {{buf + ends[their_lo], 8 * tc}}, s);
      if (rc) return rc;
      bl_credit_pair(c, OKT_PHASE_DENSE, mc, tc);
    }
  }
  if ((rc = c->wait_stream(s))) return rc;
  *d_out = buf;
  return OKT_OK;
}

// topka_allreduce (collectives.cpp:152-159): exact local top-k, sparse_allgatherv,
// sparse_sum.
int okt_topka_allreduce(okt_comm* c, const float* d_g, size_t n, size_t k, okt_sparse* out, void* stream) {
  OKT_COMM_CHECK(c);
  int rc = bl_check(c, "topka_allreduce", d_g, n, k, out);
  if (rc) return rc;
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  const int P = c->P;
  if ((rc = c->ensure(c->tk_parts, 8 * k * size_t(P)))) return rc;
  if (P == 1 && ((rc = c->ensure(c->sel_idx, 4 * k)) || (rc = c->ensure(c->sel_val, 8 * k)))) return rc;
  bool bad = false;
  rc = bl_local_topk(c, d_g, n, k, P > 1 ? c->tk_parts.as<uint64_t>() + k * uint64_t(c->rank) : nullptr,
                     P == 1 ? c->sel_idx.as<uint32_t>() : nullptr, P == 1 ? c->sel_val.as<double>() : nullptr, bad,
                     s);
  if (rc) return rc;
  std::vector<uint64_t> counts;
  if ((rc = bl_agree(c, "topka_allreduce", k, bad, counts, s))) return rc;
  for (int q = 0; q < P; ++q)
    if (counts[q] != k) return set_err(OKT_ERR_PROTOCOL, "topka_allreduce: ranks disagree on k");
  if (P == 1) {
    *out = okt_sparse{c->sel_idx.as<uint32_t>(), c->sel_val.as<double>(), k, n};
    return OKT_OK;
  }
  return bl_allgather_sum_aos(c, n, counts, out, s);
}

// gtopk_allreduce (collectives.cpp:300-325): log2 P rounds of pairwise
// exchange; each rank sums its k entries with its partner's (merge_two) and
// keeps the exact top-k of the sum.  Every list has exactly k entries.
int okt_gtopk_allreduce(okt_comm* c, const float* d_g, size_t n, size_t k, okt_sparse* out, void* stream) {
  OKT_COMM_CHECK(c);
  int rc = bl_check(c, "gtopk_allreduce", d_g, n, k, out);
  if (rc) return rc;
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  const int P = c->P, rank = c->rank;
  if ((rc = c->ensure(c->bl_ai, 4 * k)) || (rc = c->ensure(c->bl_av, 8 * k)) || (rc = c->ensure(c->bl_bi, 4 * k)) ||
      (rc = c->ensure(c->bl_bv, 8 * k)) || (rc = c->ensure(c->bl_ci, 8 * k)) || (rc = c->ensure(c->bl_cv, 16 * k)))
    return rc;
  SpRef A{c->bl_ai.as<uint32_t>(), c->bl_av.as<double>(), k};
  SpRef B{c->bl_bi.as<uint32_t>(), c->bl_bv.as<double>(), k};
  SpRef C{c->bl_ci.as<uint32_t>(), c->bl_cv.as<double>(), 0};
  bool bad = false;
  if ((rc = bl_local_topk(c, d_g, n, k, nullptr, A.idx, A.val, bad, s))) return rc;
  std::vector<uint64_t> counts;
  if ((rc = bl_agree(c, "gtopk_allreduce", k, bad, counts, s))) return rc;
  for (int q = 0; q < P; ++q)
    if (counts[q] != k) return set_err(OKT_ERR_PROTOCOL, "gtopk_allreduce: ranks disagree on k");
  for (int level = 0; (1 << level) < P; ++level) {
    const int partner = rank ^ (1 << level);
    rc = bl_swap(c, partner, {{A.idx, 4 * k}, {A.val, 8 * k}}, {{B.idx, 4 * k}, {B.val, 8 * k}}, s);
    if (rc) return rc;
    bl_credit_pair(c, OKT_PHASE_SPLIT, 2 * k, 2 * k);
    if ((rc = bl_merge(c, A, B, C, s))) return rc;
    // topk_exact(SparseGrad, k), sparse.cpp:82-92: C.nnz >= k always.
    rc = c->ck(okt::launch_radix_select(c->L, okt::RadixSrc::kF64, C.val, C.nnz, nullptr, C.nnz, k, &c->d()->rs,
                                        c->hist.as<uint32_t>(), &c->d()->th_arg, false), "radix");
    if (rc || (rc = c->sync(s))) return rc;
    if ((rc = bl_trim(c, nullptr, C.idx, C.val, C.nnz, c->h->th_arg, k, nullptr, A.idx, A.val, s))) return rc;
  }
  if ((rc = c->ensure(c->sel_idx, 4 * k)) || (rc = c->ensure(c->sel_val, 8 * k))) return rc;
  rc = c->ck(cudaMemcpyAsync(c->sel_idx.p, A.idx, 4 * k, cudaMemcpyDeviceToDevice, s), "copy");
  if (!rc) rc = c->ck(cudaMemcpyAsync(c->sel_val.p, A.val, 8 * k, cudaMemcpyDeviceToDevice, s), "copy");
  if (rc || (rc = c->wait_stream(s))) return rc;
  *out = okt_sparse{c->sel_idx.as<uint32_t>(), c->sel_val.as<double>(), k, n};
  return OKT_OK;
}

// topkdsa_allreduce (collectives.cpp:184-297): recursive-halving reduce-scatter
// of the exact local top-k whose working set switches from COO to a dense fp64
// window once 2·nnz >= the window width, then sparse_allgatherv of the owned
// segments (disjoint, ascending: concatenation is the sum).
int okt_topkdsa_allreduce(okt_comm* c, const float* d_g, size_t n, size_t k, okt_sparse* out, void* stream) {
  OKT_COMM_CHECK(c);
  int rc = bl_check(c, "topkdsa_allreduce", d_g, n, k, out);
  if (rc) return rc;
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  const int P = c->P, rank = c->rank;
  // two COO ping-pong sets of capacity n, a partner COO, two dense windows
  if ((rc = c->ensure(c->bl_ai, 4 * n)) || (rc = c->ensure(c->bl_av, 8 * n)) || (rc = c->ensure(c->bl_ci, 4 * n)) ||
      (rc = c->ensure(c->bl_cv, 8 * n)) || (rc = c->ensure(c->bl_bi, 4 * n)) || (rc = c->ensure(c->bl_bv, 8 * n)) ||
      (rc = c->ensure(c->bl_win, 8 * n)) || (rc = c->ensure(c->bl_win_in, 8 * n)) || (rc = c->ensure(c->bl_small, 64)))
    return rc;
  SpRef A{c->bl_ai.as<uint32_t>(), c->bl_av.as<double>(), k};
  SpRef B{c->bl_bi.as<uint32_t>(), c->bl_bv.as<double>(), 0};
  bool bad = false;
  if ((rc = bl_local_topk(c, d_g, n, k, nullptr, A.idx, A.val, bad, s))) return rc;
  std::vector<uint64_t> counts;
  if ((rc = bl_agree(c, "topkdsa_allreduce", k, bad, counts, s))) return rc;
  if (P == 1) {
    if ((rc = c->ensure(c->sel_idx, 4 * k)) || (rc = c->ensure(c->sel_val, 8 * k))) return rc;
    rc = c->ck(cudaMemcpyAsync(c->sel_idx.p, A.idx, 4 * k, cudaMemcpyDeviceToDevice, s), "copy");
    if (!rc) rc = c->ck(cudaMemcpyAsync(c->sel_val.p, A.val, 8 * k, cudaMemcpyDeviceToDevice, s), "copy");
    if (rc || (rc = c->wait_stream(s))) return rc;
    *out = okt_sparse{c->sel_idx.as<uint32_t>(), c->sel_val.as<double>(), k, n};
    return OKT_OK;
  }
  const std::vector<uint64_t> ends = equal_slice_ends(n, P);
  bool dense = false;
  double* wbase = nullptr;  // window over [win_lo, win_hi)
  uint64_t win_lo = 0, win_hi = 0;
  auto densify = [&](uint64_t lo, uint64_t hi) -> int {  // dsa_densify, collectives.cpp:172-182
    wbase = c->bl_win.as<double>();
    int r = c->ck(cudaMemsetAsync(wbase, 0, 8 * (hi - lo), s), "memset");
    if (!r) r = c->ck(okt::launch_window_scatter(c->L, A.idx, A.val, A.nnz, lo, wbase, false), "densify");
    win_lo = lo;
    win_hi = hi;
    dense = true;
    A.nnz = 0;
    return r;
  };
  uint64_t* hb = reinterpret_cast<uint64_t*>(&c->hup->prop[0]);  // 4 words of pinned staging
  int lo = 0, hi = P;
  for (int mask = P >> 1; mask > 0; mask >>= 1) {
    const int partner = rank ^ mask, mid = lo + mask;
    int keep_lo, keep_hi, send_lo, send_hi;
    if ((rank & mask) == 0) {
      keep_lo = lo; keep_hi = mid; send_lo = mid; send_hi = hi;
    } else {
      keep_lo = mid; keep_hi = hi; send_lo = lo; send_hi = mid;
    }
    const uint64_t s0 = ends[send_lo], s1 = ends[send_hi], k0 = ends[keep_lo], k1 = ends[keep_hi];
    // sparse_slice bounds of the send and keep halves
    uint64_t a_s0 = 0, a_s1 = 0, a_k0 = 0, a_k1 = 0;
    if (!dense) {
      uint64_t* sb = c->bl_small.as<uint64_t>();
      rc = c->ck(okt::launch_slice_bounds(c->L, A.idx, A.nnz, s0, s1, sb), "slice");
      if (!rc) rc = c->ck(okt::launch_slice_bounds(c->L, A.idx, A.nnz, k0, k1, sb + 2), "slice");
      if (!rc) rc = c->ck(cudaMemcpyAsync(hb, sb, 32, cudaMemcpyDeviceToHost, s), "d2h");
      if (rc || (rc = c->wait_stream(s))) return rc;
      a_s0 = hb[0]; a_s1 = hb[1]; a_k0 = hb[2]; a_k1 = hb[3];
    }
    // header {kind, count}: 1 = dense half, 0 = COO
    const uint32_t my_kind = dense ? 1u : 0u;
    const uint64_t my_cnt = dense ? s1 - s0 : a_s1 - a_s0;
    c->hup->small[0] = my_kind;
    c->hup->small[1] = uint32_t(my_cnt);
    if ((rc = c->ck(cudaMemcpyAsync(&c->d()->small[0], &c->hup->small[0], 8, cudaMemcpyHostToDevice, s), "h2d")))
      return rc;
    rc = bl_swap(c, partner, {{&c->d()->small[0], 8}}, {{&c->d()->small_all[0], 8}}, s);
    if (rc) return rc;
    if ((rc = c->sync(s))) return rc;
    const uint32_t th_kind = c->h->small_all[0];
    const uint64_t th_cnt = c->h->small_all[1];
    if (th_kind == 1 && th_cnt != k1 - k0) return set_err(OKT_ERR_PROTOCOL, "topkdsa: dense half length mismatch");
    std::vector<std::pair<const void*, size_t>> outs;
    std::vector<std::pair<void*, size_t>> ins;
    if (dense) outs.push_back({wbase + (s0 - win_lo), 8 * my_cnt});
    else outs = {{A.idx + a_s0, 4 * my_cnt}, {A.val + a_s0, 8 * my_cnt}};
    if (th_kind == 1) ins.push_back({c->bl_win_in.p, 8 * th_cnt});
    else ins = {{B.idx, 4 * th_cnt}, {B.val, 8 * th_cnt}};
    if ((rc = bl_swap(c, partner, outs, ins, s))) return rc;
    bl_credit_pair(c, OKT_PHASE_SPLIT, dense ? my_cnt : 2 * my_cnt, th_kind == 1 ? th_cnt : 2 * th_cnt);
    // restrict the working set to the kept half
    if (dense) {
      wbase += k0 - win_lo;
      win_lo = k0;
      win_hi = k1;
    } else {
      A.idx += a_k0;
      A.val += a_k0;
      A.nnz = a_k1 - a_k0;
    }
    // fold in the partner's contribution
    if (th_kind == 1) {
      if (!dense && (rc = densify(k0, k1))) return rc;
      if ((rc = c->ck(okt::launch_window_add(c->L, wbase, c->bl_win_in.as<double>(), k1 - k0), "window_add")))
        return rc;
    } else {
      B.nnz = th_cnt;
      if (dense) {
        if ((rc = c->ck(okt::launch_window_scatter(c->L, B.idx, B.val, B.nnz, win_lo, wbase, true), "scatter_add")))
          return rc;
      } else {
        // lower-rank contribution first (the bracket); the adds commute
        const bool in_first = A.idx >= c->bl_ai.as<uint32_t>() && A.idx < c->bl_ai.as<uint32_t>() + n;
        SpRef dst{in_first ? c->bl_ci.as<uint32_t>() : c->bl_ai.as<uint32_t>(),
                  in_first ? c->bl_cv.as<double>() : c->bl_av.as<double>(), 0};
        if ((rc = rank < partner ? bl_merge(c, A, B, dst, s) : bl_merge(c, B, A, dst, s))) return rc;
        A = dst;
      }
    }
    // storage crossover: COO costs two words per entry, the window one per coordinate
    if (!dense && 2 * A.nnz >= k1 - k0 && (rc = densify(k0, k1))) return rc;
    lo = keep_lo;
    hi = keep_hi;
  }
  // the owned segment
  SpRef seg = A;
  if (dense) {
    const uint64_t W = win_hi - win_lo, chunks = bl_chunks(W);
    if ((rc = c->ensure(c->tk_aux, 24 * std::max<uint64_t>(chunks, 1)))) return rc;
    uint32_t* cnt = c->tk_aux.as<uint32_t>();
    uint64_t* off = reinterpret_cast<uint64_t*>(c->tk_aux.as<char>() + 8 * chunks);
    seg = SpRef{c->bl_bi.as<uint32_t>(), c->bl_bv.as<double>(), 0};
    rc = c->ck(okt::launch_dense_nonzero(c->L, wbase, W, win_lo, cnt, nullptr, nullptr, nullptr), "nz_count");
    uint64_t total = 0;
    if (rc || (rc = bl_prefix(c, cnt, chunks, off, total, s))) return rc;
    if ((rc = c->ck(okt::launch_dense_nonzero(c->L, wbase, W, win_lo, nullptr, off, seg.idx, seg.val), "nz_write")))
      return rc;
    seg.nnz = total;
  }
  // sparse_allgatherv of the segments, concatenated in rank order
  std::vector<uint64_t> segn;
  if ((rc = bl_agree(c, "topkdsa_allreduce", seg.nnz, false, segn, s))) return rc;
  std::vector<uint64_t> off(P + 1, 0);
  for (int q = 0; q < P; ++q) off[q + 1] = off[q] + segn[q];
  const uint64_t U = off[P];
  if ((rc = c->ensure(c->sel_idx, 4 * std::max<uint64_t>(U, 1))) ||
      (rc = c->ensure(c->sel_val, 8 * std::max<uint64_t>(U, 1))))
    return rc;
  uint32_t* ui = c->sel_idx.as<uint32_t>();
  double* uv = c->sel_val.as<double>();
  rc = c->ck(cudaMemcpyAsync(ui + off[rank], seg.idx, 4 * seg.nnz, cudaMemcpyDeviceToDevice, s), "copy");
  if (!rc) rc = c->ck(cudaMemcpyAsync(uv + off[rank], seg.val, 8 * seg.nnz, cudaMemcpyDeviceToDevice, s), "copy");
  if (rc) return rc;
  std::vector<Xfer> sends, recvs;
  for (int q = 0; q < P; ++q) {
    if (q == rank) continue;
    sends.push_back({q, seg.idx, 4 * seg.nnz});
    sends.push_back({q, seg.val, 8 * seg.nnz});
    recvs.push_back({q, ui + off[q], 4 * segn[q]});
    recvs.push_back({q, uv + off[q], 8 * segn[q]});
  }
  std::string err;
  rc = c->tr->exchange(sends, recvs, s, err);
  if (rc) return c->comm_err(rc, err);
  c->credit_allgatherv(OKT_PHASE_ALLGATHERV, segn, 12);
  if ((rc = c->wait_stream(s))) return rc;
  *out = okt_sparse{ui, uv, U, n};
  return OKT_OK;
}

// gaussian_threshold (sparse.cpp:167-188; scale_to_floor = 0, the raw value)
// or gaussiank_scaled_threshold (collectives.cpp:327-340; 1: clamped at 0 and
// scaled by 0.9 until more than 3k/4 coordinates pass).  Mean and unbiased
// variance in fp64 by a fixed-shape tree (the reference sums sequentially: the
// two agree to a few ulp), the normal quantile at 1 - k/(2n) on the host.
int okt_gaussiank_threshold(okt_comm* c, const float* d_g, size_t n, size_t k, int scale_to_floor, double* th,
                            void* stream) {
  OKT_COMM_CHECK(c);
  if (!th || (!d_g && n)) return set_err(OKT_ERR_INVALID_ARGUMENT, "gaussian_threshold: null argument");
  if (n < 2) return set_err(OKT_ERR_INVALID_ARGUMENT, "gaussian_threshold: need n >= 2");
  if (k < 1 || k > n) return set_err(OKT_ERR_INVALID_ARGUMENT, "gaussian_threshold: k must be in [1, n]");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  int rc;
  if ((rc = c->ensure(c->bl_small, 8 * 1024 + 64))) return rc;
  double* partial = c->bl_small.as<double>() + 8;
  double* dm = c->bl_small.as<double>();
  rc = c->ck(okt::launch_moments(c->L, d_g, n, partial, dm, dm + 1), "moments");
  double* hm = reinterpret_cast<double*>(&c->hup->prop[0]);
  if (!rc) rc = c->ck(cudaMemcpyAsync(hm, dm, 16, cudaMemcpyDeviceToHost, s), "d2h");
  if (rc || (rc = c->wait_stream(s))) return rc;
  const double mean = hm[0], var = hm[1];
  if (!std::isfinite(mean) || !std::isfinite(var))
    return set_err(OKT_ERR_NUMERIC, "gaussian_threshold: non-finite input");
  if (var == 0.0) return set_err(OKT_ERR_NUMERIC, "DegenerateDistributionError: gaussian_threshold: zero variance input");
  const double p = 1.0 - double(k) / (2.0 * double(n));
  double t = mean + std::sqrt(var) * inverse_normal_cdf(p);
  if (scale_to_floor) {
    t = std::max(t, 0.0);
    auto* hc = reinterpret_cast<unsigned long long*>(&c->hup->prop[2]);
    auto* dc = reinterpret_cast<unsigned long long*>(dm + 2);
    for (;;) {
      rc = c->ck(okt::launch_count_ge(c->L, d_g, n, t, dc), "count_ge");
      if (!rc) rc = c->ck(cudaMemcpyAsync(hc, dc, 8, cudaMemcpyDeviceToHost, s), "d2h");
      if (rc || (rc = c->wait_stream(s))) return rc;
      if (4 * uint64_t(*hc) > 3 * uint64_t(k)) break;
      t *= 0.9;
    }
  }
  *th = t;
  return OKT_OK;
}

// gaussiank_allreduce (collectives.cpp:342-352): Gaussian-fit threshold,
// select_by_threshold, sparse_allgatherv, sparse_sum.
int okt_gaussiank_allreduce(okt_comm* c, const float* d_g, size_t n, size_t k, int scale_to_floor, okt_sparse* out,
                            void* stream) {
  OKT_COMM_CHECK(c);
  if (!out) return set_err(OKT_ERR_INVALID_ARGUMENT, "gaussiank_allreduce: null output");
  if (n > 0xffffffffull) return set_err(OKT_ERR_INVALID_ARGUMENT, "gaussiank_allreduce: n exceeds 32-bit indices");
  DeviceGuard g(c->device);
  cudaStream_t s = c->pick(stream);
  c->L.s = s;
  const int P = c->P;
  double th = 0.0;
  int rc = okt_gaussiank_threshold(c, d_g, n, k, scale_to_floor, &th, stream);
  // a numeric failure (non-finite or zero-variance input) still joins the
  // agreement below, so the other ranks fail instead of waiting
  const bool bad = rc == OKT_ERR_NUMERIC;
  const std::string why = bad ? std::string(okt_last_error()) : std::string();
  if (rc && !bad) return rc;
  th = std::max(th, 0.0);
  uint64_t m = 0;
  if (!bad) {
    if ((rc = c->reserve(n))) return rc;
    if ((rc = c->upload_f64(&c->d()->th_arg, th, &c->hup->th_arg, s))) return rc;
    rc = c->ck(okt::launch_k1(c->L, c->S, okt::K1Mode::kSelect, d_g, nullptr, nullptr, 0.f, n, &c->d()->th_arg,
                              nullptr, okt::OutCoo{c->coo.as<uint64_t>(), nullptr, nullptr}, &c->d()->m, nullptr,
                              &c->d()->flags, nullptr), "k1");
    if (rc || (rc = c->sync(s))) return rc;
    m = c->h->m;
  }
  std::vector<uint64_t> counts;
  if ((rc = bl_agree(c, "gaussiank_allreduce", m, bad, counts, s))) {
    if (bad && rc == OKT_ERR_NUMERIC) set_err(OKT_ERR_NUMERIC, why);
    return rc;
  }
  uint64_t total = 0;
  for (int q = 0; q < P; ++q) total += counts[q];
  if (P == 1) {
    if ((rc = c->ensure(c->sel_idx, 4 * std::max<uint64_t>(m, 1))) ||
        (rc = c->ensure(c->sel_val, 8 * std::max<uint64_t>(m, 1))))
      return rc;
    const uint64_t chunks = bl_chunks(m);
    if ((rc = c->ensure(c->tk_aux, 24 * std::max<uint64_t>(chunks, 1)))) return rc;
    std::vector<uint64_t> ho(chunks);
    for (uint64_t i = 0; i < chunks; ++i) ho[i] = i * okt::kTopkTrimChunk;
    uint64_t* off = c->tk_aux.as<uint64_t>();
    if (chunks && (rc = c->ck(cudaMemcpyAsync(off, ho.data(), 8 * chunks, cudaMemcpyHostToDevice, s), "h2d")))
      return rc;
    rc = c->ck(okt::launch_aos_to_soa(c->L, c->coo.as<uint64_t>(), m, off, c->sel_idx.as<uint32_t>(),
                                      c->sel_val.as<double>()), "aos_to_soa");
    if (rc || (rc = c->wait_stream(s))) return rc;
    *out = okt_sparse{c->sel_idx.as<uint32_t>(), c->sel_val.as<double>(), m, n};
    return OKT_OK;
  }
  // parts back to back by rank
  if ((rc = c->ensure(c->tk_parts, 8 * std::max<uint64_t>(total, 1)))) return rc;
  uint64_t my_off = 0;
  for (int q = 0; q < c->rank; ++q) my_off += counts[q];
  rc = c->ck(cudaMemcpyAsync(c->tk_parts.as<uint64_t>() + my_off, c->coo.p, 8 * m, cudaMemcpyDeviceToDevice, s),
             "copy");
  if (rc) return rc;
  return bl_allgather_sum_aos(c, n, counts, out, s);
}

// ---- host planning (no GPU) ------------------------------------------------------------
int okt_plan_cuts(const uint64_t* proposals, int P, uint64_t n, uint64_t* cuts) {
  if (!proposals || !cuts || P < 1 || P > OKT_MAX_WORLD) return set_err(OKT_ERR_INVALID_ARGUMENT, "bad argument");
  const std::vector<uint64_t> c = okt::plan::cuts_from_proposals(proposals, P, n);
  std::memcpy(cuts, c.data(), sizeof(uint64_t) * (P + 1));
  return OKT_OK;
}

int okt_plan_balance(int rank, int P, const uint64_t* sizes, int* balanced, okt_piece* sends, int* nsends,
                     okt_piece* recvs, int* nrecvs, okt_piece* own, uint64_t* part_off, uint64_t* part_sz) {
  if (!sizes || P < 1 || P > OKT_MAX_WORLD || rank < 0 || rank >= P)
    return set_err(OKT_ERR_INVALID_ARGUMENT, "bad argument");
  const okt::plan::Balance B = okt::plan::balance(rank, P, std::vector<uint64_t>(sizes, sizes + P));
  if (balanced) *balanced = B.on ? 1 : 0;
  auto put = [](const std::vector<okt::plan::Piece>& v, okt_piece* out, int* cnt) {
    if (cnt) *cnt = int(v.size());
    if (out)
      for (size_t i = 0; i < v.size(); ++i) out[i] = okt_piece{v[i].peer, v[i].a, v[i].b};
  };
  put(B.sends, sends, nsends);
  put(B.recvs, recvs, nrecvs);
  if (own) *own = okt_piece{B.own.peer, B.own.a, B.own.b};
  for (int q = 0; q < P; ++q) {
    if (part_off) part_off[q] = B.part_off[q];
    if (part_sz) part_sz[q] = B.part_sz[q];
  }
  return OKT_OK;
}

int okt_plan_ledger(int rank, int P, int kind, const uint64_t* sizes, uint64_t len, uint32_t bucket,
                    okt_counters* out) {
  if (!out || P < 1 || P > OKT_MAX_WORLD || rank < 0 || rank >= P)
    return set_err(OKT_ERR_INVALID_ARGUMENT, "bad argument");
  std::memset(out, 0, sizeof(*out));
  switch (kind) {
    case OKT_PLAN_SPLIT: okt::plan::ledger_split(*out, rank, P, sizes, bucket); break;
    case OKT_PLAN_ALLGATHERV: okt::plan::ledger_allgatherv(*out, rank, P, sizes); break;
    case OKT_PLAN_AVG: okt::plan::ledger_avg(*out, P, len); break;
    case OKT_PLAN_ALLGATHER_U32: okt::plan::ledger_allgather_u32(*out, P); break;
    case OKT_PLAN_BALANCE:
      okt::plan::ledger_balance(*out, okt::plan::balance(rank, P, std::vector<uint64_t>(sizes, sizes + P)));
      break;
    default: return set_err(OKT_ERR_INVALID_ARGUMENT, "unknown ledger kind");
  }
  return OKT_OK;
}

// ---- instrumentation --------------------------------------------------------------------
int okt_set_profiling(okt_comm* c, int on) {
  OKT_COMM_CHECK(c);
  c->prof = on != 0;
  c->L.k1_event = c->prof ? &okt_comm::k1_event_cb : nullptr;
  c->L.k1_ctx = c;
  // Events are created up front: creation is not allowed inside a capture.
  while (c->prof && c->k1_pool.size() < 16) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    c->k1_pool.push_back(e);
  }
  while (c->prof && c->ev_pool.size() < 64) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    c->ev_pool.push_back(e);
  }
  return OKT_OK;
}

int okt_phase_times(okt_comm* c, double* ms, uint64_t* calls) {
  OKT_COMM_CHECK(c);
  for (int i = 0; i < OKT_T_COUNT; ++i) {
    if (ms) ms[i] = c->t_ms[i];
    if (calls) calls[i] = c->t_calls[i];
  }
  return OKT_OK;
}

int okt_phase_bytes(okt_comm* c, double* bytes) {
  OKT_COMM_CHECK(c);
  for (int i = 0; i < OKT_T_COUNT; ++i)
    if (bytes) bytes[i] = c->t_bytes[i];
  return OKT_OK;
}

int okt_reset_phase_times(okt_comm* c) {
  OKT_COMM_CHECK(c);
  std::memset(c->t_bytes, 0, sizeof(c->t_bytes));
  std::memset(c->t_ms, 0, sizeof(c->t_ms));
  std::memset(c->t_calls, 0, sizeof(c->t_calls));
  return OKT_OK;
}

int okt_kernel_launches(const okt_comm* c, uint64_t* out) {
  OKT_COMM_CHECK(c);
  if (out) *out = c->L.launches;
  return OKT_OK;
}

int okt_debug_p2p_trace(okt_comm* c, uint64_t* out, size_t n_words) {
  OKT_COMM_CHECK(c);
  if (!c->trbuf.p) return OKT_ERR_CONFIG;
  const size_t words = std::min(n_words, size_t(okt::kTraceKinds) * okt::kTraceCtas * 4);
  cudaSetDevice(c->device);
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(out, c->trbuf.p, 8 * words, cudaMemcpyDeviceToHost) != cudaSuccess)
    return OKT_ERR_CUDA;
  return OKT_OK;
}

// ---- COO wire codec ------------------------------------------------------------
int okt_wire_encode(const uint32_t* d_idx, const double* d_val, size_t nnz, void* d_out, void* stream) {
  if (!d_out || (nnz && (!d_idx || !d_val))) return set_err(OKT_ERR_INVALID_ARGUMENT, "wire_encode: null buffer");
  if (reinterpret_cast<uintptr_t>(d_out) & 3u) return set_err(OKT_ERR_INVALID_ARGUMENT, "wire_encode: unaligned image");
  if (nnz > 0xffffffffull) return set_err(OKT_ERR_INVALID_ARGUMENT, "wire_encode: nnz does not fit the u32 header");
  okt::Launch L;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&L.sms, cudaDevAttrMultiProcessorCount, dev);
  L.s = static_cast<cudaStream_t>(stream);
  cudaError_t e = okt::launch_wire_encode(L, d_idx, d_val, nnz, static_cast<uint32_t*>(d_out));
  if (e == cudaSuccess) e = cudaStreamSynchronize(L.s);
  if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, std::string("wire_encode: ") + cudaGetErrorString(e));
  return OKT_OK;
}

int okt_wire_decode(const void* d_in, size_t bytes, size_t n, uint32_t* d_idx, double* d_val, size_t cap,
                    size_t* nnz_out, void* stream) {
  if (!d_in || !nnz_out) return set_err(OKT_ERR_INVALID_ARGUMENT, "wire_decode: null buffer");
  if (reinterpret_cast<uintptr_t>(d_in) & 3u) return set_err(OKT_ERR_INVALID_ARGUMENT, "wire_decode: unaligned image");
  if (bytes < 4) return set_err(OKT_ERR_DECODE, "wire_decode: missing header");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t nnz = 0;
  cudaError_t e = cudaMemcpyAsync(&nnz, d_in, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, std::string("wire_decode: ") + cudaGetErrorString(e));
  if (bytes != 4 + 8 * size_t(nnz)) return set_err(OKT_ERR_DECODE, "wire_decode: buffer length does not match nnz header");
  if (nnz > cap || (nnz && (!d_idx || !d_val)))
    return set_err(OKT_ERR_DECODE, "wire_decode: output capacity below nnz");
  okt::Launch L;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&L.sms, cudaDevAttrMultiProcessorCount, dev);
  L.s = s;
  uint32_t* d_err = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&d_err), 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_err, 0, 4, s);
  if (e == cudaSuccess && nnz)
    e = okt::launch_wire_decode(L, static_cast<const uint32_t*>(d_in), nnz, n, d_idx, d_val, d_err);
  uint32_t err = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, s);
  if (d_err) cudaFreeAsync(d_err, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_err(OKT_ERR_CUDA, std::string("wire_decode: ") + cudaGetErrorString(e));
  if (err) return set_err(OKT_ERR_DECODE, "wire_decode: index out of range or not strictly increasing");
  *nnz_out = nnz;
  return OKT_OK;
}

}  // extern "C"
