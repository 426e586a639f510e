/*
 * okt.h — C-ABI of the B200-native Ok-Topk sparse allreduce (arXiv 2201.07598).
 *
 * This is the drop-in boundary for the reference's hot path.  Every entry point
 * below names the reference interface it replaces (paths relative to the
 * reference tree, `proj/core/...`).  Plain pointers and sizes only: no C++ or
 * torch types cross this boundary.  Device pointers are marked `d_`; they must
 * be CUDA device memory on the comm's device.
 *
 *   reference                                            replaced by
 *   ---------------------------------------------------  ---------------------------
 *   ok_sparse_allreduce   include/oklab/oktopk.hpp:118    okt_sparse_allreduce
 *   oktopk_sgd_step       include/oklab/trainer.hpp:149   okt_sgd_step (+ okt_residual_*)
 *   th_re_evaluate(Dense) include/oklab/oktopk.hpp:41     okt_th_re_evaluate_dense
 *   th_re_evaluate(Sparse)include/oklab/oktopk.hpp:42     okt_th_re_evaluate_sparse
 *   select_by_threshold   include/oklab/sparse.hpp:87     okt_select_by_threshold
 *   space_repartition     include/oklab/oktopk.hpp:58     okt_space_repartition
 *   split_and_reduce      include/oklab/oktopk.hpp:77     okt_split_and_reduce
 *   balance_and_allgatherv include/oklab/oktopk.hpp:92    okt_balance_and_allgatherv
 *   dense_allreduce       include/oklab/collectives.hpp:28  okt_dense_allreduce (Table-1 baselines)
 *   topka_allreduce       include/oklab/collectives.hpp:33  okt_topka_allreduce
 *   gtopk_allreduce       include/oklab/collectives.hpp:53  okt_gtopk_allreduce
 *   topkdsa_allreduce     include/oklab/collectives.hpp:45  okt_topkdsa_allreduce
 *   gaussiank_allreduce   include/oklab/collectives.hpp:70  okt_gaussiank_allreduce
 *   gaussian_threshold    include/oklab/sparse.hpp:102, collectives.hpp:64  okt_gaussiank_threshold
 *   WorkerCtx / Transport include/oklab/transport.hpp:91-122  okt_world / okt_comm
 *   TrafficLedger         include/oklab/transport.hpp:52  okt_ledger
 *   OkState/ThresholdState include/oklab/oktopk.hpp:30, sparse.hpp:56  okt_state
 *   errors.hpp exception types                           okt_status codes
 *
 * Threading: one okt_comm per rank; a comm is thread-compatible, not
 * thread-safe.  Every collective entry point must be called by all P ranks of
 * the world with the same (n, t, k) — from one host thread per rank
 * (okt_world_create_local, the reference's run_ranks model,
 * proj/tests/test_util.hpp:38-76) or from one process per GPU
 * (okt_comm_init_nccl).
 *
 * Precision: dense state (gradient, accumulator, residual, model) is fp32 in
 * HBM.  The O(k) region reduction, the global threshold and the reduced values
 * u are fp64, so for fp32-representable inputs every index set, threshold and
 * value equals the reference's fp64 result bit-for-bit.
 */
#ifndef OKT_H_
#define OKT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OKT_ABI_VERSION 1
#define OKT_MAX_WORLD 8

/* Status codes; one per reference exception type (include/oklab/errors.hpp). */
typedef enum okt_status {
  OKT_OK = 0,
  OKT_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  OKT_ERR_NUMERIC = 2,          /* NumericError (non-finite input / iterate) */
  OKT_ERR_PROTOCOL = 3,         /* ProtocolError (malformed exchange) */
  OKT_ERR_TRANSPORT = 4,        /* TransportError (world closed / peer failed) */
  OKT_ERR_CONFIG = 5,           /* ConfigError (non power-of-two P, P > 8) */
  OKT_ERR_CUDA = 6,             /* CUDA runtime failure */
  OKT_ERR_NCCL = 7,             /* NCCL failure */
  OKT_ERR_INTERNAL = 8,
  OKT_ERR_DECODE = 9            /* DecodeError: a malformed wire image */
} okt_status;

/* Ledger phases, numbered as oklab::Phase (include/oklab/transport.hpp:15-22). */
typedef enum okt_phase {
  OKT_PHASE_SPLIT = 0,
  OKT_PHASE_BALANCE = 1,
  OKT_PHASE_ALLGATHERV = 2,
  OKT_PHASE_CONSENSUS = 3,
  OKT_PHASE_DENSE = 4,
  OKT_PHASE_GATHER = 5,
  OKT_PHASE_COUNT = 6
} okt_phase;

typedef struct okt_world okt_world; /* shared by the P ranks of one process */
typedef struct okt_comm okt_comm;   /* one per rank */

/* TrafficLedger::Counters (transport.hpp:54-59) plus the bytes this
 * implementation actually moved over NVLink / NCCL for the phase. */
typedef struct okt_counters {
  uint64_t words_sent;
  uint64_t words_recv;
  uint64_t msgs_sent;
  uint64_t msgs_recv;
  uint64_t bytes_sent;
  uint64_t bytes_recv;
} okt_counters;

/* OkState (oktopk.hpp:30-35) + ThresholdState (sparse.hpp:56-63). */
typedef struct okt_state {
  double local_th;
  double global_th;
  uint32_t tau;       /* boundary period (reference default 64) */
  uint32_t tau_prime; /* threshold period (reference default 32) */
  int64_t last_local_eval;
  int64_t last_global_eval;
  int32_t regions;    /* RegionBoundaries::regions(): -1 when cuts are empty */
  uint32_t bucket_size; /* split-phase message granularity in entries (default 4) */
  uint64_t cuts[OKT_MAX_WORLD + 1];
  int64_t t;          /* last executed iteration */
} okt_state;

/* A COO sparse vector in device memory (library-owned, valid until the next
 * call on the same comm).  Indices strictly increasing, values fp64. */
typedef struct okt_sparse {
  const uint32_t* d_idx;
  const double* d_val;
  uint64_t nnz;
  uint64_t n;
} okt_sparse;

/* OkAllreduceResult (oktopk.hpp:95-99). */
typedef struct okt_result {
  okt_sparse u;               /* reduced, globally selected gradient */
  const uint32_t* d_indexes;  /* local selection ∩ u.indices, ascending */
  uint64_t n_indexes;
  uint64_t local_selected;    /* entries this rank selected by local_th */
} okt_result;

/* ---- library ---------------------------------------------------------- */
int okt_abi_version(void);
const char* okt_status_string(int status);
/* Message of the last failing call on this host thread. */
const char* okt_last_error(void);

/* ---- worlds and comms (WorkerCtx + Transport, transport.hpp:91-122) ---- */

/* Single-process world of P ranks driven by P host threads (the reference's
 * InprocTransport + run_ranks model).  devices[r] is rank r's CUDA device;
 * NULL puts every rank on the current device.  Exchanges are device-to-device
 * (NVLink peer) copies between the ranks' own buffers. */
int okt_world_create_local(okt_world** world, int P, const int* devices);
/* Transport::close(): wakes every rank blocked in an exchange; their calls and
 * all later collective calls fail with OKT_ERR_TRANSPORT. */
int okt_world_close(okt_world* world);
int okt_world_destroy(okt_world* world);
int okt_comm_init_local(okt_comm** comm, okt_world* world, int rank);

/* One process per GPU: ranks rendezvous through an NCCL unique id (128 bytes)
 * created by rank 0 and broadcast by the caller. */
int okt_nccl_unique_id(void* out, size_t len);
int okt_comm_init_nccl(okt_comm** comm, int rank, int P, int device,
                       const void* unique_id, size_t len);
int okt_comm_destroy(okt_comm* comm);
int okt_comm_info(const okt_comm* comm, int* rank, int* P, int* device);
/* Pre-size every per-rank buffer for gradients of length n_max (optional; the
 * library grows buffers on demand). */
int okt_comm_reserve(okt_comm* comm, size_t n_max);

/* ---- state and accounting --------------------------------------------- */
int okt_get_state(const okt_comm* comm, okt_state* out);
int okt_set_state(okt_comm* comm, const okt_state* in);
int okt_set_params(okt_comm* comm, uint32_t tau, uint32_t tau_prime,
                   uint32_t bucket_size);
int okt_ledger(const okt_comm* comm, int phase, okt_counters* out);
int okt_ledger_reset(okt_comm* comm);

/* ---- the hot path -------------------------------------------------------- */

/* ok_sparse_allreduce (oktopk.cpp:246-307): one Ok-Topk sparse allreduce of the
 * accumulated gradient d_acc (n fp32) at iteration t (1-based) keeping ~k
 * entries.  Collective.  `stream` may be NULL (the comm's own stream). */
int okt_sparse_allreduce(okt_comm* comm, const float* d_acc, size_t n,
                         int64_t t, size_t k, okt_result* out, void* stream);

/* Error-feedback residual (trainer.hpp:32-37), owned by the comm so a step
 * that fails leaves it untouched. */
int okt_residual_reset(okt_comm* comm, size_t n, const float* d_init,
                       void* stream);
int okt_residual(okt_comm* comm, float** d_eps, size_t* n);

/* oktopk_sgd_step (trainer.cpp:466-488) minus the problem evaluation: given the
 * local gradient d_grad, acc = eps + alpha*grad (fused with selection),
 * ok_sparse_allreduce(acc), eps = acc zeroed at indexes, w[i] -= u_i / P. */
int okt_sgd_step(okt_comm* comm, const float* d_grad, float* d_w, size_t n,
                 double alpha, int64_t t, size_t k, okt_result* out,
                 void* stream);

/* Asynchronous forms: enqueue the step on `stream` and return.  On the steady
 * device-driven iterations (one CUDA graph for P = 1, the NVLink window path
 * for P > 1) nothing waits on the host until okt_step_wait; other iterations
 * synchronise internally as the synchronous calls do.  okt_step_wait
 * finishes the step (state commit, result, error status).  Any other call on
 * the comm — including the next step — waits for a step still in flight. */
int okt_sparse_allreduce_async(okt_comm* comm, const float* d_acc, size_t n,
                               int64_t t, size_t k, void* stream);
int okt_sgd_step_async(okt_comm* comm, const float* d_grad, float* d_w,
                       size_t n, double alpha, int64_t t, size_t k,
                       void* stream);
int okt_step_wait(okt_comm* comm, okt_result* out);
/* Device-side barrier of all ranks, enqueued on `stream` (NULL = the comm's
 * stream): work enqueued after it starts on every GPU within one NVLink flag
 * latency of the others (collective; the host does not wait).  Without a
 * peer-mapped world it is a host barrier. */
int okt_device_barrier(okt_comm* comm, void* stream);

/* Host-buffer forms of the two hot entry points: the reference's own calling
 * convention (DenseGrad in, SparseGrad out, both in host memory).  The
 * gradient is copied host->device into a comm-owned buffer, the step runs, and
 * u is copied back into h_u_idx / h_u_val (capacity u_cap entries; a larger
 * result fails with OKT_ERR_INVALID_ARGUMENT after the step committed).
 * h_indexes (capacity u_cap) is optional. */
int okt_sparse_allreduce_host(okt_comm* comm, const float* h_acc, size_t n,
                              int64_t t, size_t k, uint32_t* h_u_idx,
                              double* h_u_val, uint32_t* h_indexes,
                              size_t u_cap, okt_result* out, void* stream);
int okt_sgd_step_host(okt_comm* comm, const float* h_grad, float* d_w,
                      size_t n, double alpha, int64_t t, size_t k,
                      uint32_t* h_u_idx, double* h_u_val, size_t u_cap,
                      okt_result* out, void* stream);

/* Plain copies on the comm's device (stream may be NULL = synchronous). */
int okt_memcpy_h2d(void* d_dst, const void* h_src, size_t bytes, void* stream);
int okt_memcpy_d2h(void* h_dst, const void* d_src, size_t bytes, void* stream);

/* ---- sub-phases (called directly by the reference's tests) -------------- */
int okt_th_re_evaluate_dense(okt_comm* comm, const float* d_g, size_t n,
                             size_t k, double* th, void* stream);
int okt_th_re_evaluate_sparse(okt_comm* comm, const double* d_val, size_t nnz,
                              size_t k, double* th, void* stream);
int okt_select_by_threshold(okt_comm* comm, const float* d_g, size_t n,
                            double th, okt_sparse* out, void* stream);
/* space_repartition(ctx, selected): d_sel_idx are the m selected indices of a
 * length-n vector; cuts_out receives P+1 boundaries (host memory). */
int okt_space_repartition(okt_comm* comm, const uint32_t* d_sel_idx, size_t m,
                          size_t n, uint64_t* cuts_out, void* stream);
/* split_and_reduce: region = this rank's reduced region (fp64), local = the
 * local selection (indices + fp64 values). */
int okt_split_and_reduce(okt_comm* comm, const float* d_g, size_t n,
                         double local_th, const uint64_t* cuts,
                         uint32_t bucket_size, okt_sparse* region,
                         okt_sparse* local, void* stream);
int okt_balance_and_allgatherv(okt_comm* comm, const uint32_t* d_idx,
                               const double* d_val, size_t nnz, size_t n,
                               double global_th, okt_sparse* u, void* stream);

/* ---- Table-1 baseline ------------------------------------------------------
 * topka_allreduce(ctx, g, k) (collectives.cpp:152-159): exact local top-k of
 * the fp32 gradient (magnitude-descending, ties toward the smaller index),
 * allgathered and summed in the reference's stride-doubling order (fp64).
 * 1 <= k <= n (OKT_ERR_INVALID_ARGUMENT otherwise); a non-finite gradient
 * fails with OKT_ERR_NUMERIC on its rank and OKT_ERR_TRANSPORT on the others.
 * `out` points into comm-owned device memory valid until the next call.
 * The other Table-1 baselines follow the same contract:
 *   gtopk_allreduce   collectives.cpp:300-325  log2 P pairwise merge + top-k rounds
 *   topkdsa_allreduce collectives.cpp:184-297  reduce-scatter with the dense switch,
 *                                              then allgatherv of the segments
 *   gaussiank_allreduce collectives.cpp:342-352 Gaussian-fit threshold (0.9
 *                     rescaling when scale_to_floor), select, allgatherv, sum
 * okt_gaussiank_threshold returns gaussian_threshold (scale_to_floor = 0, raw)
 * or gaussiank_scaled_threshold (1); the fp64 moments come from a tree
 * reduction, within a few ulp of the reference's sequential sums.  Zero-variance
 * input fails with OKT_ERR_NUMERIC ("DegenerateDistributionError"). */
int okt_topka_allreduce(okt_comm* comm, const float* d_g, size_t n, size_t k,
                        okt_sparse* out, void* stream);
/* dense_allreduce (collectives.cpp:89-150; collectives.hpp:28): the fp32
 * gradient widened to fp64 and summed by recursive halving / doubling in the
 * reference's order; *d_out = comm-owned fp64 vector of n, valid until the
 * next call.  Ranks with different n fail with OKT_ERR_PROTOCOL. */
int okt_dense_allreduce(okt_comm* comm, const float* d_g, size_t n, double** d_out,
                        void* stream);
int okt_gtopk_allreduce(okt_comm* comm, const float* d_g, size_t n, size_t k,
                        okt_sparse* out, void* stream);
int okt_topkdsa_allreduce(okt_comm* comm, const float* d_g, size_t n, size_t k,
                          okt_sparse* out, void* stream);
int okt_gaussiank_threshold(okt_comm* comm, const float* d_g, size_t n, size_t k,
                            int scale_to_floor, double* th, void* stream);
int okt_gaussiank_allreduce(okt_comm* comm, const float* d_g, size_t n, size_t k,
                            int scale_to_floor, okt_sparse* out, void* stream);

/* ---- host planning (pure functions, no GPU) ------------------------------
 * The exchange plans every rank derives from the sizes it already agreed on;
 * the device orchestration uses the same code.  Exported so the multi-rank
 * planning can be exercised on CPU ranks. */
typedef struct okt_piece {
  int32_t peer;
  uint64_t begin; /* range of the rank-concatenated survivor stream */
  uint64_t end;
} okt_piece;
enum okt_plan_kind {
  OKT_PLAN_SPLIT = 0,         /* sizes: P x P send counts, row = sender */
  OKT_PLAN_ALLGATHERV = 1,    /* sizes: P part sizes */
  OKT_PLAN_AVG = 2,           /* small_allreduce_avg of `len` reals */
  OKT_PLAN_ALLGATHER_U32 = 3, /* small_allgather_u32 of one word */
  OKT_PLAN_BALANCE = 4        /* sizes: P survivor counts */
};
/* space_repartition consensus (oktopk.cpp:51-61): proposals is P x (P+1). */
int okt_plan_cuts(const uint64_t* proposals, int P, uint64_t n, uint64_t* cuts);
/* balance_and_allgatherv's plan (oktopk.cpp:172-231); arrays hold <= P. */
int okt_plan_balance(int rank, int P, const uint64_t* sizes, int* balanced,
                     okt_piece* sends, int* nsends, okt_piece* recvs,
                     int* nrecvs, okt_piece* own, uint64_t* part_off,
                     uint64_t* part_sz);
/* Ledger words / messages the reference's transport credits for one phase. */
int okt_plan_ledger(int rank, int P, int kind, const uint64_t* sizes,
                    uint64_t len, uint32_t bucket, okt_counters* out);

/* ---- instrumentation ------------------------------------------------------ */
enum okt_timer {
  OKT_T_SELECT = 0,   /* K1 fused accumulate/select/compact */
  OKT_T_THRESHOLD,    /* K2 radix select of local_th */
  OKT_T_SPLIT,        /* counts exchange + slice exchange */
  OKT_T_MERGE,        /* K3 region merge */
  OKT_T_GLOBAL,       /* K4 global threshold refresh + survivor select */
  OKT_T_ALLGATHER,    /* K5/K6 balance + allgatherv */
  OKT_T_APPLY,        /* K7 residual / model scatter */
  OKT_T_STEP,         /* whole call */
  OKT_T_K1,           /* the K1 streaming kernel alone (phase A) */
  OKT_T_COUNT
};
/* When on, the library records CUDA events around each phase on its stream
 * and accumulates the elapsed device time. */
int okt_set_profiling(okt_comm* comm, int on);
int okt_phase_times(okt_comm* comm, double* ms_out /* OKT_T_COUNT */,
                    uint64_t* calls_out /* OKT_T_COUNT, nullable */);
/* Algorithmic HBM bytes the timed phases were charged. */
int okt_phase_bytes(okt_comm* comm, double* bytes_out /* OKT_T_COUNT */);
int okt_reset_phase_times(okt_comm* comm);
/* Number of kernels this comm has launched since creation. */
int okt_kernel_launches(const okt_comm* comm, uint64_t* out);
/* Diagnostics: per-CTA %globaltimer stamps (ns) of the last graph step,
 * [7 kinds: K1, merge, compact (P = 1), pull 0, pull 1, L publish, survivor
 * publish] x [2048 CTAs] x [start, after waits, end, extra].  Recorded only
 * when the comm was created with OKT_P2P_TRACE in the environment (else
 * OKT_ERR_CONFIG). */
int okt_debug_p2p_trace(okt_comm* comm, uint64_t* out, size_t n_words);

/* ---- COO wire codec (proj/core/src/sparse.cpp:275-312) ----------------------
 * The reference's wire image of a SparseGrad: [nnz u32][indices u32 x nnz]
 * [values f32 x nnz], little endian, 4 + 8 nnz bytes.  Device buffers, on the
 * current device; d_out / d_in 4-byte aligned.  Encode rounds each fp64 value
 * to fp32 (round to nearest).  Decode checks what wire_decode checks — header
 * present, length 4 + 8 nnz, every index < n and strictly increasing — and
 * returns OKT_ERR_DECODE otherwise (also when nnz > cap); *nnz_out is set on
 * success. */
int okt_wire_encode(const uint32_t* d_idx, const double* d_val, size_t nnz, void* d_out, void* stream);
int okt_wire_decode(const void* d_in, size_t bytes, size_t n, uint32_t* d_idx, double* d_val, size_t cap,
                    size_t* nnz_out, void* stream);

/* ---- seeded input generators (bit-exact ports of the reference's rng.hpp
 * streams, rounded to fp32; not on the hot path) ---------------------------- */
/* random_dense (proj/tests/test_util.hpp:135-140). */
int okt_gen_random_dense(float* d_out, size_t n, uint64_t seed, void* stream);
/* drifting_gradient_process (proj/core/src/trainer.cpp:338-388). */
int okt_gen_drift(float* d_out, size_t n, int64_t t, uint64_t seed,
                  uint64_t rank_key, int fixed_positions, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* OKT_H_ */
