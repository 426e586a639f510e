/*
 * okt_oracle.h — CPU restatement of the reference's Ok-Topk hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests compare the
 * CUDA library against; nothing in the product (libokt.so, paper_2201_07598_b200/)
 * links, imports or calls it.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may use it.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/proj) in plain C99, fp64 throughout, with all P ranks
 * simulated in lockstep (the reference runs them as threads exchanging
 * messages; every exchange on this path is deterministic, so a central
 * simulation produces the same per-rank results and ledger counters).
 *
 * Pinning: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer tests (tests/test_oktopk.cpp,
 * tests/test_sparse_core.cpp, acceptance.cpp criteria 1/2/8) and, when
 * oracle/_ref/libokref.so is built, against the reference itself on random
 * instances; tests/golden/ holds vectors produced by the reference.
 */
#ifndef OKT_ORACLE_H_
#define OKT_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_P 8
#define ORC_PHASES 6

typedef struct orc_state {
  double local_th, global_th;
  uint32_t tau, tau_prime;
  int64_t last_local_eval, last_global_eval;
  int32_t regions; /* -1: empty cuts */
  uint32_t bucket_size;
  uint64_t cuts[ORC_MAX_P + 1];
  int64_t t;
} orc_state;

typedef struct orc_counters {
  uint64_t words_sent, words_recv, msgs_sent, msgs_recv;
} orc_counters;

/* rng.hpp:11-49 and tests/test_util.hpp:135-153 */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_mix64(uint64_t a, uint64_t b);
void orc_random_dense(uint64_t seed, size_t n, double* out);
void orc_random_int_dense(uint64_t seed, size_t n, int hi, double* out);
/* trainer.cpp:338-388 drifting_gradient_process */
int orc_drift(int64_t t, uint64_t seed, size_t n, uint64_t rank_key, int fixed_positions, double* out);

void orc_state_init(orc_state* s);

/* oktopk.cpp:12-26 -> sparse.cpp:43-80: the min(k, count)-th largest |v|. */
double orc_kth_largest_mag(const double* v, size_t count, size_t k);
/* sparse.cpp:94-120: {i : |g_i| >= th}; returns the count. */
size_t orc_select(const double* g, size_t n, double th, uint32_t* idx, double* val);
/* collectives.cpp:79-87 */
void orc_equal_slice_ends(uint64_t n, int P, uint64_t* ends);
/* sparse.cpp:206-257: stride-doubling union sum of P sorted parts; returns nnz. */
size_t orc_sparse_sum(int P, const uint32_t* const* idx, const double* const* val, const size_t* nnz,
                      uint32_t* out_idx, double* out_val);
/* topk_exact (sparse.cpp:43-80) of a dense vector: the k largest magnitudes,
 * ties toward the smaller index, returned in coordinate order; 1 <= k <= n. */
size_t orc_topk_exact(const double* g, size_t n, size_t k, uint32_t* idx, double* val);
/* topka_allreduce (collectives.cpp:152-159) of P dense vectors: sparse_sum of
 * the P exact top-k parts; out holds up to P*k entries. */
size_t orc_topka_allreduce(int P, const double* const* g, size_t n, size_t k, uint32_t* out_idx,
                           double* out_val);
/* dense_allreduce (collectives.cpp:89-150): rank 0's fp64 sum in out (n). */
void orc_dense_allreduce(int P, const double* const* g, size_t n, double* out, orc_counters* ledger);
/* gtopk_allreduce (collectives.cpp:300-325) / topkdsa_allreduce (:184-297):
 * rank 0's result (all ranks agree); ledger P*6 counters or NULL. */
size_t orc_gtopk_allreduce(int P, const double* const* g, size_t n, size_t k, uint32_t* out_idx, double* out_val,
                           orc_counters* ledger);
size_t orc_topkdsa_allreduce(int P, const double* const* g, size_t n, size_t k, uint32_t* out_idx, double* out_val,
                             orc_counters* ledger);
/* gaussian_threshold / gaussiank_scaled_threshold (sparse.cpp:167-188,
 * collectives.cpp:327-340); NAN for n < 2, k outside [1, n] or zero variance. */
double orc_inverse_normal_cdf(double p);
double orc_gaussian_threshold(const double* g, size_t n, size_t k, int scale_to_floor);
size_t orc_gaussiank_allreduce(int P, const double* const* g, size_t n, size_t k, int scale_to_floor,
                               uint32_t* out_idx, double* out_val, orc_counters* ledger);
/* oktopk.cpp:28-61 for all ranks: cuts from each rank's selected indices. */
void orc_space_repartition(int P, const uint32_t* const* sel, const size_t* m, uint64_t n,
                           uint64_t* cuts, orc_counters* ledger /* P*6, may be NULL */);

/* ok_sparse_allreduce (oktopk.cpp:246-307) for all P ranks.
 *   g[r]       rank r's accumulated gradient (n doubles)
 *   st[r]      rank r's OkState, updated in place
 *   ledger     P*6 counters (rank-major), accumulated
 *   u_idx/u_val  capacity n; *U receives |u| (identical on all ranks)
 *   indexes[r] capacity n; n_indexes[r]; local_selected[r]
 * Returns 0, -1 (invalid_argument), -2 (NumericError), -5 (ConfigError). */
int orc_ok_sparse_allreduce(int P, orc_state* st, const double* const* g, size_t n, int64_t t, size_t k,
                            orc_counters* ledger, uint32_t* u_idx, double* u_val, size_t* U,
                            uint32_t* const* indexes, size_t* n_indexes, size_t* local_selected);

/* oktopk_sgd_step (trainer.cpp:466-488) minus the problem: for all ranks,
 * acc = eps + alpha*grad; allreduce; eps = acc zeroed at indexes; w -= u/P. */
int orc_sgd_step(int P, orc_state* st, const double* const* grad, double* const* eps, double* const* w,
                 size_t n, double alpha, int64_t t, size_t k, orc_counters* ledger, uint32_t* u_idx,
                 double* u_val, size_t* U);

/* COO wire codec (proj/core/src/sparse.cpp:275-312): [nnz u32][indices u32 *
 * nnz][values f32 * nnz], little endian.  encode writes 4 + 8 nnz bytes;
 * decode returns 0, or 1 for a malformed buffer (the reference's DecodeError):
 * short header, length not 4 + 8 nnz, an index >= n, indices not strictly
 * increasing. */
void orc_wire_encode(const uint32_t* idx, const double* val, size_t nnz, uint8_t* out);
int orc_wire_decode(const uint8_t* in, size_t bytes, size_t n, uint32_t* idx, double* val, size_t* nnz);

#ifdef __cplusplus
}
#endif

#endif
