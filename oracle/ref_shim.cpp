// ref_shim.cpp — extern "C" wrapper around the REFERENCE implementation.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together
// with the reference's own sources (/root/reference/proj/core/src/*.cpp, used
// in place, never copied) into oracle/_ref/libokref.so.  It lets the tests pin
// the C restatement (okt_oracle.c) against the real reference and lets
// bench.py time the reference's CPU path (`--impl reference`, cpu_baseline).
//
// The ranks are threads over the reference's InprocTransport, exactly as the
// reference's own tests run them (proj/tests/test_util.hpp:22-76).
#include <pthread.h>
#include <sched.h>

#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <span>
#include <thread>
#include <vector>

#include "oklab/collectives.hpp"
#include "oklab/errors.hpp"
#include "oklab/inproc.hpp"
#include "oklab/oktopk.hpp"
#include "oklab/sparse.hpp"
#include "oklab/trainer.hpp"
#include "oklab/transport.hpp"

using namespace oklab;

extern "C" {

struct okref_state {  // layout of orc_state / okt_state
  double local_th, global_th;
  uint32_t tau, tau_prime;
  int64_t last_local_eval, last_global_eval;
  int32_t regions;
  uint32_t bucket_size;
  uint64_t cuts[9];
  int64_t t;
};

struct okref_counters {
  uint64_t words_sent, words_recv, msgs_sent, msgs_recv;
};

}  // extern "C"

namespace {

OkState to_ref(const okref_state& s) {
  OkState o;
  o.th.local_th = s.local_th;
  o.th.global_th = s.global_th;
  o.th.tau = s.tau;
  o.th.tau_prime = s.tau_prime;
  o.th.last_local_eval = s.last_local_eval;
  o.th.last_global_eval = s.last_global_eval;
  if (s.regions >= 0) o.bounds.cuts.assign(s.cuts, s.cuts + s.regions + 1);
  o.t = s.t;
  o.bucket_size = s.bucket_size;
  return o;
}

void from_ref(const OkState& o, okref_state& s) {
  s.local_th = o.th.local_th;
  s.global_th = o.th.global_th;
  s.tau = o.th.tau;
  s.tau_prime = o.th.tau_prime;
  s.last_local_eval = o.th.last_local_eval;
  s.last_global_eval = o.th.last_global_eval;
  s.regions = o.bounds.regions();
  for (int i = 0; i <= s.regions && i < 9; ++i) s.cuts[i] = o.bounds.cuts[i];
  s.t = o.t;
  s.bucket_size = o.bucket_size;
}

int code_of(std::exception_ptr e, char* err, size_t errlen) {
  try {
    std::rethrow_exception(e);
  } catch (const std::invalid_argument& x) {
    std::snprintf(err, errlen, "%s", x.what());
    return 1;
  } catch (const NumericError& x) {
    std::snprintf(err, errlen, "%s", x.what());
    return 2;
  } catch (const ProtocolError& x) {
    std::snprintf(err, errlen, "%s", x.what());
    return 3;
  } catch (const TransportError& x) {
    std::snprintf(err, errlen, "%s", x.what());
    return 4;
  } catch (const ConfigError& x) {
    std::snprintf(err, errlen, "%s", x.what());
    return 5;
  } catch (const std::exception& x) {
    std::snprintf(err, errlen, "%s", x.what());
    return 8;
  }
}

// run_ranks (test_util.hpp:38-76) with root-cause selection.
template <typename F>
int run_ranks(InprocTransport& tr, int P, F body, char* err, size_t errlen) {
  std::vector<std::exception_ptr> errs(P);
  {
    std::vector<std::jthread> th;
    for (int r = 0; r < P; ++r)
      th.emplace_back([&, r] {
        try {
          body(r);
        } catch (...) {
          errs[r] = std::current_exception();
          tr.close();
        }
      });
  }
  std::exception_ptr first, root;
  for (auto& e : errs) {
    if (!e) continue;
    if (!first) first = e;
    if (!root) {
      try {
        std::rethrow_exception(e);
      } catch (const TransportError&) {
      } catch (...) {
        root = e;
      }
    }
  }
  if (root) return code_of(root, err, errlen);
  if (first) return code_of(first, err, errlen);
  return 0;
}

void pin_to_core(int core) {
  cpu_set_t set;
  CPU_ZERO(&set);
  CPU_SET(core, &set);
  pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
}

}  // namespace

extern "C" {

// One oklab::ok_sparse_allreduce on P rank threads.
int okref_allreduce(int P, const double* const* g, size_t n, int64_t t, size_t k, okref_state* st,
                    okref_counters* ledger, uint32_t* u_idx, double* u_val, size_t* U,
                    uint32_t* const* indexes, size_t* n_indexes, size_t* local_selected, char* err,
                    size_t errlen) {
  InprocTransport tr(P, 64);
  TrafficLedger led(P);
  std::vector<OkAllreduceResult> res(P);
  std::vector<OkState> states(P);
  for (int r = 0; r < P; ++r) states[r] = to_ref(st[r]);
  const int rc = run_ranks(
      tr, P,
      [&](int r) {
        WorkerCtx ctx{r, P, &tr, &led};
        DenseGrad dg(std::vector<double>(g[r], g[r] + n));
        res[r] = ok_sparse_allreduce(ctx, states[r], dg, t, k);
      },
      err, errlen);
  for (int r = 0; r < P; ++r) {
    from_ref(states[r], st[r]);
    for (int ph = 0; ph < kPhaseCount; ++ph) {
      const auto& c = led.at(r, static_cast<Phase>(ph));
      okref_counters& o = ledger[r * kPhaseCount + ph];
      o.words_sent += c.words_sent;
      o.words_recv += c.words_recv;
      o.msgs_sent += c.msgs_sent;
      o.msgs_recv += c.msgs_recv;
    }
  }
  if (rc) return rc;
  *U = res[0].u.nnz();
  std::memcpy(u_idx, res[0].u.indices.data(), res[0].u.nnz() * sizeof(uint32_t));
  std::memcpy(u_val, res[0].u.values.data(), res[0].u.nnz() * sizeof(double));
  for (int r = 0; r < P; ++r) {
    if (res[r].u != res[0].u) {
      std::snprintf(err, errlen, "ranks disagree on u");
      return 8;
    }
    n_indexes[r] = res[r].indexes.size();
    if (indexes && indexes[r])
      std::memcpy(indexes[r], res[r].indexes.data(), res[r].indexes.size() * sizeof(uint32_t));
    local_selected[r] = res[r].local_selected;
  }
  return 0;
}

double okref_th_re_evaluate_dense(const double* g, size_t n, size_t k) {
  return th_re_evaluate(DenseGrad(std::vector<double>(g, g + n)), k);
}

// drifting_gradient_process rounded to fp32 (the inputs the GPU run sees).
void okref_drift_f32(int64_t t, uint64_t seed, size_t n, uint64_t rank_key, double* out) {
  DriftOptions o;
  o.rank_key = rank_key;
  DenseGrad g = drifting_gradient_process(t, seed, n, o);
  for (size_t i = 0; i < n; ++i) out[i] = double(float(g[i]));
}

// Times the reference's Ok-Topk EF-SGD step (trainer.cpp:466-488 minus the
// problem evaluation: all_finite(grad), acc = eps + alpha*grad,
// ok_sparse_allreduce, eps = acc zeroed at indexes, w -= u/P, all_finite(w))
// on P rank threads over InprocTransport, one core each when pin != 0.
// Inputs: drifting_gradient_process(t, seed, n, rank_key = r+1) rounded to
// fp32, generated outside the timed region.  ms[i] = wall time of iteration
// warmup+i between two barriers (the max over ranks).
int okref_bench_sgd(int P, size_t n, size_t k, int warmup, int iters, uint32_t tau, uint32_t tau_prime,
                    uint32_t bucket, double alpha, uint64_t seed, int pin, double* ms, char* err,
                    size_t errlen) {
  InprocTransport tr(P, 64);
  TrafficLedger led(P);
  std::barrier sync_point(P);
  std::vector<std::chrono::steady_clock::time_point> t0(warmup + iters), t1(warmup + iters);
  const int ncpu = int(std::thread::hardware_concurrency());
  const int rc = run_ranks(
      tr, P,
      [&](int r) {
        if (pin && P <= ncpu) pin_to_core(r);
        WorkerCtx ctx{r, P, &tr, &led};
        OkState ok;
        ok.th.tau = tau;
        ok.th.tau_prime = tau_prime;
        ok.bucket_size = bucket;
        DenseGrad eps(n), w(n);
        DriftOptions o;
        o.rank_key = uint64_t(r) + 1;
        for (int it = 0; it < warmup + iters; ++it) {
          const int64_t t = it + 1;
          DenseGrad grad = drifting_gradient_process(t, seed, n, o);
          for (double& v : grad.values) v = double(float(v));
          sync_point.arrive_and_wait();
          if (r == 0) t0[it] = std::chrono::steady_clock::now();
          if (!grad.all_finite()) throw NumericError("oktopk_sgd_step: non-finite gradient");
          DenseGrad acc(n);
          for (size_t i = 0; i < n; ++i) acc[i] = eps[i] + alpha * grad[i];
          OkAllreduceResult res = ok_sparse_allreduce(ctx, ok, acc, t, k);
          eps = std::move(acc);
          for (Index idx : res.indexes) eps[idx] = 0.0;
          const double p = double(P);
          for (size_t i = 0; i < res.u.nnz(); ++i) w[res.u.indices[i]] -= res.u.values[i] / p;
          if (!w.all_finite()) throw NumericError("oktopk_sgd_step: non-finite iterate");
          sync_point.arrive_and_wait();
          if (r == 0) t1[it] = std::chrono::steady_clock::now();
        }
      },
      err, errlen);
  if (rc) return rc;
  for (int i = 0; i < iters; ++i)
    ms[i] = std::chrono::duration<double, std::milli>(t1[warmup + i] - t0[warmup + i]).count();
  return 0;
}

// The reference's COO wire codec (sparse.cpp:275-312) on flat buffers.
int okref_wire_encode(const uint32_t* idx, const double* val, size_t nnz, size_t n, uint8_t* out) {
  oklab::SparseGrad sg(n);
  sg.indices.assign(idx, idx + nnz);
  sg.values.assign(val, val + nnz);
  const std::vector<std::uint8_t> b = oklab::wire_encode(sg);
  std::memcpy(out, b.data(), b.size());
  return 0;
}
int okref_wire_decode(const uint8_t* in, size_t bytes, size_t n, uint32_t* idx, double* val, size_t* nnz) {
  try {
    const oklab::SparseGrad sg = oklab::wire_decode(std::span<const std::uint8_t>(in, bytes), n);
    std::copy(sg.indices.begin(), sg.indices.end(), idx);
    std::copy(sg.values.begin(), sg.values.end(), val);
    *nnz = sg.nnz();
    return 0;
  } catch (const oklab::DecodeError&) {
    return 1;
  }
}

// One oklab::topka_allreduce on P rank threads (collectives.cpp:152-159).
int okref_topka(int P, const double* const* g, size_t n, size_t k, uint32_t* u_idx, double* u_val, size_t* U,
                char* err, size_t errlen) {
  InprocTransport tr(P, 64);
  TrafficLedger led(P);
  std::vector<SparseGrad> res(P);
  const int rc = run_ranks(
      tr, P,
      [&](int r) {
        WorkerCtx ctx{r, P, &tr, &led};
        DenseGrad dg(std::vector<double>(g[r], g[r] + n));
        res[r] = topka_allreduce(ctx, dg, k);
      },
      err, errlen);
  if (rc) return rc;
  for (int r = 1; r < P; ++r)
    if (res[r] != res[0]) {
      std::snprintf(err, errlen, "ranks disagree on u");
      return 8;
    }
  *U = res[0].nnz();
  std::memcpy(u_idx, res[0].indices.data(), res[0].nnz() * sizeof(uint32_t));
  std::memcpy(u_val, res[0].values.data(), res[0].nnz() * sizeof(double));
  return 0;
}

// gtopk (0) / topkdsa (1) / gaussiank (2, scaled) / gaussiank (3, raw) on P rank threads.
int okref_baseline(int which, int P, const double* const* g, size_t n, size_t k, uint32_t* u_idx, double* u_val,
                   size_t* U, okref_counters* ledger, char* err, size_t errlen) {
  InprocTransport tr(P, 64);
  TrafficLedger led(P);
  std::vector<SparseGrad> res(P);
  const int rc = run_ranks(
      tr, P,
      [&](int r) {
        WorkerCtx ctx{r, P, &tr, &led};
        DenseGrad dg(std::vector<double>(g[r], g[r] + n));
        if (which == 0) res[r] = gtopk_allreduce(ctx, dg, k);
        else if (which == 1) res[r] = topkdsa_allreduce(ctx, dg, k);
        else res[r] = gaussiank_allreduce(ctx, dg, k, GaussiankOptions{which == 2});
      },
      err, errlen);
  for (int r = 0; r < P && ledger; ++r)
    for (int ph = 0; ph < kPhaseCount; ++ph) {
      const auto& c = led.at(r, static_cast<Phase>(ph));
      okref_counters& o = ledger[r * kPhaseCount + ph];
      o.words_sent += c.words_sent;
      o.words_recv += c.words_recv;
      o.msgs_sent += c.msgs_sent;
      o.msgs_recv += c.msgs_recv;
    }
  if (rc) return rc;
  for (int r = 1; r < P; ++r)
    if (res[r] != res[0]) {
      std::snprintf(err, errlen, "ranks disagree on u");
      return 8;
    }
  *U = res[0].nnz();
  std::memcpy(u_idx, res[0].indices.data(), res[0].nnz() * sizeof(uint32_t));
  std::memcpy(u_val, res[0].values.data(), res[0].nnz() * sizeof(double));
  return 0;
}

double okref_gaussian_threshold(const double* g, size_t n, size_t k, int scale_to_floor) {
  DenseGrad dg(std::vector<double>(g, g + n));
  return scale_to_floor ? gaussiank_scaled_threshold(dg, k) : gaussian_threshold(dg, k);
}

// One oklab::dense_allreduce on P rank threads.
int okref_dense(int P, const double* const* g, size_t n, double* out, okref_counters* ledger, char* err,
                size_t errlen) {
  InprocTransport tr(P, 64);
  TrafficLedger led(P);
  std::vector<DenseGrad> res(P);
  const int rc = run_ranks(
      tr, P,
      [&](int r) {
        WorkerCtx ctx{r, P, &tr, &led};
        res[r] = dense_allreduce(ctx, DenseGrad(std::vector<double>(g[r], g[r] + n)));
      },
      err, errlen);
  for (int r = 0; r < P && ledger; ++r)
    for (int ph = 0; ph < kPhaseCount; ++ph) {
      const auto& c = led.at(r, static_cast<Phase>(ph));
      okref_counters& o = ledger[r * kPhaseCount + ph];
      o.words_sent += c.words_sent;
      o.words_recv += c.words_recv;
      o.msgs_sent += c.msgs_sent;
      o.msgs_recv += c.msgs_recv;
    }
  if (rc) return rc;
  for (int r = 1; r < P; ++r)
    if (res[r].values != res[0].values) {
      std::snprintf(err, errlen, "ranks disagree");
      return 8;
    }
  std::memcpy(out, res[0].values.data(), n * sizeof(double));
  return 0;
}

}  // extern "C"
