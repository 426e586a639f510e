// okt_oklab.hpp — the reference-side binding: oklab's own C++ signatures for
// the Ok-Topk hot path, implemented over the C-ABI of include/okt.h.
//
// A maintainer of the reference swaps the CPU path for the B200 one by
// including this header (after the oklab headers) and calling okt_oklab::
// instead of oklab:: — same arguments, same results, same exceptions, same
// ledger credits:
//
//   oklab::ok_sparse_allreduce(ctx, state, g, t, k)      (oktopk.hpp:118-120)
//   oklab::oktopk_sgd_step(ctx, model, res, problem, k, ok) (trainer.hpp:149-152)
//   oklab::topka_allreduce / topkdsa_allreduce / gtopk_allreduce /
//   gaussiank_allreduce (collectives.hpp:33-71, the Table-1 baselines)
//
// Ranks stay threads of one process over one oklab::Transport (the reference's
// run_ranks model): the first call of each rank binds it to an okt_comm of a
// single-process okt_world keyed by the Transport, on device
// (rank % device_count).  Values cross the boundary as fp32 (exact for
// fp32-representable inputs) and come back as fp64.  Link with libokt.so.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "oklab/collectives.hpp"
#include "oklab/errors.hpp"
#include "oklab/oktopk.hpp"
#include "oklab/sparse.hpp"
#include "oklab/trainer.hpp"
#include "oklab/transport.hpp"
#include "okt.h"

namespace okt_oklab {

namespace detail {

[[noreturn]] inline void raise(int status) {
  const std::string msg = okt_last_error();
  switch (status) {
    case OKT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case OKT_ERR_NUMERIC: throw oklab::NumericError(msg);
    case OKT_ERR_PROTOCOL: throw oklab::ProtocolError(msg);
    case OKT_ERR_TRANSPORT: throw oklab::TransportError(msg);
    case OKT_ERR_CONFIG: throw oklab::ConfigError(msg);
    default: throw std::runtime_error("okt: " + msg);
  }
}
inline void check(int status) {
  if (status != OKT_OK) raise(status);
}

struct Binding {
  int P = 0;
  okt_world* world = nullptr;
  std::vector<okt_comm*> comms;
  std::vector<okt_counters> seen;  // ledger already credited, per rank * phase
  ~Binding() {
    for (okt_comm* c : comms) okt_comm_destroy(c);
    if (world) okt_world_destroy(world);
  }
};

inline std::mutex& mu() {
  static std::mutex m;
  return m;
}
inline std::map<const oklab::Transport*, std::unique_ptr<Binding>>& bindings() {
  static std::map<const oklab::Transport*, std::unique_ptr<Binding>> b;
  return b;
}

inline okt_comm* comm_for(const oklab::WorkerCtx& ctx, Binding** out) {
  std::lock_guard<std::mutex> lk(mu());
  auto& slot = bindings()[ctx.transport];
  if (slot && slot->P != ctx.world) slot.reset();  // a new transport reused the address
  if (!slot) {
    slot.reset(new Binding());
    slot->P = ctx.world;
    int ndev = 1;
    cudaGetDeviceCount(&ndev);
    std::vector<int> dev(ctx.world);
    for (int r = 0; r < ctx.world; ++r) dev[r] = r % (ndev > 0 ? ndev : 1);
    check(okt_world_create_local(&slot->world, ctx.world, dev.data()));
    slot->comms.assign(ctx.world, nullptr);
    slot->seen.assign(size_t(ctx.world) * OKT_PHASE_COUNT, okt_counters{});
  }
  if (!slot->comms[ctx.rank]) check(okt_comm_init_local(&slot->comms[ctx.rank], slot->world, ctx.rank));
  *out = slot.get();
  return slot->comms[ctx.rank];
}

// Credit the caller's TrafficLedger with what the library accounted since the
// last call (one on_send / on_recv per message, like WorkerCtx::send / recv).
inline void credit(const oklab::WorkerCtx& ctx, Binding* b, okt_comm* c) {
  for (int ph = 0; ph < OKT_PHASE_COUNT; ++ph) {
    okt_counters now{};
    check(okt_ledger(c, ph, &now));
    okt_counters& was = b->seen[size_t(ctx.rank) * OKT_PHASE_COUNT + ph];
    const auto phase = static_cast<oklab::Phase>(ph);
    uint64_t msgs = now.msgs_sent - was.msgs_sent, words = now.words_sent - was.words_sent;
    for (uint64_t i = 0; i < msgs; ++i) ctx.ledger->on_send(ctx.rank, phase, i + 1 == msgs ? words : 0);
    msgs = now.msgs_recv - was.msgs_recv;
    words = now.words_recv - was.words_recv;
    for (uint64_t i = 0; i < msgs; ++i) ctx.ledger->on_recv(ctx.rank, phase, i + 1 == msgs ? words : 0);
    was = now;
  }
}

inline okt_state to_okt(const oklab::OkState& s) {
  okt_state o;
  std::memset(&o, 0, sizeof(o));
  o.local_th = s.th.local_th;
  o.global_th = s.th.global_th;
  o.tau = s.th.tau;
  o.tau_prime = s.th.tau_prime;
  o.last_local_eval = s.th.last_local_eval;
  o.last_global_eval = s.th.last_global_eval;
  o.regions = s.bounds.regions();
  for (int i = 0; i <= o.regions && i <= OKT_MAX_WORLD; ++i) o.cuts[i] = s.bounds.cuts[i];
  o.t = s.t;
  o.bucket_size = s.bucket_size;
  return o;
}

inline void from_okt(const okt_state& o, oklab::OkState& s) {
  s.th.local_th = o.local_th;
  s.th.global_th = o.global_th;
  s.th.tau = o.tau;
  s.th.tau_prime = o.tau_prime;
  s.th.last_local_eval = o.last_local_eval;
  s.th.last_global_eval = o.last_global_eval;
  s.bounds.cuts.assign(o.cuts, o.cuts + (o.regions >= 0 ? o.regions + 1 : 0));
  s.t = o.t;
  s.bucket_size = o.bucket_size;
}

inline oklab::OkAllreduceResult to_result(const okt_result& r, std::size_t n) {
  oklab::OkAllreduceResult out;
  out.u.n = n;
  out.u.indices.resize(r.u.nnz);
  out.u.values.resize(r.u.nnz);
  out.indexes.resize(r.n_indexes);
  if (r.u.nnz) {
    check(okt_memcpy_d2h(out.u.indices.data(), r.u.d_idx, 4 * r.u.nnz, nullptr));
    check(okt_memcpy_d2h(out.u.values.data(), r.u.d_val, 8 * r.u.nnz, nullptr));
  }
  if (r.n_indexes) check(okt_memcpy_d2h(out.indexes.data(), r.d_indexes, 4 * r.n_indexes, nullptr));
  out.local_selected = r.local_selected;
  return out;
}

inline oklab::SparseGrad to_sparse(const okt_sparse& u, std::size_t n) {
  oklab::SparseGrad out(n);
  out.indices.resize(u.nnz);
  out.values.resize(u.nnz);
  if (u.nnz) {
    check(okt_memcpy_d2h(out.indices.data(), u.d_idx, 4 * u.nnz, nullptr));
    check(okt_memcpy_d2h(out.values.data(), u.d_val, 8 * u.nnz, nullptr));
  }
  return out;
}

// One baseline call: the fp32 gradient staged on the rank's device, the
// collective, the ledger credit, the result back as fp64.
template <class F>
oklab::SparseGrad run_baseline(const oklab::WorkerCtx& ctx, const oklab::DenseGrad& g, F&& fn) {
  Binding* b = nullptr;
  okt_comm* c = comm_for(ctx, &b);
  int dev = 0;
  check(okt_comm_info(c, nullptr, nullptr, &dev));
  cudaSetDevice(dev);
  std::vector<float> gf(g.values.begin(), g.values.end());
  float* d_g = nullptr;
  if (!gf.empty() && cudaMalloc(&d_g, 4 * gf.size()) != cudaSuccess) raise(OKT_ERR_CUDA);
  struct Free {
    float* p;
    ~Free() { if (p) cudaFree(p); }
  } guard{d_g};
  if (!gf.empty()) check(okt_memcpy_h2d(d_g, gf.data(), 4 * gf.size(), nullptr));
  okt_sparse u{};
  const int rc = fn(c, d_g, gf.size(), &u);
  credit(ctx, b, c);
  if (rc != OKT_OK) raise(rc);
  return to_sparse(u, g.size());
}

}  // namespace detail

// Releases the device comms bound to `transport` (call before destroying it;
// otherwise a later transport allocated at the same address would inherit
// them).
inline void release(const oklab::Transport* transport) {
  std::lock_guard<std::mutex> lk(detail::mu());
  detail::bindings().erase(transport);
}

// Drop-in for oklab::ok_sparse_allreduce (oktopk.hpp:118-120).
inline oklab::OkAllreduceResult ok_sparse_allreduce(const oklab::WorkerCtx& ctx, oklab::OkState& state,
                                                    const oklab::DenseGrad& g, std::int64_t t, std::size_t k) {
  detail::Binding* b = nullptr;
  okt_comm* c = detail::comm_for(ctx, &b);
  okt_state s = detail::to_okt(state);
  detail::check(okt_set_state(c, &s));
  std::vector<float> gf(g.values.begin(), g.values.end());
  okt_result r{};
  const int rc = okt_sparse_allreduce_host(c, gf.empty() ? nullptr : gf.data(), gf.size(), t, k, nullptr, nullptr,
                                           nullptr, 0, &r, nullptr);
  detail::credit(ctx, b, c);
  if (rc != OKT_OK) detail::raise(rc);
  detail::check(okt_get_state(c, &s));
  detail::from_okt(s, state);
  return detail::to_result(r, g.size());
}

// Drop-in for oklab::oktopk_sgd_step (trainer.hpp:149-152).  The residual lives
// on the device between calls; Residual::eps is refreshed on every step.
inline oklab::StepOutcome oktopk_sgd_step(const oklab::WorkerCtx& ctx, oklab::ModelState& model,
                                          oklab::Residual& residual, const oklab::Problem& problem,
                                          std::size_t k, oklab::OkState& ok, oklab::XiProbe* probe = nullptr) {
  detail::Binding* b = nullptr;
  okt_comm* c = detail::comm_for(ctx, &b);
  const std::int64_t t = model.t + 1;
  const double alpha = model.lr.at(t);
  oklab::DenseGrad grad = problem.local_gradient(model.w, ctx.rank, ctx.world, t);
  const std::size_t n = grad.size();
  if (n != problem.dim() || !grad.all_finite())
    throw oklab::NumericError("oktopk_sgd_step: non-finite or misshaped gradient");
  if (probe != nullptr) {  // the accumulator as make_accumulator forms it (trainer.cpp:423-435, 471-474)
    probe->acc = oklab::DenseGrad(n);
    for (std::size_t i = 0; i < n; ++i) probe->acc[i] = residual.eps[i] + alpha * grad[i];
    probe->grad = grad;
  }
  // Residual and model to the device (fp32).
  std::vector<float> eps(residual.eps.values.begin(), residual.eps.values.end());
  std::vector<float> w(model.w.values.begin(), model.w.values.end()), gf(grad.values.begin(), grad.values.end());
  float* d_w = nullptr;
  float* d_eps0 = nullptr;
  detail::check(cudaMalloc(&d_w, 4 * n) == cudaSuccess ? OKT_OK : OKT_ERR_CUDA);
  detail::check(cudaMalloc(&d_eps0, 4 * n) == cudaSuccess ? OKT_OK : OKT_ERR_CUDA);
  detail::check(okt_memcpy_h2d(d_w, w.data(), 4 * n, nullptr));
  detail::check(okt_memcpy_h2d(d_eps0, eps.data(), 4 * n, nullptr));
  detail::check(okt_residual_reset(c, n, d_eps0, nullptr));
  okt_state s = detail::to_okt(ok);
  detail::check(okt_set_state(c, &s));
  okt_result r{};
  const int rc = okt_sgd_step_host(c, gf.data(), d_w, n, alpha, t, k, nullptr, nullptr, 0, &r, nullptr);
  detail::credit(ctx, b, c);
  if (rc != OKT_OK) {
    cudaFree(d_w);
    cudaFree(d_eps0);
    detail::raise(rc);
  }
  detail::check(okt_get_state(c, &s));
  detail::from_okt(s, ok);
  float* d_eps = nullptr;
  size_t en = 0;
  detail::check(okt_residual(c, &d_eps, &en));
  detail::check(okt_memcpy_d2h(eps.data(), d_eps, 4 * n, nullptr));
  detail::check(okt_memcpy_d2h(w.data(), d_w, 4 * n, nullptr));
  cudaFree(d_w);
  cudaFree(d_eps0);
  for (std::size_t i = 0; i < n; ++i) {
    residual.eps[i] = eps[i];
    model.w[i] = w[i];
  }
  model.t = t;
  oklab::StepOutcome out;
  out.objective = problem.objective(model.w, t);
  out.selected_local = r.local_selected;
  out.selected_global = r.u.nnz;
  return out;
}

// Drop-in for oklab::dense_allreduce (collectives.hpp:28).
inline oklab::DenseGrad dense_allreduce(const oklab::WorkerCtx& ctx, const oklab::DenseGrad& g) {
  detail::Binding* b = nullptr;
  okt_comm* c = detail::comm_for(ctx, &b);
  int dev = 0;
  detail::check(okt_comm_info(c, nullptr, nullptr, &dev));
  cudaSetDevice(dev);
  std::vector<float> gf(g.values.begin(), g.values.end());
  float* d_g = nullptr;
  if (!gf.empty() && cudaMalloc(&d_g, 4 * gf.size()) != cudaSuccess) detail::raise(OKT_ERR_CUDA);
  struct Free {
    float* p;
    ~Free() { if (p) cudaFree(p); }
  } guard{d_g};
  if (!gf.empty()) detail::check(okt_memcpy_h2d(d_g, gf.data(), 4 * gf.size(), nullptr));
  double* d_out = nullptr;
  const int rc = okt_dense_allreduce(c, d_g, gf.size(), &d_out, nullptr);
  detail::credit(ctx, b, c);
  if (rc != OKT_OK) detail::raise(rc);
  oklab::DenseGrad out(g.size());
  if (g.size()) detail::check(okt_memcpy_d2h(out.values.data(), d_out, 8 * g.size(), nullptr));
  return out;
}

// Drop-ins for the Table-1 baselines (collectives.hpp:33-71).
inline oklab::SparseGrad topka_allreduce(const oklab::WorkerCtx& ctx, const oklab::DenseGrad& g, std::size_t k) {
  return detail::run_baseline(ctx, g, [&](okt_comm* c, const float* d, std::size_t n, okt_sparse* u) {
    return okt_topka_allreduce(c, d, n, k, u, nullptr);
  });
}
inline oklab::SparseGrad gtopk_allreduce(const oklab::WorkerCtx& ctx, const oklab::DenseGrad& g, std::size_t k) {
  return detail::run_baseline(ctx, g, [&](okt_comm* c, const float* d, std::size_t n, okt_sparse* u) {
    return okt_gtopk_allreduce(c, d, n, k, u, nullptr);
  });
}
inline oklab::SparseGrad topkdsa_allreduce(const oklab::WorkerCtx& ctx, const oklab::DenseGrad& g, std::size_t k) {
  return detail::run_baseline(ctx, g, [&](okt_comm* c, const float* d, std::size_t n, okt_sparse* u) {
    return okt_topkdsa_allreduce(c, d, n, k, u, nullptr);
  });
}
inline oklab::SparseGrad gaussiank_allreduce(const oklab::WorkerCtx& ctx, const oklab::DenseGrad& g, std::size_t k,
                                             oklab::GaussiankOptions opts = {}) {
  return detail::run_baseline(ctx, g, [&](okt_comm* c, const float* d, std::size_t n, okt_sparse* u) {
    return okt_gaussiank_allreduce(c, d, n, k, opts.scale_to_floor ? 1 : 0, u, nullptr);
  });
}

}  // namespace okt_oklab
