// The reference's own acceptance gate (proj/tests/acceptance.cpp, compiled
// from where it lies under /root/reference) with its two Ok-Topk entry points
// rerouted to the B200 library.  The link wraps oklab::ok_sparse_allreduce
// and oklab::oktopk_sgd_step (-Wl,--wrap, see oracle/Makefile), so every call
// the reference's harness (run_experiment, harness.cpp:441-444) and the gate
// itself (acceptance.cpp:125) make into them lands in okt_oklab:: — the
// integration a reference maintainer gets from include/okt_oklab.hpp
// (INTEGRATION.md §2), exercised by the reference's own criteria.
#include "oklab/oktopk.hpp"
#include "oklab/trainer.hpp"
#include "okt_oklab.hpp"

extern "C" {
// oklab::ok_sparse_allreduce(WorkerCtx const&, OkState&, DenseGrad const&, long, unsigned long)
oklab::OkAllreduceResult __wrap__ZN5oklab19ok_sparse_allreduceERKNS_9WorkerCtxERNS_7OkStateERKNS_9DenseGradElm(
    const oklab::WorkerCtx& ctx, oklab::OkState& state, const oklab::DenseGrad& g, std::int64_t t, std::size_t k) {
  return okt_oklab::ok_sparse_allreduce(ctx, state, g, t, k);
}
// oklab::oktopk_sgd_step(WorkerCtx const&, ModelState&, Residual&, Problem const&, unsigned long, OkState&, XiProbe*)
oklab::StepOutcome
__wrap__ZN5oklab15oktopk_sgd_stepERKNS_9WorkerCtxERNS_10ModelStateERNS_8ResidualERKNS_7ProblemEmRNS_7OkStateEPNS_7XiProbeE(
    const oklab::WorkerCtx& ctx, oklab::ModelState& model, oklab::Residual& residual, const oklab::Problem& problem,
    std::size_t k, oklab::OkState& ok, oklab::XiProbe* probe) {
  return okt_oklab::oktopk_sgd_step(ctx, model, residual, problem, k, ok, probe);
}
}
