// adapter_parity.cpp — the reference's own scenarios run twice: through
// oklab:: (the CPU reference, compiled from /root/reference) and through
// okt_oklab:: (include/okt_oklab.hpp over libokt.so on the GPU).  Every
// OkAllreduceResult, OkState and ledger row must be identical.
// Built by oracle/Makefile into oracle/_ref/adapter_parity; run by
// tests/test_gpu_adapter.py.  Exit code = number of mismatching scenarios.
#include <cmath>
#include <cstdio>
#include <functional>
#include <vector>

#include "okt_oklab.hpp"
#include "test_util.hpp"

using namespace oklab;
using oklab::test::World;
using oklab::test::run_ranks;

namespace {

DenseGrad f32(DenseGrad g) {
  for (double& v : g.values) v = double(float(v));
  return g;
}

bool same_ledger(const TrafficLedger& a, const TrafficLedger& b, int P) {
  for (int r = 0; r < P; ++r)
    for (int ph = 0; ph < kPhaseCount; ++ph) {
      const auto& x = a.at(r, Phase(ph));
      const auto& y = b.at(r, Phase(ph));
      if (x.words_sent != y.words_sent || x.words_recv != y.words_recv || x.msgs_sent != y.msgs_sent ||
          x.msgs_recv != y.msgs_recv)
        return false;
    }
  return true;
}

bool same_state(const OkState& a, const OkState& b) {
  return a.th.local_th == b.th.local_th && a.th.global_th == b.th.global_th &&
         a.th.last_local_eval == b.th.last_local_eval && a.th.last_global_eval == b.th.last_global_eval &&
         a.bounds.cuts == b.bounds.cuts && a.t == b.t;
}

// Runs `iters` iterations of ok_sparse_allreduce on both implementations.
int scenario(const char* name, int P, std::size_t n, std::size_t k, int iters, std::uint32_t tau,
             std::uint32_t tau_prime, std::uint32_t bucket,
             const std::function<DenseGrad(int, std::int64_t)>& input) {
  World wr(P), wg(P);
  std::vector<OkState> sr(P), sg(P);
  for (int r = 0; r < P; ++r) {
    sr[r].th.tau = sg[r].th.tau = tau;
    sr[r].th.tau_prime = sg[r].th.tau_prime = tau_prime;
    sr[r].bucket_size = sg[r].bucket_size = bucket;
  }
  for (std::int64_t t = 1; t <= iters; ++t) {
    std::vector<DenseGrad> in;
    for (int r = 0; r < P; ++r) in.push_back(f32(input(r, t)));
    auto ref = run_ranks(wr, [&](const WorkerCtx& ctx) {
      return oklab::ok_sparse_allreduce(ctx, sr[ctx.rank], in[ctx.rank], t, k);
    });
    auto gpu = run_ranks(wg, [&](const WorkerCtx& ctx) {
      return okt_oklab::ok_sparse_allreduce(ctx, sg[ctx.rank], in[ctx.rank], t, k);
    });
    for (int r = 0; r < P; ++r) {
      if (!(ref[r].u == gpu[r].u) || ref[r].indexes != gpu[r].indexes ||
          ref[r].local_selected != gpu[r].local_selected || !same_state(sr[r], sg[r])) {
        std::printf("FAIL %s: t=%lld rank %d result/state differs\n", name, (long long)t, r);
        okt_oklab::release(&wg.transport);
        return 1;
      }
    }
    if (!same_ledger(wr.ledger, wg.ledger, P)) {
      std::printf("FAIL %s: t=%lld ledger differs\n", name, (long long)t);
      okt_oklab::release(&wg.transport);
      return 1;
    }
  }
  std::printf("PASS %s\n", name);
  okt_oklab::release(&wg.transport);
  return 0;
}

// One Table-1 baseline on both implementations (same inputs, same ledger).
int baseline(const char* name, int P, const std::vector<DenseGrad>& in,
             const std::function<SparseGrad(const WorkerCtx&, const DenseGrad&, bool)>& fn) {
  World wr(P), wg(P);
  auto ref = run_ranks(wr, [&](const WorkerCtx& ctx) { return fn(ctx, in[ctx.rank], false); });
  auto gpu = run_ranks(wg, [&](const WorkerCtx& ctx) { return fn(ctx, in[ctx.rank], true); });
  okt_oklab::release(&wg.transport);
  for (int r = 0; r < P; ++r)
    if (!(ref[r] == gpu[r])) {
      std::printf("FAIL %s: rank %d result differs\n", name, r);
      return 1;
    }
  if (!same_ledger(wr.ledger, wg.ledger, P)) {
    std::printf("FAIL %s: ledger differs\n", name);
    return 1;
  }
  std::printf("PASS %s\n", name);
  return 0;
}

}  // namespace

int main() {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  int fails = 0;
  // acceptance.cpp:101-145 (criterion 1), a subset of the 100 instances
  for (int m = 0; m < 12; ++m) {
    const int P = (int[]){2, 4, 8}[m % 3];
    const std::size_t n = (std::size_t[]){64, 1000}[(m / 3) % 2];
    const std::size_t k = (std::size_t[]){4, 16, 32}[(m / 6) % 3];
    const std::uint64_t seed = 1000 + m;
    char name[64];
    std::snprintf(name, sizeof(name), "c1 instance %d", m);
    fails += scenario(name, P, n, k, 1, 1, 1, 4,
                      [&](int r, std::int64_t) { return test::random_dense(seed * 8 + r, n); });
  }
  // test_oktopk.cpp:277-330
  for (int P : {2, 4})
    fails += scenario("t=1 selection-sum oracle", P, 64, 6, 1, 64, 32, 4,
                      [](int r, std::int64_t) { return test::random_dense(2026 + 11 * std::uint64_t(r), 64); });
  // drift trajectory with refreshes, learned cuts and bucketing (trainer.cpp:338-388)
  for (int P : {1, 2, 4, 8})
    fails += scenario("drift trajectory", P, 20000, 200, 12, 8, 4, 3, [](int r, std::int64_t t) {
      DriftOptions o;
      o.rank_key = std::uint64_t(r) + 1;
      return drifting_gradient_process(t, 3, 20000, o);
    });
  // off-cycle equal-width fallback (test_oktopk.cpp:382-398): first call at t = 5
  {
    World wr(2), wg(2);
    auto ref = run_ranks(wr, [&](const WorkerCtx& ctx) {
      OkState s;
      return oklab::ok_sparse_allreduce(ctx, s, f32(test::random_dense(77 + ctx.rank, 32)), 5, 4).u;
    });
    auto gpu = run_ranks(wg, [&](const WorkerCtx& ctx) {
      OkState s;
      return okt_oklab::ok_sparse_allreduce(ctx, s, f32(test::random_dense(77 + ctx.rank, 32)), 5, 4).u;
    });
    okt_oklab::release(&wg.transport);
    const bool ok = ref[0] == gpu[0] && ref[1] == gpu[1] && gpu[0].nnz() == 32;
    std::printf("%s off-cycle fallback\n", ok ? "PASS" : "FAIL");
    fails += ok ? 0 : 1;
  }
  // errors map onto the reference's exception types (test_oktopk.cpp:400-419)
  {
    World w(1);
    WorkerCtx ctx = w.ctx(0);
    OkState s;
    int ok = 0;
    try { okt_oklab::ok_sparse_allreduce(ctx, s, DenseGrad{}, 1, 1); } catch (const std::invalid_argument&) { ++ok; }
    try { okt_oklab::ok_sparse_allreduce(ctx, s, DenseGrad(std::vector<double>{1.0}), 0, 1); } catch (const std::invalid_argument&) { ++ok; }
    try { okt_oklab::ok_sparse_allreduce(ctx, s, DenseGrad(std::vector<double>{1.0, std::nan("")}), 1, 1); } catch (const NumericError&) { ++ok; }
    okt_oklab::release(&w.transport);
    std::printf("%s exception mapping\n", ok == 3 ? "PASS" : "FAIL");
    fails += ok == 3 ? 0 : 1;
  }
  // Table-1 baselines (test_collectives.cpp:167-350 inputs)
  {
    auto ins = [](int P, std::size_t n, std::uint64_t seed, int kind) {
      std::vector<DenseGrad> v;
      for (int r = 0; r < P; ++r) {
        DenseGrad g = kind == 0   ? test::random_int_dense(seed + r, n, 1000)
                      : kind == 2 ? test::random_int_dense(seed + 3 * r, n, 9)
                                  : f32(test::random_dense(seed + r, n));
        if (kind == 2)  // test_collectives.cpp:227-231: strictly positive integers
          for (double& x : g.values) x = std::fabs(x) + 1.0;
        v.push_back(std::move(g));
      }
      return v;
    };
    fails += baseline("topka_allreduce", 4, ins(4, 200, 900, 0), [](const WorkerCtx& c, const DenseGrad& g, bool b) {
      return b ? okt_oklab::topka_allreduce(c, g, 12) : oklab::topka_allreduce(c, g, 12);
    });
    fails += baseline("topkdsa_allreduce", 4, ins(4, 120, 7100, 0), [](const WorkerCtx& c, const DenseGrad& g, bool b) {
      return b ? okt_oklab::topkdsa_allreduce(c, g, 10) : oklab::topkdsa_allreduce(c, g, 10);
    });
    fails += baseline("topkdsa crossover", 4, ins(4, 64, 8200, 2), [](const WorkerCtx& c, const DenseGrad& g, bool b) {
      return b ? okt_oklab::topkdsa_allreduce(c, g, 24) : oklab::topkdsa_allreduce(c, g, 24);
    });
    for (int P : {2, 4, 8})
      fails += baseline("gtopk_allreduce", P, ins(P, 150, 4400, 1), [](const WorkerCtx& c, const DenseGrad& g, bool b) {
        return b ? okt_oklab::gtopk_allreduce(c, g, 8) : oklab::gtopk_allreduce(c, g, 8);
      });
    fails += baseline("gaussiank_allreduce", 4, ins(4, 300, 6600, 0), [](const WorkerCtx& c, const DenseGrad& g, bool b) {
      return b ? okt_oklab::gaussiank_allreduce(c, g, 20) : oklab::gaussiank_allreduce(c, g, 20);
    });
    fails += baseline("gaussiank raw", 2, ins(2, 5000, 6800, 1), [](const WorkerCtx& c, const DenseGrad& g, bool b) {
      GaussiankOptions o;
      o.scale_to_floor = false;
      return b ? okt_oklab::gaussiank_allreduce(c, g, 400, o) : oklab::gaussiank_allreduce(c, g, 400, o);
    });
  }
  // dense_allreduce (collectives.cpp:89-150) on fp32-representable inputs
  for (int P : {2, 4, 8}) {
    World wr(P), wg(P);
    std::vector<DenseGrad> in;
    for (int r = 0; r < P; ++r) in.push_back(f32(test::random_dense(5100 + r, 1001)));
    auto ref = run_ranks(wr, [&](const WorkerCtx& c) { return oklab::dense_allreduce(c, in[c.rank]); });
    auto gpu = run_ranks(wg, [&](const WorkerCtx& c) { return okt_oklab::dense_allreduce(c, in[c.rank]); });
    okt_oklab::release(&wg.transport);
    bool ok = same_ledger(wr.ledger, wg.ledger, P);
    for (int r = 0; r < P; ++r) ok = ok && ref[r].values == gpu[r].values;
    std::printf("%s dense_allreduce P=%d\n", ok ? "PASS" : "FAIL", P);
    fails += ok ? 0 : 1;
  }
  std::printf("%d failing scenarios\n", fails);
  return fails;
}
