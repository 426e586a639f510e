"""GPU parity: the CUDA path (through the C-ABI) against the pinned oracle.

Mirrors proj/tests/test_oktopk.cpp, test_sparse_core.cpp and acceptance.cpp
criterion 1.  Inputs are rounded to fp32 first (the device computes on fp32
dense state); on fp32-representable inputs every index set, threshold, ledger
counter and fp64 value must equal the reference's bit for bit.
"""
import numpy as np
import pytest

from oracle import OrcState

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def okm(gpus):
    from paper_2201_07598_b200 import oktopk
    return oktopk


def devices_for(P, gpus):
    return [r % gpus for r in range(P)]


def gpu_world(okm, P, gpus):
    return okm.World(P, devices_for(P, gpus))


def ledger_array(w, P):
    out = np.zeros((P, 6, 4), np.uint64)
    for r in range(P):
        for ph in range(6):
            c = w.ledger.at(r, ph)
            out[r, ph] = (c.words_sent, c.words_recv, c.msgs_sent, c.msgs_recv)
    return out


# ---- th_re_evaluate / select (test_oktopk.cpp:46-65, test_sparse_core.cpp:119-140) ----
def test_th_re_evaluate_known_answers(okm):
    g = [0.5, -2.0, 1.0, 0.25]
    assert okm.th_re_evaluate(g, 1) == 2.0
    assert okm.th_re_evaluate(g, 2) == 1.0
    assert okm.th_re_evaluate(g, 3) == 0.5
    assert okm.th_re_evaluate(g, 400) == 0.25
    with pytest.raises(okm.InvalidArgument):
        okm.th_re_evaluate([], 1)
    with pytest.raises(okm.InvalidArgument):
        okm.th_re_evaluate(g, 0)


def test_th_re_evaluate_sparse_min_magnitude(okm):
    s = okm.SparseGrad(8, np.array([0, 1, 2], np.uint32), np.array([0.9, -0.2, 0.5]))
    assert okm.th_re_evaluate(s, 3) == 0.2
    assert okm.th_re_evaluate(s, 9) == 0.2
    assert okm.th_re_evaluate(s, 1) == 0.9
    with pytest.raises(okm.InvalidArgument):
        okm.th_re_evaluate(okm.SparseGrad(8), 1)


@pytest.mark.parametrize("n", [1, 7, 4096, 4097, 100_003, 1_000_000])
def test_th_re_evaluate_matches_oracle(okm, oracle, n):
    g = f32(oracle.random_dense(31 + n, n))
    for k in sorted({1, 2, max(1, n // 100), max(1, n // 2), n, n + 5}):
        assert okm.th_re_evaluate(g, k) == oracle.kth_largest_mag(g, k), (n, k)


def test_th_re_evaluate_ties_and_zeros(okm, oracle):
    g = f32(np.array([0.0, -0.0, 1.0, -1.0, 1.0, 0.5, 0.5, 0.0] * 1000))
    for k in (1, 2, 3, 2999, 3000, 3001, 5000, 7999, 8000, 9000):
        assert okm.th_re_evaluate(g, k) == oracle.kth_largest_mag(g, k), k


def test_select_inclusive_keeps_signs(okm):
    g = [0.0, -1.0, 0.5, 2.0, -0.5]
    s = okm.select_by_threshold(g, 0.5)
    assert list(s.indices) == [1, 2, 3, 4]
    assert list(s.values) == [-1.0, 0.5, 2.0, -0.5]
    assert okm.select_by_threshold(g, 0.0).nnz() == 5  # zero threshold keeps zeros
    with pytest.raises(okm.InvalidArgument):
        okm.select_by_threshold([1.0], -0.1)
    with pytest.raises(okm.InvalidArgument):
        okm.select_by_threshold([1.0], float("nan"))


@pytest.mark.parametrize("n", [1, 5, 4095, 4096, 4097, 65_537, 2_000_003])
def test_select_matches_oracle(okm, oracle, n):
    g = f32(oracle.random_dense(77 + n, n))
    for th in (0.0, 0.5, 0.99, 2.0, float(np.float32(0.3)) + 1e-12):
        s = okm.select_by_threshold(g, th)
        idx, val = oracle.select(g, th)
        assert np.array_equal(s.indices, idx) and np.array_equal(s.values, val), (n, th)


# ---- space_repartition (test_oktopk.cpp:67-116) ----
def test_space_repartition_two_ranks(okm, gpus):
    w = gpu_world(okm, 2, gpus)
    sel = {0: [0, 1, 2, 3], 1: [4, 5, 6, 7]}
    got = okm.run_ranks(w, lambda ctx: okm.space_repartition(
        ctx, okm.SparseGrad(8, np.array(sel[ctx.rank], np.uint32), np.ones(4))).cuts)
    assert got[0] == [0, 4, 8] and got[1] == got[0]


def test_space_repartition_four_asymmetric(okm, gpus):
    w = gpu_world(okm, 4, gpus)
    sel = {0: list(range(8)), 1: list(range(8, 16)), 2: [], 3: [0, 15]}
    got = okm.run_ranks(w, lambda ctx: okm.space_repartition(
        ctx, okm.SparseGrad(16, np.array(sel[ctx.rank], np.uint32), np.ones(len(sel[ctx.rank])))).cuts)
    for r in range(4):
        assert got[r] == [0, 4, 10, 12, 16]
    # consensus ledger: log2(4) rounds of P+1 words each way
    assert w.ledger.at(0, okm.Phase.consensus).words_sent == 2 * 5


def test_space_repartition_all_empty(okm, gpus):
    w = gpu_world(okm, 4, gpus)
    got = okm.run_ranks(w, lambda ctx: okm.space_repartition(ctx, okm.SparseGrad(12)).cuts)
    for r in range(4):
        assert got[r] == [0, 3, 6, 9, 12]


# ---- split_and_reduce (test_oktopk.cpp:118-187) ----
def test_split_and_reduce_routes_and_sums(okm, gpus):
    w = gpu_world(okm, 2, gpus)
    b = okm.RegionBoundaries([0, 5, 10])

    def body(ctx):
        g = np.zeros(10)
        if ctx.rank == 0:
            g[5:10] = [1, 2, 3, 4, 5]
        else:
            g[2], g[5] = 7, 9
        return okm.split_and_reduce(ctx, g, 0.5, b, 2)

    got = okm.run_ranks(w, body)
    assert got[0].region_reduced.as_map() == {2: 7.0}
    assert got[1].region_reduced.as_map() == {5: 10.0, 6: 2.0, 7: 3.0, 8: 4.0, 9: 5.0}
    assert list(got[0].local_topk_indexes) == [5, 6, 7, 8, 9]
    assert list(got[1].local_topk_indexes) == [2, 5]
    assert w.ledger.at(0, okm.Phase.split).msgs_sent == 3
    assert w.ledger.at(0, okm.Phase.split).words_sent == 10
    assert w.ledger.at(1, okm.Phase.split).msgs_sent == 1
    assert w.ledger.at(1, okm.Phase.split).words_sent == 2


def test_split_and_reduce_empty_slice_sends_one_message(okm, gpus):
    w = gpu_world(okm, 2, gpus)
    b = okm.RegionBoundaries([0, 4, 8])

    def body(ctx):
        g = np.zeros(8)
        g[4 * ctx.rank] = 1.0
        return okm.split_and_reduce(ctx, g, 0.5, b, 4)

    got = okm.run_ranks(w, body)
    for r in range(2):
        assert got[r].region_reduced.nnz() == 1
        assert w.ledger.at(r, okm.Phase.split).msgs_sent == 1
        assert w.ledger.at(r, okm.Phase.split).words_sent == 0


def test_split_and_reduce_bracket_and_explicit_zero(okm, gpus):
    # Stride-doubling bracket (sparse.cpp:238-245): (p0 + p2) + (p1 + p3).
    w = gpu_world(okm, 4, gpus)
    big = float(2 ** 54)
    vals = [big, 1.0, -big, 1.0]
    b = okm.RegionBoundaries([0, 2, 2, 2, 2])

    def body(ctx):
        g = np.zeros(2)
        g[0] = vals[ctx.rank]
        g[1] = 1.5 if ctx.rank % 2 == 0 else -1.5  # cancels to an explicit zero
        return okm.split_and_reduce(ctx, g, 0.25, b, 0)

    got = okm.run_ranks(w, body)
    assert got[0].region_reduced.as_map() == {0: 2.0, 1: 0.0}
    for r in range(1, 4):
        assert got[r].region_reduced.nnz() == 0


# ---- balance_and_allgatherv (test_oktopk.cpp:225-275) ----
def test_balance_no_skew_is_pure_allgather(okm, gpus):
    n = 40
    w = gpu_world(okm, 4, gpus)

    def body(ctx):
        idx = [10 * ctx.rank + j for j in range(3)] + [10 * ctx.rank + 5]
        val = [2.0 + ctx.rank + 0.125 * j for j in range(3)] + [0.5]
        return okm.balance_and_allgatherv(ctx, okm.SparseGrad(n, np.array(idx, np.uint32), np.array(val)), 1.0)

    got = okm.run_ranks(w, body)
    assert got[0].nnz() == 12 and got[0].valid()
    for r in range(4):
        assert got[r] == got[0]
        assert w.ledger.at(r, okm.Phase.balance).words_sent == 0
        assert w.ledger.at(r, okm.Phase.balance).msgs_sent == 0
    assert 5 not in got[1].as_map()
    assert got[2].as_map()[12] == 3.25


def test_balance_rebalances_all_at_one_rank(okm, gpus):
    n = 100
    w = gpu_world(okm, 4, gpus)

    def body(ctx):
        if ctx.rank == 0:
            return okm.balance_and_allgatherv(
                ctx, okm.SparseGrad(n, np.arange(12, dtype=np.uint32), 2.0 + np.arange(12.0)), 1.0)
        return okm.balance_and_allgatherv(ctx, okm.SparseGrad(n), 1.0)

    got = okm.run_ranks(w, body)
    for r in range(4):
        assert got[r].nnz() == 12 and got[r] == got[0] and got[r].valid()
    assert w.ledger.at(0, okm.Phase.balance).words_sent == 18
    assert w.ledger.at(0, okm.Phase.balance).msgs_sent == 3
    for r in range(1, 4):
        assert w.ledger.at(r, okm.Phase.balance).words_recv == 6
        assert w.ledger.at(r, okm.Phase.balance).words_sent == 0


# ---- ok_sparse_allreduce (test_oktopk.cpp:277-419, acceptance.cpp:101-145) ----
def run_both(okm, oracle, P, gpus, inputs_at, ts, k, tau=64, tau_prime=32, bucket=4, fresh=True):
    """Run the GPU path and the oracle over iterations `ts`; assert equality of
    u, indexes, local_selected, states and ledgers after every iteration."""
    w = gpu_world(okm, P, gpus)
    st_gpu = [okm.OkState(okm.ThresholdState(tau=tau, tau_prime=tau_prime), bucket_size=bucket) for _ in range(P)]
    st_orc = [OrcState.fresh(tau, tau_prime, bucket) for _ in range(P)]
    led = np.zeros((P, 6, 4), np.uint64)
    for t in ts:
        inputs = [f32(inputs_at(t, r)) for r in range(P)]
        rc, want = oracle.ok_sparse_allreduce(inputs, st_orc, t, k, led)
        assert rc == 0
        got = okm.run_ranks(w, lambda ctx: okm.ok_sparse_allreduce(ctx, st_gpu[ctx.rank], inputs[ctx.rank], t, k))
        for r in range(P):
            assert np.array_equal(got[r].u.indices, want["u_idx"]), (t, r, "u indices")
            assert np.array_equal(got[r].u.values, want["u_val"]), (t, r, "u values")
            assert np.array_equal(got[r].indexes, want["indexes"][r]), (t, r, "indexes")
            assert got[r].local_selected == want["local_selected"][r], (t, r)
            s, o = st_gpu[r], st_orc[r]
            assert (s.th.local_th, s.th.global_th) == (o.local_th, o.global_th), (t, r)
            assert (s.th.last_local_eval, s.th.last_global_eval) == (o.last_local_eval, o.last_global_eval)
            assert s.bounds.cuts == o.cuts_list(), (t, r)
            assert s.t == o.t
        assert np.array_equal(ledger_array(w, P), led), (t, "ledger")
    return w, st_gpu


@pytest.mark.parametrize("P", [2, 4])
def test_allreduce_t1_matches_selection_sum_oracle(okm, oracle, gpus, P):
    run_both(okm, oracle, P, gpus, lambda t, r: oracle.random_dense(2026 + 11 * r, 64), [1], 6)


def test_acceptance_c1_oracle_equivalence(okm, oracle, gpus):
    for m in range(100):
        P = [2, 4, 8][m % 3]
        n = [64, 1000][(m // 3) % 2]
        k = [4, 16, 32][(m // 6) % 3]
        seed = 1000 + m
        run_both(okm, oracle, P, gpus, lambda t, r: oracle.random_dense(seed * 8 + r, n), [1], k, 1, 1)


def test_stale_threshold_reuse(okm, oracle, gpus):
    n, k, P = 48, 5, 4
    rng = np.random.default_rng(900)
    data = {}
    for t in range(1, 6):
        for r in range(P):
            bias = np.where((t < 5) == (np.arange(n) < n // 2), 3.0, 0.0)
            data[(t, r)] = rng.uniform(-1, 1, n) + np.where(rng.uniform(size=n) < 0.3, bias, 0.0)
    w, st = run_both(okm, oracle, P, gpus, lambda t, r: data[(t, r)], range(1, 6), k, tau=4, tau_prime=2)
    assert st[0].bounds.cuts  # learned at t = 1, re-learned at t = 5


def test_off_cycle_equal_width_fallback(okm, oracle, gpus):
    w, st = run_both(okm, oracle, 2, gpus, lambda t, r: oracle.random_dense(77 + r, 32), [5], 4)
    assert st[0].bounds.cuts == [0, 16, 32]


def test_single_rank_and_validation(okm, gpus):
    w = gpu_world(okm, 1, gpus)
    ctx = w.ctx(0)
    res = okm.ok_sparse_allreduce(ctx, okm.OkState(), [3.0, -1.0, 0.5, 2.0], 1, 2)
    assert res.u.as_map() == {0: 3.0, 3: 2.0}
    assert list(res.indexes) == [0, 3]
    assert res.local_selected == 2
    s2 = okm.OkState()
    with pytest.raises(okm.InvalidArgument):
        okm.ok_sparse_allreduce(ctx, s2, [], 1, 1)
    with pytest.raises(okm.InvalidArgument):
        okm.ok_sparse_allreduce(ctx, s2, [3.0, 1.0], 0, 1)
    with pytest.raises(okm.InvalidArgument):
        okm.ok_sparse_allreduce(ctx, s2, [3.0, 1.0], 1, 0)
    with pytest.raises(okm.NumericError):
        okm.ok_sparse_allreduce(ctx, s2, [1.0, float("nan")], 1, 1)
    assert s2.t == 0 and s2.th.local_th == 0.0  # failed calls leave the state alone


def test_nonfinite_on_one_rank_is_root_cause(okm, oracle, gpus):
    w = gpu_world(okm, 4, gpus)

    def body(ctx):
        g = f32(oracle.random_dense(5 + ctx.rank, 256))
        if ctx.rank == 2:
            g[17] = np.inf
        return okm.ok_sparse_allreduce(ctx, okm.OkState(), g, 1, 8)

    with pytest.raises(okm.NumericError):
        okm.run_ranks(w, body)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_drift_trajectory_matches_oracle(okm, oracle, gpus, P):
    # D1 drift inputs, tau = 8, tau' = 4, bucket 3: refreshes, stale reuse and
    # learned boundaries across 17 iterations.
    n, k = 20_000, 200
    run_both(okm, oracle, P, gpus, lambda t, r: oracle.drift(t, 3, n, r + 1), range(1, 18), k, 8, 4, 3)


@pytest.mark.parametrize("P", [1, 4])
def test_one_million_drift(okm, oracle, gpus, P):
    n, k = 1_000_000, 10_000
    run_both(okm, oracle, P, gpus, lambda t, r: oracle.drift(t, 1, n, r + 1), [1, 2, 3], k, 64, 2)


def test_uniform_inputs_skew_balance(okm, oracle, gpus):
    # All mass on one rank's region: exercises the balance phase end to end.
    P, n, k = 4, 4096, 64

    def inputs(t, r):
        g = f32(oracle.random_dense(50 + r + 10 * t, n)) * 1e-3
        g[: n // 8] += 1.0 + 0.001 * r  # heavy prefix lands in region 0
        return g

    run_both(okm, oracle, P, gpus, inputs, [1, 2, 3], k, 2, 1)


# ---- error-feedback SGD step (trainer.cpp:466-488), exact-sum inputs (D3) ----
@pytest.mark.parametrize("P", [1, 2, 4])
def test_sgd_trajectory_exact_sum(okm, oracle, gpus, P):
    n, k, steps = 5000, 50, 24
    w = gpu_world(okm, P, gpus)
    st_gpu = [okm.OkState(okm.ThresholdState(tau=8, tau_prime=4), bucket_size=4) for _ in range(P)]
    st_orc = [OrcState.fresh(8, 4, 4) for _ in range(P)]
    models = [okm.ModelState(np.zeros(n), w.devices[r], okm.LrSchedule(1.0)) for r in range(P)]
    res = [okm.Residual(n) for _ in range(P)]
    eps = [np.zeros(n) for _ in range(P)]
    ws = [np.zeros(n) for _ in range(P)]
    for t in range(1, steps + 1):
        grads = [oracle.random_int_dense(1000 * t + r, n, 3) for r in range(P)]
        rc, u_idx, u_val = oracle.sgd_step(grads, eps, ws, st_orc, 1.0, t, k)
        assert rc == 0
        got = okm.run_ranks(w, lambda ctx: okm.oktopk_sgd_step(ctx, models[ctx.rank], res[ctx.rank],
                                                               grads[ctx.rank], k, st_gpu[ctx.rank]))
        for r in range(P):
            assert np.array_equal(got[r].u.indices, u_idx) and np.array_equal(got[r].u.values, u_val), (t, r)
            assert np.array_equal(res[r].eps(w.ctx(r)), eps[r]), (t, r, "residual")
            wm = models[r].w.cpu().numpy().astype(np.float64)
            assert np.array_equal(wm, ws[r]), (t, r, "model")


# ---- golden vectors produced by the reference itself (tests/golden) ----
from . import _golden  # noqa: E402


@pytest.mark.parametrize("name", _golden.cases())
def test_gpu_reproduces_reference_golden(okm, gpus, name):
    fx = _golden.load(name)
    P = int(fx["P"])
    w = gpu_world(okm, P, gpus)
    st = [okm.OkState(okm.ThresholdState(tau=int(fx["tau"]), tau_prime=int(fx["tau_prime"])),
                      bucket_size=int(fx["bucket"])) for _ in range(P)]
    prev = np.zeros((P, 6, 4), np.uint64)
    for t in fx["ts"]:
        t = int(t)
        ins = fx[f"in_t{t}"]
        got = okm.run_ranks(w, lambda ctx: okm.ok_sparse_allreduce(ctx, st[ctx.rank], ins[ctx.rank], t, int(fx["k"])))
        led = ledger_array(w, P)
        _golden.check_step(fx, t, P, got[0].u.indices, got[0].u.values, [g.indexes for g in got],
                           [g.local_selected for g in got], led - prev)
        prev = led
        for r in range(1, P):
            assert got[r].u == got[0].u


# ---- asynchronous entry points (okt_*_async + okt_step_wait) ----
@pytest.mark.parametrize("P", [1, 2])
def test_async_steps_match_sync_steps(okm, oracle, gpus, P):
    import ctypes
    import torch
    from paper_2201_07598_b200 import _lib
    L = _lib.lib()
    n, k, steps = 50_000, 500, 40
    worlds = [gpu_world(okm, P, gpus), gpu_world(okm, P, gpus)]
    for w in worlds:
        for r in range(P):
            assert L.okt_set_params(w.ctx(r).comm, 8, 4, 2) == 0
    grads = {(t, r): torch.from_numpy(oracle.drift(t, 4, n, r + 1).astype(np.float32)).to(f"cuda:{w.devices[r]}")
             for t in range(1, steps + 1) for r in range(P) for w in worlds[:1]}
    models = [[torch.zeros(n, dtype=torch.float32, device=f"cuda:{w.devices[r]}") for r in range(P)] for w in worlds]

    def run(wi, asynchronous):
        w = worlds[wi]

        def body(ctx):
            torch.cuda.set_device(w.devices[ctx.rank])
            out = []
            for t in range(1, steps + 1):
                g = grads[(t, ctx.rank)].to(f"cuda:{w.devices[ctx.rank]}")
                res = _lib.OktResult()
                args = (ctx.comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(models[wi][ctx.rank].data_ptr()),
                        n, 1.0, t, k)
                if asynchronous:
                    assert L.okt_sgd_step_async(*args, None) == 0, L.okt_last_error()
                    assert L.okt_step_wait(ctx.comm, ctypes.byref(res)) == 0, L.okt_last_error()
                else:
                    assert L.okt_sgd_step(*args, ctypes.byref(res), None) == 0, L.okt_last_error()
                out.append(okm._sparse_from(res.u, n))
            return out
        return okm.run_ranks(w, body)

    a = run(0, False)
    b = run(1, True)
    for r in range(P):
        for t in range(steps):
            assert a[r][t] == b[r][t], (r, t)
        assert torch.equal(models[0][r].cpu(), models[1][r].cpu())


# ---- shape and value edge cases (sizes off the 16-byte / tile grid, k >= n,
# all-zero and tie-heavy inputs, cancelling ranks), several iterations each so
# the steady path (graph at P = 1, P2P or host-synced at P > 1) runs too ----
def _edge_inputs(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "normal":
        return lambda t, r: rng.standard_normal(n) * (1 + t)
    if kind == "zeros":
        return lambda t, r: np.zeros(n)
    if kind == "ties":
        return lambda t, r: rng.choice([-2.0, -1.0, 0.0, 1.0, 2.0], n)
    if kind == "cancel":  # ranks pair up with opposite signs: explicit zeros in the regions
        base = {t: rng.standard_normal(n) for t in range(1, 8)}
        return lambda t, r: base[t] * (1.0 if r % 2 == 0 else -1.0)
    raise ValueError(kind)


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("n,k,kind", [
    (1, 1, "normal"), (3, 2, "normal"), (4097, 40, "normal"), (8195, 9000, "normal"), (5000, 5000, "ties"),
    (6000, 60, "zeros"), (20_003, 200, "ties"), (12_289, 120, "cancel"),
])
def test_edge_shapes_match_oracle(okm, oracle, gpus, P, n, k, kind):
    run_both(okm, oracle, P, gpus, _edge_inputs(kind, n, 17 * n + k), range(1, 7), k, tau=4, tau_prime=2)
