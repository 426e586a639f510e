"""CPU: the oracle restatement (oracle/okt_oracle.c) pinned against the
reference's own known answers (proj/tests/test_oktopk.cpp,
test_sparse_core.cpp), against golden vectors produced by the reference, and —
where oracle/_ref is built — against the reference itself."""
import numpy as np
import pytest

from oracle import OrcState

from . import _golden


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


# ---- known answers ---------------------------------------------------------------
def test_kth_largest_magnitude(oracle):
    g = np.array([0.5, -2.0, 1.0, 0.25])
    assert [oracle.kth_largest_mag(g, k) for k in (1, 2, 3, 400)] == [2.0, 1.0, 0.5, 0.25]
    s = np.array([0.9, -0.2, 0.5])
    assert [oracle.kth_largest_mag(s, k) for k in (3, 9, 1)] == [0.2, 0.2, 0.9]


def test_select_inclusive(oracle):
    idx, val = oracle.select(np.array([0.0, -1.0, 0.5, 2.0, -0.5]), 0.5)
    assert list(idx) == [1, 2, 3, 4] and list(val) == [-1.0, 0.5, 2.0, -0.5]
    assert oracle.select(np.array([0.0, -1.0, 0.5]), 0.0)[0].size == 3


def test_sparse_sum_union_zero_and_bracket(oracle):
    i, v = oracle.sparse_sum([([1, 5, 9], [1.0, 2.0, 3.0]), ([5, 6], [10.0, -4.0]), ([0, 9], [7.0, -3.0])])
    assert list(i) == [0, 1, 5, 6, 9] and list(v) == [7.0, 1.0, 12.0, -4.0, 0.0]
    i, v = oracle.sparse_sum([([2], [1.5]), ([2], [-1.5])])
    assert list(i) == [2] and list(v) == [0.0]
    i, v = oracle.sparse_sum([([0], [x]) for x in (1e16, 1.0, -1e16, 1.0)])
    assert list(v) == [2.0]  # (p0 + p2) + (p1 + p3), not left to right


def test_space_repartition_known_answers(oracle):
    assert oracle.space_repartition([[0, 1, 2, 3], [4, 5, 6, 7]], 8) == [0, 4, 8]
    sels = [list(range(8)), list(range(8, 16)), [], [0, 15]]
    led = np.zeros((4, 6, 4), np.uint64)
    assert oracle.space_repartition(sels, 16, led) == [0, 4, 10, 12, 16]
    assert int(led[0, 3, 0]) == 2 * 5  # log2(4) rounds of P+1 words
    assert oracle.space_repartition([[], [], [], []], 12) == [0, 3, 6, 9, 12]


def test_equal_slice_ends(oracle):
    assert oracle.equal_slice_ends(10, 4) == [0, 3, 6, 8, 10]
    assert oracle.equal_slice_ends(3, 4) == [0, 1, 2, 3, 3]


def test_single_rank_known_answer(oracle):
    st = [OrcState.fresh()]
    rc, res = oracle.ok_sparse_allreduce([np.array([3.0, -1.0, 0.5, 2.0])], st, 1, 2)
    assert rc == 0
    assert list(res["u_idx"]) == [0, 3] and list(res["u_val"]) == [3.0, 2.0]
    assert list(res["indexes"][0]) == [0, 3] and res["local_selected"] == [2]
    assert oracle.ok_sparse_allreduce([np.array([1.0, np.nan])], [OrcState.fresh()], 1, 1)[0] == -2
    assert oracle.ok_sparse_allreduce([np.zeros(0)], [OrcState.fresh()], 1, 1)[0] == -1


def test_off_cycle_equal_width_fallback(oracle):
    ins = [oracle.random_dense(77 + r, 32) for r in range(2)]
    st = [OrcState.fresh() for _ in range(2)]
    rc, res = oracle.ok_sparse_allreduce(ins, st, 5, 4)
    assert rc == 0 and st[0].cuts_list() == [0, 16, 32] and res["u_idx"].size == 32


# ---- golden vectors produced by the reference ---------------------------------------
@pytest.mark.parametrize("name", _golden.cases())
def test_oracle_reproduces_golden(oracle, name):
    fx = _golden.load(name)
    P = int(fx["P"])
    states = [OrcState.fresh(int(fx["tau"]), int(fx["tau_prime"]), int(fx["bucket"])) for _ in range(P)]
    for t in fx["ts"]:
        t = int(t)
        led = np.zeros((P, 6, 4), np.uint64)
        rc, res = oracle.ok_sparse_allreduce(list(fx[f"in_t{t}"]), states, t, int(fx["k"]), led)
        assert rc == 0
        st = np.stack([np.frombuffer(bytes(s), np.uint8) for s in states])
        _golden.check_step(fx, t, P, res["u_idx"], res["u_val"], res["indexes"], res["local_selected"], led, st)


# ---- the reference itself --------------------------------------------------------------
def test_generators_match_reference(oracle, reference):
    for t in (1, 2, 1025):
        a = f32(oracle.drift(t, 9, 5000, 3))
        b = reference.drift_f32(t, 9, 5000, 3)
        assert np.array_equal(a, b)


def test_acceptance_c1_vs_reference(oracle, reference):
    for m in range(100):
        P = [2, 4, 8][m % 3]
        n = [64, 1000][(m // 3) % 2]
        k = [4, 16, 32][(m // 6) % 3]
        ins = [oracle.random_dense((1000 + m) * 8 + r, n) for r in range(P)]
        so = [OrcState.fresh(1, 1) for _ in range(P)]
        sr = [OrcState.fresh(1, 1) for _ in range(P)]
        lo, lr = np.zeros((P, 6, 4), np.uint64), np.zeros((P, 6, 4), np.uint64)
        rc1, a = oracle.ok_sparse_allreduce(ins, so, 1, k, lo)
        rc2, b = reference.ok_sparse_allreduce(ins, sr, 1, k, lr)
        assert rc1 == rc2 == 0
        assert np.array_equal(a["u_idx"], b["u_idx"]) and np.array_equal(a["u_val"], b["u_val"])
        assert all(np.array_equal(x, y) for x, y in zip(a["indexes"], b["indexes"]))
        assert np.array_equal(lo, lr)
        assert all(bytes(x) == bytes(y) for x, y in zip(so, sr))


@pytest.mark.parametrize("P,bucket", [(2, 0), (4, 3), (8, 4)])
def test_drift_trajectory_vs_reference(oracle, reference, P, bucket):
    n, k = 4000, 40
    so = [OrcState.fresh(6, 3, bucket) for _ in range(P)]
    sr = [OrcState.fresh(6, 3, bucket) for _ in range(P)]
    lo, lr = np.zeros((P, 6, 4), np.uint64), np.zeros((P, 6, 4), np.uint64)
    for t in range(1, 15):
        ins = [reference.drift_f32(t, 11, n, r + 1) for r in range(P)]
        rc1, a = oracle.ok_sparse_allreduce(ins, so, t, k, lo)
        rc2, b = reference.ok_sparse_allreduce(ins, sr, t, k, lr)
        assert rc1 == rc2 == 0
        assert np.array_equal(a["u_idx"], b["u_idx"]) and np.array_equal(a["u_val"], b["u_val"]), t
        assert all(bytes(x) == bytes(y) for x, y in zip(so, sr)), t
    assert np.array_equal(lo, lr)


def test_sgd_step_vs_reference_bench_path(oracle, reference):
    # The reference's EF-SGD timing loop runs end to end and is finite.
    ms = reference.bench_sgd(2, 20_000, 200, 1, 3, 64, 32, 4, 1.0, 1, False)
    assert ms.shape == (3,) and np.all(ms > 0)
