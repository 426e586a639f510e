"""CPU: the C restatements of the other Table-1 baselines (gTopk, TopkDSA,
Gaussiank; oracle/okt_oracle.c) against golden vectors produced by the
reference's own collectives (tests/golden/baselines/*.npz, made by
tests/golden/make_golden.py): outputs bit for bit, ledger counters exactly,
and the properties the reference's tests check (test_collectives.cpp:192-350)."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "baselines")
CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(HERE, "*.npz")))


def load(name):
    return dict(np.load(os.path.join(HERE, name)))


@pytest.mark.parametrize("name", CASES)
def test_oracle_baseline_reproduces_golden(oracle, name):
    fx = load(name)
    P = int(fx["P"])
    led = np.zeros((P, 6, 4), np.uint64)
    ui, uv = oracle.baseline(str(fx["which"]), list(fx["inputs"]), int(fx["k"]), bool(fx["scale"]), led)
    assert np.array_equal(ui, fx["u_idx"])
    assert np.array_equal(uv.view(np.uint64), fx["u_val"].view(np.uint64))
    assert np.array_equal(led, fx["ledger"])
    for r, th in enumerate(fx["th"]):
        assert oracle.gaussian_threshold(fx["inputs"][r], int(fx["k"]), bool(fx["scale"])) == th


def test_gtopk_ledger_words(oracle):
    # test_collectives.cpp:318-322: 2k words per level
    for P in (2, 4, 8):
        ins = [oracle.random_dense(4400 + 13 * r, 150) for r in range(P)]
        led = np.zeros((P, 6, 4), np.uint64)
        ui, _ = oracle.baseline("gtopk", ins, 8, ledger=led)
        assert ui.size <= 8
        assert all(int(led[r, 0, 0]) == 2 * 8 * (P.bit_length() - 1) for r in range(P))


def test_topkdsa_equals_topka_on_integer_data(oracle):
    ins = [oracle.random_int_dense(7100 + r, 120, 50) for r in range(4)]
    a = oracle.baseline("topkdsa", ins, 10)
    b = oracle.topka_allreduce(ins, 10)
    da = {i: v for i, v in zip(*a) if v != 0.0}
    db = {i: v for i, v in zip(*b) if v != 0.0}
    assert da == db


def test_gaussiank_scaling_stops_at_floor(oracle):
    g = oracle.random_dense(31, 400)
    k = 40
    raw = max(oracle.gaussian_threshold(g, k, False), 0.0)
    sc = oracle.gaussian_threshold(g, k, True)
    assert sc <= raw
    assert 4 * int(np.sum(np.abs(g) >= sc)) > 3 * k
    if sc < raw:
        assert 4 * int(np.sum(np.abs(g) >= sc / 0.9)) <= 3 * k


DENSE = sorted(os.path.basename(p) for p in glob.glob(os.path.join(os.path.dirname(HERE), "dense", "*.npz")))


@pytest.mark.parametrize("name", DENSE)
def test_oracle_dense_reproduces_golden(oracle, name):
    fx = dict(np.load(os.path.join(os.path.dirname(HERE), "dense", name)))
    P = int(fx["P"])
    led = np.zeros((P, 6, 4), np.uint64)
    out = oracle.dense_allreduce(list(fx["inputs"]), led)
    assert np.array_equal(out.view(np.uint64), fx["out"].view(np.uint64))
    assert np.array_equal(led, fx["ledger"])
