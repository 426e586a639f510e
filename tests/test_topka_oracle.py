"""CPU: the TopkA restatement (oracle/okt_oracle.c orc_topk_exact /
orc_topka_allreduce) against golden vectors produced by the reference's own
topka_allreduce (collectives.cpp:152-159; tests/golden/topka/*.npz, made by
tests/golden/make_golden.py), plus the reference test's properties
(test_collectives.cpp:167-190)."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "topka")
CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(HERE, "*.npz")))


def load(name):
    return dict(np.load(os.path.join(HERE, name)))


@pytest.mark.parametrize("name", CASES)
def test_oracle_topka_reproduces_golden(oracle, name):
    fx = load(name)
    ui, uv = oracle.topka_allreduce(list(fx["inputs"]), int(fx["k"]))
    assert np.array_equal(ui, fx["u_idx"])
    assert np.array_equal(uv.view(np.uint64), fx["u_val"].view(np.uint64))


def test_topk_exact_ties_toward_smaller_index(oracle):
    g = np.array([0.5, -1.0, 0.5, 1.0, -0.5, 0.25])
    idx, val = oracle.topk_exact(g, 4)
    assert list(idx) == [0, 1, 2, 3]       # |1| x2, then the first two 0.5 ties
    assert list(val) == [0.5, -1.0, 0.5, 1.0]


def test_topka_union_of_local_topk_int_data(oracle):
    P, n, k = 4, 200, 12
    ins = [oracle.random_int_dense(900 + r, n, 1000) for r in range(P)]
    exp = {}
    for g in ins:
        order = sorted(range(n), key=lambda i: (-abs(g[i]), i))[:k]
        for i in order:
            exp[i] = exp.get(i, 0.0) + g[i]
    ui, uv = oracle.topka_allreduce(ins, k)
    assert dict(zip(ui.tolist(), uv.tolist())) == exp
