"""GPU parity of the Table-1 TopkA baseline (okt_topka_allreduce, the CUDA
restatement of collectives.cpp:152-159) through the C-ABI: golden vectors made
by the reference itself, the pinned oracle on larger seeded inputs (ties that
straddle the trim kernel's 1024-entry chunks included), the reference test's
ledger property (test_collectives.cpp:186-188) and the error behaviour."""
import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "topka")
CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(HERE, "*.npz")))


@pytest.fixture(scope="module")
def okm(gpus):
    from paper_2201_07598_b200 import oktopk
    return oktopk


def run_topka(okm, gpus, inputs, k):
    P = len(inputs)
    w = okm.World(P, [r % gpus for r in range(P)])
    try:
        got = okm.run_ranks(w, lambda ctx: okm.topka_allreduce(ctx, inputs[ctx.rank].astype(np.float32), k))
        led = [w.ledger.at(r, okm.Phase.allgatherv) for r in range(P)]
    finally:
        w.destroy()
    for r in range(1, P):
        assert np.array_equal(got[r].indices, got[0].indices)
        assert np.array_equal(got[r].values.view(np.uint64), got[0].values.view(np.uint64))
    return got[0], led


def same(got, ui, uv):
    assert np.array_equal(got.indices.astype(np.uint32), ui)
    assert np.array_equal(got.values.astype(np.float64).view(np.uint64), uv.view(np.uint64))


@pytest.mark.parametrize("name", CASES)
def test_topka_golden(okm, gpus, name):
    fx = dict(np.load(os.path.join(HERE, name)))
    got, led = run_topka(okm, gpus, list(fx["inputs"]), int(fx["k"]))
    same(got, fx["u_idx"], fx["u_val"])
    P, k = int(fx["P"]), int(fx["k"])
    for c in led:  # test_collectives.cpp:186-188
        assert c.words_sent == 2 * k * (P - 1) and c.words_recv == 2 * k * (P - 1)


@pytest.mark.parametrize("P,n,k,kind", [
    (1, 200_000, 2_000, "f32"), (2, 300_000, 3_000, "f32"), (4, 100_000, 20_000, "ties"),
    (8, 50_000, 7_000, "ties"), (4, 65_536, 1, "f32"), (2, 4_096, 4_096, "ties"), (4, 30_000, 900, "int"),
])
def test_topka_matches_oracle(okm, gpus, oracle, P, n, k, kind):
    rng = np.random.default_rng(P * 1000 + k)
    if kind == "f32":
        ins = [rng.standard_normal(n).astype(np.float32).astype(np.float64) for _ in range(P)]
    elif kind == "ties":
        ins = [rng.choice([-1.0, 1.0, 0.5, -0.5, 0.0, 0.25], n) for _ in range(P)]
    else:
        ins = [rng.integers(-50, 51, n).astype(np.float64) for _ in range(P)]
    got, _ = run_topka(okm, gpus, ins, k)
    ui, uv = oracle.topka_allreduce(ins, k)
    same(got, ui, uv)


def test_topka_rejects_bad_k(okm, gpus):
    w = okm.World(1, [0])
    try:
        for k in (0, 11):
            with pytest.raises(okm.InvalidArgument):
                okm.topka_allreduce(w.ctx(0), np.ones(10, np.float32), k)
    finally:
        w.destroy()


def test_topka_non_finite_fails_everywhere(okm, gpus):
    ins = [np.ones(64, np.float32), np.ones(64, np.float32)]
    ins[1][5] = np.nan
    w = okm.World(2, [r % gpus for r in range(2)])
    errs = [None, None]

    def body(ctx):
        try:
            okm.topka_allreduce(ctx, ins[ctx.rank], 4)
        except okm.OkError as e:
            errs[ctx.rank] = e
    try:
        okm.run_ranks(w, body)
    finally:
        w.destroy()
    assert isinstance(errs[1], okm.NumericError)
    assert isinstance(errs[0], okm.TransportError)
