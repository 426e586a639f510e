"""GPU parity of the host-buffer entry points (okt_sgd_step_host,
okt_sparse_allreduce_host) — the reference's calling convention: the dense
gradient lives in host memory (oktopk.hpp:118-120 takes a DenseGrad by
reference).  Pinned and pageable host gradients must both give the oracle's
trajectory bit for bit (exact-sum integer inputs, as in
test_sgd_trajectory_exact_sum).
"""
import ctypes

import numpy as np
import pytest

from oracle import OrcState

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def okm(gpus):
    from paper_2201_07598_b200 import oktopk
    return oktopk


def _host_grad(x, pinned):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t.pin_memory() if pinned else t


@pytest.mark.parametrize("P", [1, 2])
@pytest.mark.parametrize("pinned", [True, False])
def test_sgd_step_host_matches_oracle(okm, oracle, gpus, P, pinned):
    import torch
    from paper_2201_07598_b200 import _lib
    L = _lib.lib()
    n, k, steps = 50001, 500, 12  # odd n: the last K1 tile is partial
    w = okm.World(P, [r % gpus for r in range(P)])
    for r in range(P):
        assert L.okt_set_params(w.ctx(r).comm, 8, 4, 4) == 0
    st_orc = [OrcState.fresh(8, 4, 4) for _ in range(P)]
    eps = [np.zeros(n) for _ in range(P)]
    ws = [np.zeros(n) for _ in range(P)]
    d_w = [torch.zeros(n, dtype=torch.float32, device=f"cuda:{w.devices[r]}") for r in range(P)]
    h_idx = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(P)]
    h_val = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(P)]
    for t in range(1, steps + 1):
        grads = [oracle.random_int_dense(7000 * t + r, n, 3) for r in range(P)]
        rc, u_idx, u_val = oracle.sgd_step(grads, eps, ws, st_orc, 1.0, t, k)
        assert rc == 0
        hg = [_host_grad(g, pinned) for g in grads]

        def body(ctx):
            r = ctx.rank
            res = _lib.OktResult()
            rc = L.okt_sgd_step_host(ctx.comm, ctypes.c_void_p(hg[r].data_ptr()), ctypes.c_void_p(d_w[r].data_ptr()),
                                     n, 1.0, t, k, ctypes.c_void_p(h_idx[r].data_ptr()),
                                     ctypes.c_void_p(h_val[r].data_ptr()), n, ctypes.byref(res), None)
            assert rc == 0, L.okt_last_error().decode()
            return int(res.u.nnz)

        U = okm.run_ranks(w, body)
        for r in range(P):
            assert U[r] == u_idx.size, (t, r)
            assert np.array_equal(h_idx[r][:U[r]].numpy().view(np.uint32), u_idx), (t, r)
            assert np.array_equal(h_val[r][:U[r]].numpy(), u_val), (t, r)
            assert np.array_equal(d_w[r].cpu().numpy().astype(np.float64), ws[r]), (t, r, "model")


@pytest.mark.parametrize("pinned", [True, False])
def test_sparse_allreduce_host_matches_device_call(okm, gpus, pinned):
    """The host-buffer allreduce returns what the device-buffer call returns."""
    import torch
    from paper_2201_07598_b200 import _lib
    L = _lib.lib()
    n, k = 40000, 400
    rng = np.random.default_rng(5)
    w_host, w_dev = okm.World(1, [0]), okm.World(1, [0])
    st = okm.OkState()
    h_idx = torch.empty(n, dtype=torch.int32).pin_memory()
    h_val = torch.empty(n, dtype=torch.float64).pin_memory()
    h_ind = torch.empty(n, dtype=torch.int32).pin_memory()
    for t in range(1, 6):
        g = rng.standard_normal(n).astype(np.float32)
        ref = okm.ok_sparse_allreduce(w_dev.ctx(0), st, g, t, k)
        res = _lib.OktResult()
        hg = _host_grad(g, pinned)
        rc = L.okt_sparse_allreduce_host(w_host.ctx(0).comm, ctypes.c_void_p(hg.data_ptr()), n, t, k,
                                         ctypes.c_void_p(h_idx.data_ptr()), ctypes.c_void_p(h_val.data_ptr()),
                                         ctypes.c_void_p(h_ind.data_ptr()), n, ctypes.byref(res), None)
        assert rc == 0, L.okt_last_error().decode()
        U = int(res.u.nnz)
        assert np.array_equal(h_idx[:U].numpy().view(np.uint32), ref.u.indices)
        assert np.array_equal(h_val[:U].numpy(), ref.u.values)
        assert np.array_equal(h_ind[:int(res.n_indexes)].numpy().view(np.uint32), ref.indexes)


@pytest.mark.parametrize("P", [2, 4])
def test_device_barrier(okm, gpus, P):
    """okt_device_barrier is collective and leaves the comms usable (peer-mapped
    worlds run it as a flag kernel, shared-GPU worlds as a host barrier)."""
    from paper_2201_07598_b200 import _lib
    L = _lib.lib()
    w = okm.World(P, [r % gpus for r in range(P)])
    for _ in range(3):
        rcs = okm.run_ranks(w, lambda ctx: L.okt_device_barrier(ctx.comm, None))
        assert rcs == [0] * P
    g = [np.random.default_rng(r).standard_normal(4096).astype(np.float32) for r in range(P)]
    st = [okm.OkState() for _ in range(P)]
    res = okm.run_ranks(w, lambda ctx: okm.ok_sparse_allreduce(ctx, st[ctx.rank], g[ctx.rank], 1, 40))
    assert all(np.array_equal(r.u.indices, res[0].u.indices) for r in res)
