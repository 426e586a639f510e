"""GPU robustness of the C-ABI: state handed in through okt_set_state survives
steady steps, a closed world wakes a rank blocked in an exchange, and a dead
NCCL peer turns into TransportError (never a hang).

Reference semantics: thresholds change only on refresh iterations
(proj/core/src/oktopk.cpp:258-293); InprocTransport::close() wakes every
blocked waiter with TransportError (proj/core/src/inproc.cpp:54-61); the
harness reports a failed worker instead of hanging
(proj/core/src/harness.cpp:336-344,455-462).
"""
import ctypes
import os
import socket
import threading
import time

import numpy as np
import pytest

from oracle import OrcState

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def okm(gpus):
    from paper_2201_07598_b200 import oktopk
    return oktopk


def _state(okm, P, n, local_th, global_th, t):
    st = okm.OkState(okm.ThresholdState(local_th=local_th, global_th=global_th, tau=64, tau_prime=32,
                                        last_local_eval=1, last_global_eval=1), bucket_size=4)
    st.bounds.cuts = [r * n // P for r in range(P)] + [n]
    st.t = t
    return st


def _orc_state(P, n, local_th, global_th, t):
    s = OrcState.fresh(64, 32, 4)
    s.local_th, s.global_th = local_th, global_th
    s.last_local_eval = s.last_global_eval = 1
    s.regions = P
    for r in range(P):
        s.cuts[r] = r * n // P
    s.cuts[P] = n
    s.t = t
    return s


@pytest.mark.parametrize("P", [1, 2])
def test_set_state_thresholds_survive_a_steady_step(okm, oracle, P):
    """A fresh comm resumed at a steady t (a checkpoint restore): the step must
    select with the thresholds it was given and hand them back unchanged."""
    n, k = 40_000, 400
    lth, gth = 1.25, 1.5
    w = okm.World(P, [0] * P)
    try:
        grads = [oracle.random_dense(31 + r, n) * 2.0 for r in range(P)]
        grads = [g.astype(np.float32).astype(np.float64) for g in grads]
        sts = [_state(okm, P, n, lth, gth, 5) for _ in range(P)]
        models = [okm.ModelState(np.zeros(n), 0, okm.LrSchedule(1.0)) for _ in range(P)]
        for m in models:
            m.t = 5  # the step runs at t = 6: steady for tau = 64, tau' = 32
        res = [okm.Residual(n) for _ in range(P)]
        got = okm.run_ranks(w, lambda ctx: okm.oktopk_sgd_step(ctx, models[ctx.rank], res[ctx.rank],
                                                                grads[ctx.rank], k, sts[ctx.rank]))
        orc_st = [_orc_state(P, n, lth, gth, 5) for _ in range(P)]
        eps = [np.zeros(n) for _ in range(P)]
        ws = [np.zeros(n) for _ in range(P)]
        rc, ui, uv = oracle.sgd_step(grads, eps, ws, orc_st, 1.0, 6, k)
        assert rc == 0
        for r in range(P):
            assert sts[r].th.local_th == lth and sts[r].th.global_th == gth, (r, sts[r].th)
            assert sts[r].t == 6
            assert np.array_equal(got[r].u.indices, ui) and np.array_equal(got[r].u.values, uv), r
        assert ui.size > 0
    finally:
        w.destroy()


def test_world_close_wakes_a_blocked_rank(okm):
    """Rank 0 enters a refresh step (host-synchronised exchange); rank 1 never
    arrives.  Closing the world must return TransportError to rank 0."""
    import torch
    L = okm._lib.lib()
    w = okm.World(2, [0, 0])
    out = {}
    try:
        g = torch.ones(10_000, dtype=torch.float32, device="cuda")
        ctx = w.ctx(0)

        def rank0():
            torch.cuda.set_device(0)
            res = okm._lib.OktResult()
            t0 = time.time()
            out["rc"] = L.okt_sparse_allreduce(ctx.comm, ctypes.c_void_p(g.data_ptr()), g.numel(), 1, 100,
                                               ctypes.byref(res), None)
            out["err"] = L.okt_last_error().decode()
            out["s"] = time.time() - t0

        th = threading.Thread(target=rank0)
        th.start()
        time.sleep(1.0)
        assert th.is_alive(), "rank 0 returned without its peer"
        w.close()
        th.join(timeout=30)
        assert not th.is_alive(), "okt_world_close did not wake the blocked rank"
        assert out["rc"] == 4, out  # OKT_ERR_TRANSPORT
        assert "TransportError" in out["err"] or "closed" in out["err"], out
    finally:
        w.destroy()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dead_peer_worker(rank, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        os.environ["OKT_NCCL_TIMEOUT_MS"] = "4000"
        import torch
        import torch.distributed as dist
        from paper_2201_07598_b200 import _lib
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(rank)
        L = _lib.lib()
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            assert L.okt_nccl_unique_id(uid, 128) == 0
        obj = [bytes(uid)] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        ctypes.memmove(uid, obj[0], 128)
        comm = ctypes.c_void_p()
        assert L.okt_comm_init_nccl(ctypes.byref(comm), rank, 2, rank, uid, 128) == 0, L.okt_last_error()
        assert L.okt_set_params(comm, 8, 4, 4) == 0
        n, k = 100_000, 1_000
        gen = torch.Generator().manual_seed(7 + rank)
        g = torch.randn(n, generator=gen).cuda()
        wm = torch.zeros(n, device="cuda")
        res = _lib.OktResult()
        for t in range(1, 5):  # t = 1 refresh, 2..4 steady
            rc = L.okt_sgd_step(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(wm.data_ptr()), n, 1.0, t, k,
                                ctypes.byref(res), None)
            assert rc == 0, L.okt_last_error()
        dist.barrier()
        if rank == 1:
            q.put((rank, "exited", None))
            q.close()
            q.join_thread()  # (os._exit skips the queue's feeder thread)
            os._exit(0)  # the peer dies before the t = 5 refresh
        time.sleep(0.5)
        t0 = time.time()
        rc = L.okt_sgd_step(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(wm.data_ptr()), n, 1.0, 5, k,
                            ctypes.byref(res), None)
        dt = time.time() - t0
        err = L.okt_last_error().decode()
        t1 = time.time()
        rc2 = L.okt_sgd_step(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(wm.data_ptr()), n, 1.0, 6, k,
                             ctypes.byref(res), None)
        dt2 = time.time() - t1
        q.put((rank, (rc, dt, err, rc2, dt2), None))
        q.close()
        q.join_thread()
        os._exit(0)  # (no collective teardown with a dead peer)
    except Exception:
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_nccl_dead_peer_is_a_transport_error(gpus):
    if gpus < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    for attempt in range(3):  # (a rendezvous port taken in between is retried on a fresh one)
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_dead_peer_worker, args=(r, port, q), daemon=True) for r in range(2)]
        for p in procs:
            p.start()
        results, errs = dict(), []
        try:
            for _ in range(2):
                r, v, err = q.get(timeout=300)
                if err is not None:
                    errs.append(err)
                    break
                results[r] = v
        finally:
            for p in procs:
                p.join(timeout=30)
                if p.is_alive():
                    p.kill()
        if errs and "EADDRINUSE" in errs[0] and attempt < 2:
            continue
        assert not errs, errs[0]
        break
    rc, dt, err, rc2, dt2 = results[0]
    assert rc == 4, (rc, err)  # OKT_ERR_TRANSPORT
    assert "TransportError" in err, err
    assert dt < 60, dt  # bounded by OKT_NCCL_TIMEOUT_MS (4 s) or the P2P bound (20 s)
    assert rc2 == 4 and dt2 < 30, (rc2, dt2)  # the comm stays failed: the next call fails at once
