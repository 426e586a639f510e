"""GPU, one process per GPU over NCCL (the bench's multi-GPU transport):
P ranks each build an okt_comm with okt_comm_init_nccl and run an Ok-Topk
trajectory on drift inputs; every rank must match the oracle bit for bit.
Needs >= P visible GPUs (gpurun --gpus 2/4)."""
import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, P, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist
        from oracle import Oracle, OrcState
        from paper_2201_07598_b200 import _lib
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=P)
        torch.cuda.set_device(rank)
        L = _lib.lib()
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            assert L.okt_nccl_unique_id(uid, 128) == 0
        obj = [bytes(uid)] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        ctypes.memmove(uid, obj[0], 128)
        comm = ctypes.c_void_p()
        assert L.okt_comm_init_nccl(ctypes.byref(comm), rank, P, rank, uid, 128) == 0, L.okt_last_error()
        assert L.okt_set_params(comm, 8, 4, 3) == 0
        orc = Oracle()
        n, k = 200_000, 2_000
        states = [OrcState.fresh(8, 4, 3) for _ in range(P)]
        ok = True
        for t in range(1, 11):
            ins = [orc.drift(t, 2, n, r + 1).astype(np.float32).astype(np.float64) for r in range(P)]
            rc, want = orc.ok_sparse_allreduce(ins, states, t, k)
            assert rc == 0
            g = torch.from_numpy(ins[rank].astype(np.float32)).cuda()
            res = _lib.OktResult()
            rc = L.okt_sparse_allreduce(comm, ctypes.c_void_p(g.data_ptr()), n, t, k, ctypes.byref(res), None)
            assert rc == 0, L.okt_last_error()
            U = res.u.nnz
            ui = np.empty(U, np.uint32)
            uv = np.empty(U, np.float64)
            ix = np.empty(res.n_indexes, np.uint32)
            L.okt_memcpy_d2h(ui.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res.u.d_idx), 4 * U, None)
            L.okt_memcpy_d2h(uv.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res.u.d_val), 8 * U, None)
            L.okt_memcpy_d2h(ix.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res.d_indexes), 4 * ix.size, None)
            ok &= np.array_equal(ui, want["u_idx"]) and np.array_equal(uv, want["u_val"])
            ok &= np.array_equal(ix, want["indexes"][rank])
            ok &= res.local_selected == want["local_selected"][rank]
        L.okt_comm_destroy(comm)
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        import traceback
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_nccl_world_matches_oracle(gpus, P):
    if gpus < P:
        pytest.skip(f"needs {P} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(P)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in results:
        assert err is None, err
        assert ok, f"rank {rank} differs from the oracle"
