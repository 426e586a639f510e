"""GPU, one process per GPU: the DistributedDataParallel comm hook
(paper_2201_07598_b200/ddp.py).  At density 1 (k = n:
every coordinate is selected, the residual stays zero) the hook must train
exactly like DDP's own mean allreduce up to fp32 rounding of the fp64 sum;
at 1% density it must run several buckets and steps and keep the model finite."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _train(rank, hook_density, steps=4, bucket_cap_mb=0.25):
    import torch
    from torch.nn.parallel import DistributedDataParallel as DDP
    from paper_2201_07598_b200.ddp import OkTopkHookState, oktopk_hook
    torch.manual_seed(1234)
    model = torch.nn.Sequential(torch.nn.Linear(64, 512), torch.nn.ReLU(), torch.nn.Linear(512, 256)).cuda()
    ddp = DDP(model, device_ids=[rank], bucket_cap_mb=bucket_cap_mb)
    st = None
    if hook_density is not None:
        st = OkTopkHookState(density=hook_density, tau=4, tau_prime=2)
        ddp.register_comm_hook(st, oktopk_hook)
    opt = torch.optim.SGD(ddp.parameters(), lr=0.05)
    gen = torch.Generator(device="cuda").manual_seed(100 + rank)
    for _ in range(steps):
        x = torch.randn(32, 64, device="cuda", generator=gen)
        y = torch.randn(32, 256, device="cuda", generator=gen)
        opt.zero_grad()
        torch.nn.functional.mse_loss(ddp(x), y).backward()
        opt.step()
    torch.cuda.synchronize()
    params = [p.detach().clone() for p in model.parameters()]
    nb = len(st.buckets) if st else 0
    if st:
        st.close()
    return params, nb


def _worker(rank, P, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=P, device_id=torch.device("cuda", rank))
        ref, _ = _train(rank, None)
        full, nb = _train(rank, 1.0)
        err = max(float((a - b).abs().max() / (b.abs().max() + 1e-12)) for a, b in zip(full, ref))
        sparse, nb2 = _train(rank, 0.01)
        finite = all(bool(torch.isfinite(p).all()) for p in sparse)
        moved = any(float((a - b).abs().max()) > 0 for a, b in zip(sparse, ref))
        dist.destroy_process_group()
        q.put((rank, err, nb, nb2, finite, moved, None))
    except Exception as e:  # pragma: no cover - reported below
        import traceback
        q.put((rank, None, 0, 0, False, False, traceback.format_exc()))


@pytest.mark.parametrize("P", [2])
def test_ddp_comm_hook(gpus, P):
    if gpus < P:
        pytest.skip(f"needs {P} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(P)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, nb, nb2, finite, moved, tb in out:
        assert tb is None, tb
        assert err < 1e-5, (rank, err)      # density 1: DDP's mean allreduce, up to fp32 rounding
        assert nb >= 2 and nb2 >= 2, (nb, nb2)  # several buckets, each with its own comm
        assert finite and moved


def test_ddp_hook_single_rank_matches_oracle(gpus, oracle):
    """The hook at density 5% on a one-process DDP world, per call against the
    oracle: each bucket's comm keeps its own Ok-Topk state and residual, so for
    every (bucket, step) the oracle's ok_sparse_allreduce on acc = eps + g
    (fp32, the residual read from the comm before the step; trainer.cpp:
    466-488 with alpha = 1) must give exactly the hook's output u / P."""
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist
    from torch.nn.parallel import DistributedDataParallel as DDP

    from oracle import OrcState
    from paper_2201_07598_b200 import _lib
    from paper_2201_07598_b200.ddp import OkTopkHookState, oktopk_hook

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        L = _lib.lib()
        torch.manual_seed(77)
        model = torch.nn.Sequential(torch.nn.Linear(64, 512), torch.nn.ReLU(), torch.nn.Linear(512, 256)).cuda()
        ddp = DDP(model, device_ids=[0], bucket_cap_mb=0.25)
        st = OkTopkHookState(density=0.05, tau=4, tau_prime=2)
        records = []

        def eps_of(comm):
            p, n = ctypes.c_void_p(), ctypes.c_size_t()
            assert L.okt_residual(comm, ctypes.byref(p), ctypes.byref(n)) == 0
            out = np.empty(n.value, np.float32)
            if n.value:
                assert L.okt_memcpy_d2h(out.ctypes.data_as(ctypes.c_void_p), p, out.nbytes, None) == 0
            return out

        def recording_hook(state, bucket):
            g = bucket.buffer().detach().float().contiguous()
            b = state._comm_for(bucket.index(), g)
            eps = eps_of(b.comm)
            fut = oktopk_hook(state, bucket)
            records.append((id(b), b.t, b.k, g.cpu().numpy().copy(), eps, fut.value().detach().cpu().numpy().copy()))
            return fut

        ddp.register_comm_hook(st, recording_hook)
        opt = torch.optim.SGD(ddp.parameters(), lr=0.05)
        gen = torch.Generator(device="cuda").manual_seed(5)
        for _ in range(5):
            x = torch.randn(32, 64, device="cuda", generator=gen)
            y = torch.randn(32, 256, device="cuda", generator=gen)
            opt.zero_grad()
            torch.nn.functional.mse_loss(ddp(x), y).backward()
            opt.step()
        torch.cuda.synchronize()
        st.close()
        states = {}
        checked = 0
        for key, t, k, g, eps, out in records:
            if t == 1:
                states[key] = OrcState.fresh(4, 2, 4)
            acc = (eps + g).astype(np.float32)  # one fp32 rounding, as fmaf(1, g, eps)
            rc, want = oracle.ok_sparse_allreduce([acc.astype(np.float64)], [states[key]], t, k)
            assert rc == 0
            exp = np.zeros_like(out)
            exp[want["u_idx"]] = want["u_val"].astype(np.float32)  # -(0 - u) in fp32 at P = 1
            assert np.array_equal(out, exp), (t, k, int((out != exp).sum()))
            assert want["u_idx"].size > 0
            checked += 1
        assert checked >= 8 and len({r[0] for r in records}) >= 2
    finally:
        dist.destroy_process_group()
