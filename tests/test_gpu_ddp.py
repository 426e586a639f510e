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
