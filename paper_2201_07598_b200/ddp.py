"""PyTorch DistributedDataParallel front end for the Ok-Topk sparse allreduce
(the paper's deployment is PyTorch data parallelism,
`PAPER.md:370-375`, which the reference itself omits).

    from paper_2201_07598_b200.ddp import OkTopkHookState, oktopk_hook
    model = DistributedDataParallel(model, device_ids=[local_rank])
    model.register_comm_hook(OkTopkHookState(density=0.01), oktopk_hook)

Each DDP bucket gets its own `okt_comm` (one process per GPU over the
library's NCCL communicator and, when every rank owns a GPU, its NVLink
peer windows), its own Ok-Topk state and its own error-feedback residual,
which lives inside the comm: one `okt_sgd_step` per bucket and step runs the
fused accumulate + select kernel on the bucket's gradient (α = 1), the
exchange, and the model scatter — here into a zeroed per-bucket buffer, so
the buffer ends up holding −u/P and the hook returns u/P as the bucket's
gradient.  The optimizer then applies its learning rate to the averaged
sparse update, the usual EF-SGD arrangement.

Requirements: CUDA buckets of fp32 gradients; world size a power of two ≤ 8
(the reference's rule); the default process group initialised (any backend:
it only carries the NCCL unique id of each bucket's comm).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Dict

from . import _lib
from .oktopk import _check


@dataclass
class _Bucket:
    comm: ctypes.c_void_p
    n: int
    k: int
    t: int
    w: "object"  # torch.Tensor: the zero-based model buffer the step scatters -u/P into


@dataclass
class OkTopkHookState:
    """Per-process state of the hook: density (k = ceil(density · n) per
    bucket, as `ExperimentConfig::k`, harness.cpp:82-86), τ, τ′, bucket size
    of the ledger, and the process group that carries the comm rendezvous."""
    density: float = 0.01
    tau: int = 64
    tau_prime: int = 32
    bucket: int = 4
    process_group: object = None
    buckets: Dict[int, _Bucket] = field(default_factory=dict)

    def _comm_for(self, index: int, g) -> _Bucket:
        import torch
        import torch.distributed as dist
        b = self.buckets.get(index)
        n = g.numel()
        L = _lib.lib()
        if b is not None:
            if b.n == n:
                return b
            # DDP rebuilds its buckets once, after the first iteration: start
            # that bucket afresh (its residual restarts from zero)
            L.okt_comm_destroy(b.comm)
            del self.buckets[index]
        pg = self.process_group
        rank, P = dist.get_rank(pg), dist.get_world_size(pg)
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            _check(L.okt_nccl_unique_id(uid, 128))
        obj = [bytes(uid)] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(pg, 0) if pg is not None else 0, group=pg)
        ctypes.memmove(uid, obj[0], 128)
        comm = ctypes.c_void_p()
        _check(L.okt_comm_init_nccl(ctypes.byref(comm), rank, P, g.device.index, uid, 128))
        _check(L.okt_set_params(comm, self.tau, self.tau_prime, self.bucket))
        _check(L.okt_comm_reserve(comm, n))
        stream = ctypes.c_void_p(torch.cuda.current_stream(g.device).cuda_stream)
        _check(L.okt_residual_reset(comm, n, None, stream))
        k = max(1, min(n, int(math.ceil(self.density * float(n) * (1.0 - 1e-12)))))
        b = _Bucket(comm, n, k, 0, torch.zeros(n, dtype=torch.float32, device=g.device))
        self.buckets[index] = b
        return b

    def close(self) -> None:
        L = _lib.lib()
        for b in self.buckets.values():
            L.okt_comm_destroy(b.comm)
        self.buckets.clear()


def oktopk_hook(state: OkTopkHookState, bucket):
    """DDP comm hook: Ok-Topk sparse allreduce of the bucket's gradient with
    error feedback; the returned future holds u/P (dense)."""
    import torch
    g = bucket.buffer()
    if g.dtype != torch.float32 or not g.is_cuda:
        raise TypeError("oktopk_hook: CUDA fp32 buckets only")
    g = g.contiguous()
    b = state._comm_for(bucket.index(), g)
    b.t += 1
    b.w.zero_()
    res = _lib.OktResult()
    stream = ctypes.c_void_p(torch.cuda.current_stream(g.device).cuda_stream)
    _check(_lib.lib().okt_sgd_step(b.comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(b.w.data_ptr()), b.n, 1.0,
                                   b.t, b.k, ctypes.byref(res), stream))
    out = b.w.neg_()  # w = -u/P  ->  u/P
    fut = torch.futures.Future()
    fut.set_result(out)
    return fut
