#!/usr/bin/env python3
"""Table-1 comparison on B200: Ok-Topk (ok_sparse_allreduce, steady + refresh
steps in their natural proportion) against the GPU baselines TopkA, gTopk,
TopkDSA and Gaussiank, the reference's fp64 dense allreduce (dense64) and a dense
fp32 NCCL allreduce, on the same inputs.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_baselines.py \
        [--elements n] [--density d] [--steps K] [--warmup W] [--algos a,b,..]

One process per GPU over the library's NCCL communicator.  Per algorithm and
step: device barrier, CUDA events around the call on the comm's stream, max
over ranks; the baselines are host-orchestrated (they synchronise per exchange
round, as the reference's blocking send/recv), so their time includes those
host round trips.  L2 is flushed before every step.  Prints one JSON line per
algorithm (rank 0); diagnostic tool, not the driver's bench contract.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import VGG_N, L2Flush, dist_env, k_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elements", type=int, default=VGG_N)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--algos", default="oktopk,topka,gtopk,topkdsa,gaussiank,dense64,dense")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2201_07598_b200 import lib
    from paper_2201_07598_b200._lib import OktResult, OktSparse

    rank, P, local = dist_env()
    torch.cuda.set_device(local)
    L = lib()
    if P > 1:
        dist.init_process_group("gloo", rank=rank, world_size=P)
    comm = ctypes.c_void_p()
    if P > 1:
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            assert L.okt_nccl_unique_id(uid, 128) == 0
        obj = [bytes(uid)] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        ctypes.memmove(uid, obj[0], 128)
        rc = L.okt_comm_init_nccl(ctypes.byref(comm), rank, P, local, uid, 128)
    else:
        w = ctypes.c_void_p()
        rc = L.okt_world_create_local(ctypes.byref(w), 1, (ctypes.c_int * 1)(local))
        rc = rc or L.okt_comm_init_local(ctypes.byref(comm), w, 0)
    assert rc == 0, L.okt_last_error()
    n, k = args.elements, k_for(args.elements, args.density)
    assert L.okt_set_params(comm, 64, 32, 4) == 0
    assert L.okt_comm_reserve(comm, n) == 0
    stream = torch.cuda.Stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    ring = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(8)]
    for i, buf in enumerate(ring):
        assert L.okt_gen_drift(ctypes.c_void_p(buf.data_ptr()), n, i + 1, 1, rank + 1, 0, sp) == 0
    wmodel = torch.zeros(n, dtype=torch.float32, device="cuda")
    flush = L2Flush(256 << 20)
    res, out = OktResult(), OktSparse()
    dense = torch.empty(n, dtype=torch.float32, device="cuda")

    def call(algo, t):
        g = ctypes.c_void_p(ring[(t - 1) % len(ring)].data_ptr())
        if algo == "oktopk":
            rc = L.okt_sgd_step(comm, g, ctypes.c_void_p(wmodel.data_ptr()), n, 1.0, t, k, ctypes.byref(res), sp)
        elif algo == "gaussiank":
            rc = L.okt_gaussiank_allreduce(comm, g, n, k, 1, ctypes.byref(out), sp)
        elif algo == "dense64":  # the reference's fp64 recursive-halving dense allreduce
            p = ctypes.c_void_p()
            rc = L.okt_dense_allreduce(comm, g, n, ctypes.byref(p), sp)
            if rc:
                raise SystemExit(f"dense64 failed: {L.okt_last_error().decode()}")
            return n
        elif algo == "dense":
            with torch.cuda.stream(stream):
                dense.copy_(ring[(t - 1) % len(ring)])
                if P > 1:
                    dist.all_reduce(dense, group=nccl_pg)
            return n
        else:
            rc = getattr(L, f"okt_{algo}_allreduce")(comm, g, n, k, ctypes.byref(out), sp)
        if rc:
            raise SystemExit(f"{algo} failed: {L.okt_last_error().decode()}")
        return int(res.u.nnz) if algo == "oktopk" else int(out.nnz)

    nccl_pg = None
    algos = args.algos.split(",")
    if "dense" in algos and P > 1:
        nccl_pg = dist.new_group(backend="nccl")
    for algo in algos:
        if algo == "oktopk":
            assert L.okt_residual_reset(comm, n, None, sp) == 0
        t = 0
        for _ in range(args.warmup):
            t += 1
            call(algo, t)
        ms, nnz = [], 0
        for _ in range(args.steps):
            t += 1
            flush.fill_(t & 0xff)
            torch.cuda.synchronize()
            if P > 1:
                dist.barrier()
                assert L.okt_device_barrier(comm, sp) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            nnz = call(algo, t)
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        mt = torch.tensor(ms, dtype=torch.float64)
        if P > 1:
            dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        if rank == 0:
            v = mt.tolist()
            print(json.dumps({"algo": algo, "P": P, "n": n, "k": k, "steps": args.steps,
                              "ms_mean": statistics.fmean(v), "ms_median": statistics.median(v),
                              "ms_min": min(v), "ms_max": max(v), "nnz_out": nnz}), flush=True)
    torch.cuda.synchronize()
    L.okt_comm_destroy(comm)
    if P > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
