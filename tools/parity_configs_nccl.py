#!/usr/bin/env python3
"""Per-call parity of the production multi-GPU path (one process per GPU,
okt_comm_init_nccl: device-driven NVLink P2P steady steps, NCCL refreshes)
against the reference itself (oracle/_ref/libokref.so) at a BASELINE config.

Each rank runs the fp32 error-feedback loop on its GPU (acc = eps + g,
ok_sparse_allreduce(acc), eps = acc zeroed at indexes; trainer.cpp:466-488)
on drifting_gradient_process(t, seed = 1, rank_key = r + 1); rank 0 gathers
every rank's acc, runs the reference's ok_sparse_allreduce (oktopk.cpp:246-307)
on them with the same prior states, and broadcasts the expected u, indexes,
local_selected, states and ledgers; every rank asserts bit-equality per call.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/parity_configs_nccl.py --n 14728266 --density 0.01 --iters 34 [--out FILE]
"""
import argparse
import ctypes
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", "--elements", dest="n", type=int, default=14_728_266)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--iters", type=int, default=34)
    ap.add_argument("--tau", type=int, default=64)
    ap.add_argument("--tau-prime", type=int, default=32)
    ap.add_argument("--bucket", type=int, default=4)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from oracle import OrcState, Reference
    from paper_2201_07598_b200 import _lib, oktopk as okm

    rank, P, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    L = _lib.lib()
    uid = (ctypes.c_char * 128)()
    if rank == 0:
        assert L.okt_nccl_unique_id(uid, 128) == 0
    obj = [bytes(uid)] if rank == 0 else [None]
    dist.broadcast_object_list(obj, src=0)
    ctypes.memmove(uid, obj[0], 128)
    comm = ctypes.c_void_p()
    assert L.okt_comm_init_nccl(ctypes.byref(comm), rank, P, local, uid, 128) == 0, L.okt_last_error()
    ctx = okm.WorkerCtx(comm.value, rank, P, local)
    n = a.n
    k = max(1, min(n, int(math.ceil(a.density * float(n) * (1.0 - 1e-12)))))
    st = okm.OkState(okm.ThresholdState(tau=a.tau, tau_prime=a.tau_prime), bucket_size=a.bucket)
    ref = Reference() if rank == 0 else None
    st_ref = [OrcState.fresh(a.tau, a.tau_prime, a.bucket) for _ in range(P)]
    led_ref = np.zeros((P, 6, 4), np.uint64)
    eps = torch.zeros(n, dtype=torch.float32, device="cuda")
    acc = torch.empty(n, dtype=torch.float32, device="cuda")
    log = []
    ok_all = True
    for t in range(1, a.iters + 1):
        assert L.okt_gen_drift(ctypes.c_void_p(acc.data_ptr()), n, t, 1, rank + 1, 0, None) == 0
        torch.cuda.synchronize()
        acc.add_(eps)
        torch.cuda.synchronize()
        mine = acc.cpu().numpy()
        gathered = [None] * P if rank == 0 else None
        dist.gather_object(mine, gathered, dst=0)
        want = None
        t_ref = 0.0
        if rank == 0:
            t0 = time.time()
            rc, want = ref.ok_sparse_allreduce([x.astype(np.float64) for x in gathered], st_ref, t, k, led_ref)
            t_ref = time.time() - t0
            assert rc == 0
            want["states"] = [(s.local_th, s.global_th, s.last_local_eval, s.last_global_eval, s.cuts_list(), s.t)
                              for s in st_ref]
            want["ledger"] = led_ref.copy()
        box = [want]
        dist.broadcast_object_list(box, src=0)
        want = box[0]
        t0 = time.time()
        got = okm.ok_sparse_allreduce(ctx, st, acc, t, k)
        t_gpu = time.time() - t0
        led = np.zeros((6, 4), np.uint64)
        for ph in range(6):
            c = okm._lib.OktCounters()
            assert L.okt_ledger(comm, ph, ctypes.byref(c)) == 0
            led[ph] = (c.words_sent, c.words_recv, c.msgs_sent, c.msgs_recv)
        s_ref = want["states"][rank]
        checks = {
            "u_idx": bool(np.array_equal(got.u.indices, want["u_idx"])),
            "u_val": bool(np.array_equal(got.u.values, want["u_val"])),
            "indexes": bool(np.array_equal(got.indexes, want["indexes"][rank])),
            "local_selected": got.local_selected == want["local_selected"][rank],
            "state": (st.th.local_th, st.th.global_th, st.th.last_local_eval, st.th.last_global_eval,
                      st.bounds.cuts, st.t) == tuple(s_ref),
            "ledger": bool(np.array_equal(led, want["ledger"][rank])),
        }
        ok = all(checks.values())
        ok_all &= ok
        log.append({"t": t, "rank": rank, "U": int(want["u_idx"].size), "ok": ok,
                    "failed": [k_ for k_, v in checks.items() if not v], "ref_s": round(t_ref, 3),
                    "gpu_s": round(t_gpu, 4)})
        eps.copy_(acc)
        if got.indexes.size:
            eps.index_fill_(0, torch.from_numpy(got.indexes.astype(np.int64)).cuda(), 0.0)
    logs = [None] * P if rank == 0 else None
    dist.gather_object(log, logs, dst=0)
    oks = [None] * P if rank == 0 else None
    dist.gather_object(ok_all, oks, dst=0)
    if rank == 0:
        summary = {"tool": "parity_configs_nccl", "n": n, "k": k, "P": P, "iters": a.iters, "tau": a.tau,
                   "tau_prime": a.tau_prime, "bucket": a.bucket, "all_bit_exact": all(oks),
                   "per_call": [e for lg in logs for e in lg]}
        line = json.dumps(summary)
        print(json.dumps({k_: v for k_, v in summary.items() if k_ != "per_call"}))
        if a.out:
            with open(a.out, "w") as f:
                f.write(line + "\n")
    L.okt_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok_all else 1


if __name__ == "__main__":
    sys.exit(main())
