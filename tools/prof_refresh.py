"""Per-phase device time of Ok-Topk refresh iterations (tau' = 1: every step
refreshes the local and global thresholds; tau = 64) at VGG size, one process
per GPU over NCCL (torchrun).  Diagnostics only.
    torchrun --nproc-per-node N tools/prof_refresh.py [steps] [tau_prime]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2201_07598_b200 import lib  # noqa: E402
from paper_2201_07598_b200._lib import OktResult  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 16
taup = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rank, P, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
L = lib()
comm = ctypes.c_void_p()
if P > 1:
    dist.init_process_group("gloo", rank=rank, world_size=P)
    uid = (ctypes.c_char * 128)()
    if rank == 0:
        assert L.okt_nccl_unique_id(uid, 128) == 0
    obj = [bytes(uid)] if rank == 0 else [None]
    dist.broadcast_object_list(obj, src=0)
    ctypes.memmove(uid, obj[0], 128)
    assert L.okt_comm_init_nccl(ctypes.byref(comm), rank, P, local, uid, 128) == 0
else:
    w = ctypes.c_void_p()
    assert L.okt_world_create_local(ctypes.byref(w), 1, (ctypes.c_int * 1)(local)) == 0
    assert L.okt_comm_init_local(ctypes.byref(comm), w, 0) == 0
n = 14_728_266
k = n // 100
assert L.okt_set_params(comm, 64, taup, 4) == 0
assert L.okt_comm_reserve(comm, n) == 0
g = torch.empty(n, dtype=torch.float32, device="cuda")
wm = torch.zeros(n, dtype=torch.float32, device="cuda")
assert L.okt_residual_reset(comm, n, None, None) == 0
res = OktResult()
names = ["select", "threshold", "split", "merge", "global", "allgather", "apply", "step", "k1"]
for t in range(1, steps + 1):
    assert L.okt_gen_drift(ctypes.c_void_p(g.data_ptr()), n, t, 1, rank + 1, 0, None) == 0
    torch.cuda.synchronize()
    if t == 4:
        L.okt_set_profiling(comm, 1)
        L.okt_reset_phase_times(comm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert L.okt_sgd_step(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(wm.data_ptr()), n, 1.0, t, k,
                          ctypes.byref(res), None) == 0, L.okt_last_error()
    e1.record()
    torch.cuda.synchronize()
ms = (ctypes.c_double * 16)()
calls = (ctypes.c_uint64 * 16)()
L.okt_phase_times(comm, ms, calls)
if rank == 0:
    print(json.dumps({"P": P, "tau_prime": taup, "steps_profiled": steps - 3,
                      "phase_ms_per_step": {str(i): round(ms[i] / max(steps - 3, 1), 4) for i in range(16) if calls[i]},
                      "calls": {str(i): int(calls[i]) for i in range(16) if calls[i]}}))
L.okt_comm_destroy(comm)
