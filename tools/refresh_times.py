"""Per-step device times of EF steps at refresh iterations (and any step over
0.3 ms): torchrun --nproc-per-node N tools/refresh_times.py n density.  Diagnostics only."""
import ctypes, os, sys, json
sys.path.insert(0, '/root/repo')
import torch, torch.distributed as dist
from paper_2201_07598_b200 import lib
from paper_2201_07598_b200._lib import OktResult
rank, P, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local); dist.init_process_group("gloo", rank=rank, world_size=P)
L = lib()
uid = (ctypes.c_char * 128)()
if rank == 0: L.okt_nccl_unique_id(uid, 128)
obj = [bytes(uid)] if rank == 0 else [None]; dist.broadcast_object_list(obj, src=0); ctypes.memmove(uid, obj[0], 128)
c = ctypes.c_void_p(); assert L.okt_comm_init_nccl(ctypes.byref(c), rank, P, local, uid, 128) == 0
n = int(sys.argv[1]); k = int(n * float(sys.argv[2]))
L.okt_set_params(c, 64, 32, 4); L.okt_comm_reserve(c, n); L.okt_residual_reset(c, n, None, None)
ring = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(4)]
for i, b in enumerate(ring): L.okt_gen_drift(ctypes.c_void_p(b.data_ptr()), n, i + 1, 1, rank + 1, 0, None)
w = torch.zeros(n, dtype=torch.float32, device="cuda"); res = OktResult(); out = []
for t in range(1, 200):
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert L.okt_sgd_step(c, ctypes.c_void_p(ring[(t - 1) % 4].data_ptr()), ctypes.c_void_p(w.data_ptr()), n, 1.0, t, k, ctypes.byref(res), None) == 0
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if (t - 1) % 32 == 0 or ms > 0.3: out.append((t, round(ms, 3)))
if rank == 0: print(json.dumps(out))
