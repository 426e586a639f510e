"""Long-run consistency check of the device-driven P2P step: S EF-SGD steps
(okt_sgd_step, drift inputs, refresh iterations included) through the P2P
path, then the same S steps on a fresh comm with the host-synchronised NCCL
path (OKT_DISABLE_P2P); every step's u must agree bit for bit, and no step may
fail.  One process per GPU:
    torchrun --nproc-per-node N tools/stress_p2p.py [steps] [n] [density]"""
import ctypes
import json
import os
import sys
import time
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2201_07598_b200 import lib  # noqa: E402
from paper_2201_07598_b200._lib import OktResult  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
density = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
k = max(1, int(n * density))
rank, P, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo", rank=rank, world_size=P)
L = lib()


def make_comm():
    uid = (ctypes.c_char * 128)()
    if rank == 0:
        assert L.okt_nccl_unique_id(uid, 128) == 0
    obj = [bytes(uid)] if rank == 0 else [None]
    dist.broadcast_object_list(obj, src=0)
    ctypes.memmove(uid, obj[0], 128)
    c = ctypes.c_void_p()
    assert L.okt_comm_init_nccl(ctypes.byref(c), rank, P, local, uid, 128) == 0, L.okt_last_error()
    assert L.okt_set_params(c, 64, 32, 4) == 0
    assert L.okt_comm_reserve(c, n) == 0
    assert L.okt_residual_reset(c, n, None, None) == 0
    return c


def run(tag):
    comm = make_comm()
    g = torch.empty(n, dtype=torch.float32, device="cuda")
    w = torch.zeros(n, dtype=torch.float32, device="cuda")
    res = OktResult()
    sums = []
    t0 = time.perf_counter()
    for t in range(1, steps + 1):
        assert L.okt_gen_drift(ctypes.c_void_p(g.data_ptr()), n, t, 7, rank + 1, 0, None) == 0
        rc = L.okt_sgd_step(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(w.data_ptr()), n, 1.0, t, k,
                            ctypes.byref(res), None)
        if rc:
            raise SystemExit(f"[{tag}] rank {rank} step {t} failed: {L.okt_last_error().decode()}")
        U = int(res.u.nnz)
        idx = np.empty(U, np.uint32)
        val = np.empty(U, np.float64)
        if U:
            assert L.okt_memcpy_d2h(idx.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res.u.d_idx), 4 * U, None) == 0
            assert L.okt_memcpy_d2h(val.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(res.u.d_val), 8 * U, None) == 0
        sums.append((U, zlib.crc32(idx.tobytes()), zlib.crc32(val.tobytes())))
    torch.cuda.synchronize()
    wsum = zlib.crc32(w.cpu().numpy().tobytes())
    el = time.perf_counter() - t0
    L.okt_comm_destroy(comm)
    return sums, wsum, el


p2p, w_p2p, t_p2p = run("p2p")
os.environ["OKT_DISABLE_P2P"] = "1"
ref, w_ref, t_ref = run("nccl")
bad = [t + 1 for t, (a, b) in enumerate(zip(p2p, ref)) if a != b]
out = torch.tensor([len(bad), int(w_p2p != w_ref)], dtype=torch.int64)
dist.all_reduce(out)
if rank == 0:
    print(json.dumps({"P": P, "n": n, "k": k, "steps": steps, "mismatched_steps": int(out[0]),
                      "model_mismatch_ranks": int(out[1]), "first_bad_rank0": bad[:5],
                      "wall_s_p2p": round(t_p2p, 2), "wall_s_nccl": round(t_ref, 2),
                      "avg_U_rank0": float(np.mean([s[0] for s in p2p]))}))
dist.destroy_process_group()
sys.exit(1 if int(out[0]) or int(out[1]) else 0)
