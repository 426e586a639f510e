"""Steady Ok-Topk iterations at VGG size with P ranks as threads on ONE GPU
(host-synchronised transport, no cross-GPU waits): a safe target for ncu on
the region scan / pull kernels.  Diagnostics only.
    python tools/prof_step.py [P] [iters]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_07598_b200 import _lib  # noqa: E402
from paper_2201_07598_b200 import oktopk as ok  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
n = 14_728_266
k = n // 100
L = _lib.lib()
w = ok.World(P, [0] * P)
gs = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(P)]
states = [ok.OkState() for _ in range(P)]
for t in range(1, iters + 1):
    for r in range(P):
        assert L.okt_gen_drift(ctypes.c_void_p(gs[r].data_ptr()), n, t, 1, r + 1, 0, None) == 0
    torch.cuda.synchronize()
    res = ok.run_ranks(w, lambda ctx: ok.ok_sparse_allreduce(ctx, states[ctx.rank], gs[ctx.rank], t, k).u.nnz())
torch.cuda.synchronize()
print("u nnz per rank", res)
