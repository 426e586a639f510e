"""Isolated region merge (split_and_reduce sub-phase) at VGG size, P ranks as
threads on one GPU: a safe target for ncu (no cross-GPU waits)."""
import ctypes
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_07598_b200 import _lib  # noqa: E402
from paper_2201_07598_b200 import oktopk as ok  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 14_728_266
L = _lib.lib()
w = ok.World(P, [0] * P)
gs = []
for r in range(P):
    g = torch.empty(n, dtype=torch.float32, device="cuda")
    assert L.okt_gen_drift(ctypes.c_void_p(g.data_ptr()), n, 3, 1, r + 1, 0, None) == 0
    gs.append(g)
th = ok.th_re_evaluate(gs[0], n // 100)
cuts = [n * q // P for q in range(P + 1)]
b = ok.RegionBoundaries(cuts)
for _ in range(iters):
    got = ok.run_ranks(w, lambda ctx: ok.split_and_reduce(ctx, gs[ctx.rank], th, b, 4).region_reduced.nnz())
torch.cuda.synchronize()
print("region nnz per rank", got)
