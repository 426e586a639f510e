"""Device-driven P2P step in ONE process (ranks = threads, direct peer
pointers instead of CUDA IPC), with the per-CTA globaltimer trace of the last
step: isolates in-process vs cross-process flag latency.  Diagnostics only.
    OKT_P2P_TRACE=1 python tools/p2p_trace_local.py [P] [steps] [outdir]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OKT_P2P_TRACE", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_07598_b200 import _lib  # noqa: E402
from paper_2201_07598_b200 import oktopk as ok  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/p2p_local"
n = int(os.environ.get("OKT_N", "14728266"))
k = n // 100
L = _lib.lib()
w = ok.World(P, list(range(P)))
gs = [torch.empty(n, dtype=torch.float32, device=f"cuda:{r}") for r in range(P)]
ws = [torch.zeros(n, dtype=torch.float32, device=f"cuda:{r}") for r in range(P)]
for t in range(1, steps + 1):
    for r in range(P):
        with torch.cuda.device(r):
            assert L.okt_gen_drift(ctypes.c_void_p(gs[r].data_ptr()), n, t, 1, r + 1, 0, None) == 0
    for r in range(P):
        torch.cuda.synchronize(r)

    def body(ctx):
        res = _lib.OktResult()
        rc = L.okt_sgd_step(ctx.comm, ctypes.c_void_p(gs[ctx.rank].data_ptr()), ctypes.c_void_p(ws[ctx.rank].data_ptr()),
                            n, 1.0, t, k, ctypes.byref(res), None)
        assert rc == 0, L.okt_last_error().decode()
        return int(res.u.nnz)

    U = ok.run_ranks(w, body)
os.makedirs(out, exist_ok=True)
kinds, ctas = 7, 2048
for r in range(P):
    buf = (ctypes.c_uint64 * (kinds * ctas * 4))()
    rc = L.okt_debug_p2p_trace(w.ctx(r).comm, buf, kinds * ctas * 4)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(kinds, ctas, 4).astype(np.int64)
    np.save(os.path.join(out, f"p2p_trace_rank{r}.npy"), a)
    print("rank", r, "trace rc", rc, "U", U[r])
    used = a[1, :, 0] > 0
    t0 = a[0, :, 0][a[0, :, 0] > 0].min()
    for kind, nm in ((0, "k1"), (1, "merge"), (3, "pull"), (2, "restore")):
        u = a[kind, :, 0] > 0
        if u.any():
            print(f"  {nm}: start {(a[kind, u, 0].min() - t0) / 1e3:.1f} us, end {(a[kind, u, 2].max() - t0) / 1e3:.1f} us,"
                  f" waited {(a[kind, u, 1].max() - t0) / 1e3:.1f} us")
    ph = a[4][(a[4] > 0).any(axis=1)]
    if ph.size:
        print("  merge phases (median per CTA, us):", [round(float(np.median(ph[:, i])) / 1e3, 1) for i in range(4)])

