"""Subprocess body of test_gpu_sanitizer.py (run under compute-sanitizer):
a few small Ok-Topk steps through every kernel family of the path, checked
against the oracle so a sanitizer-perturbed run is also a correct one.

    python tests/_sanitize_run.py single   # P = 1: K1 (+hist / dual / fused residual zero), radix, phase B
    python tests/_sanitize_run.py hostsync # P = 2 ranks on one GPU: split, scatter / region scan, filter, apply
    python tests/_sanitize_run.py p2p      # P = 2 ranks on one GPU, device-driven P2P step (merge, pull)
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
mode = sys.argv[1]
if mode == "p2p":
    os.environ["OKT_P2P_ALLOW_SHARED"] = "1"
    os.environ["OKT_P2P_GRID_DIV"] = "2"
    os.environ["OKT_P2P_TRACE"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import OrcState  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2201_07598_b200 import _lib  # noqa: E402
from paper_2201_07598_b200 import oktopk as ok  # noqa: E402

P = 1 if mode == "single" else 2
n, k, steps = 20_011, 200, 6
L = _lib.lib()
orc = Oracle()
w = ok.World(P, [0] * P)
for r in range(P):
    assert L.okt_set_params(w.ctx(r).comm, 4, 2, 4) == 0  # refreshes at t = 1, 3, 5; boundaries at t = 1, 5
st = [OrcState.fresh(4, 2, 4) for _ in range(P)]
eps = [np.zeros(n) for _ in range(P)]
ws = [np.zeros(n) for _ in range(P)]
d_w = [torch.zeros(n, dtype=torch.float32, device="cuda") for _ in range(P)]
for t in range(1, steps + 1):
    grads = [orc.random_int_dense(700 * t + r, n, 3) for r in range(P)]
    rc, u_idx, u_val = orc.sgd_step(grads, eps, ws, st, 1.0, t, k)
    assert rc == 0
    d_g = [torch.tensor(grads[r], dtype=torch.float32, device="cuda") for r in range(P)]
    torch.cuda.synchronize()

    def body(ctx):
        res = _lib.OktResult()
        rc = L.okt_sgd_step(ctx.comm, ctypes.c_void_p(d_g[ctx.rank].data_ptr()),
                            ctypes.c_void_p(d_w[ctx.rank].data_ptr()), n, 1.0, t, k, ctypes.byref(res), None)
        assert rc == 0, L.okt_last_error().decode()
        u = ok._sparse_from(res.u, n)
        return u.indices, u.values

    got = ok.run_ranks(w, body)
    for r in range(P):
        assert np.array_equal(got[r][0], u_idx) and np.array_equal(got[r][1], u_val), (t, r)
        assert np.array_equal(d_w[r].cpu().numpy().astype(np.float64), ws[r]), (t, r, "model")
# the plain allreduce entry (indexes, sub-phase kernels) once more
ins = [orc.random_dense(31 + r, n).astype(np.float32).astype(np.float64) for r in range(P)]
sts = [OrcState.fresh() for _ in range(P)]
rc, want = orc.ok_sparse_allreduce(ins, sts, 1, k)
got = ok.run_ranks(w, lambda ctx: ok.ok_sparse_allreduce(ctx, ok.OkState(), ins[ctx.rank], 1, k))
for r in range(P):
    assert np.array_equal(got[r].u.indices, want["u_idx"]) and np.array_equal(got[r].indexes, want["indexes"][r])
if mode == "p2p":
    kinds, ctas = 7, 2048
    buf = (ctypes.c_uint64 * (kinds * ctas * 4))()
    assert L.okt_debug_p2p_trace(w.ctx(0).comm, buf, kinds * ctas * 4) == 0
    assert np.frombuffer(buf, dtype=np.uint64).reshape(kinds, ctas, 4)[1, 0, 0] > 0, "P2P path not active"
w.destroy()
print("ok", mode)
