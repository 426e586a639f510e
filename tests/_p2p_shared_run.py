"""Subprocess body of test_gpu_p2p_shared.py: P ranks (threads) of one process
on fewer GPUs, with the device-driven P2P step forced on (OKT_P2P_ALLOW_SHARED
and OKT_P2P_GRID_DIV are set by the caller before the library loads).  Runs an
exact-sum EF trajectory through okt_sgd_step and compares u, the residual and
the model with the oracle every step.   python tests/_p2p_shared_run.py P GPUS"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import OrcState  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2201_07598_b200 import _lib  # noqa: E402
from paper_2201_07598_b200 import oktopk as ok  # noqa: E402

P, G = int(sys.argv[1]), int(sys.argv[2])
n, k, steps = 300_001, 3000, 14
L = _lib.lib()
orc = Oracle()
w = ok.World(P, [r % G for r in range(P)])
for r in range(P):
    assert L.okt_set_params(w.ctx(r).comm, 8, 4, 4) == 0
st = [OrcState.fresh(8, 4, 4) for _ in range(P)]
eps = [np.zeros(n) for _ in range(P)]
ws = [np.zeros(n) for _ in range(P)]
d_w = [torch.zeros(n, dtype=torch.float32, device=f"cuda:{w.devices[r]}") for r in range(P)]
for t in range(1, steps + 1):
    grads = [orc.random_int_dense(5000 * t + r, n, 3) for r in range(P)]
    rc, u_idx, u_val = orc.sgd_step(grads, eps, ws, st, 1.0, t, k)
    assert rc == 0
    d_g = [torch.tensor(grads[r], dtype=torch.float32, device=f"cuda:{w.devices[r]}") for r in range(P)]
    for r in range(P):
        torch.cuda.synchronize(w.devices[r])

    def body(ctx):
        r = ctx.rank
        res = _lib.OktResult()
        rc = L.okt_sgd_step(ctx.comm, ctypes.c_void_p(d_g[r].data_ptr()), ctypes.c_void_p(d_w[r].data_ptr()), n, 1.0,
                            t, k, ctypes.byref(res), None)
        assert rc == 0, L.okt_last_error().decode()
        u = ok._sparse_from(res.u, n)
        return u.indices, u.values

    got = ok.run_ranks(w, body)
    for r in range(P):
        assert np.array_equal(got[r][0], u_idx) and np.array_equal(got[r][1], u_val), (t, r, "u")
        assert np.array_equal(d_w[r].cpu().numpy().astype(np.float64), ws[r]), (t, r, "model")
# the device-driven path really ran: its merge kernel stamped the trace
kinds, ctas = 7, 2048
for r in range(P):
    buf = (ctypes.c_uint64 * (kinds * ctas * 4))()
    assert L.okt_debug_p2p_trace(w.ctx(r).comm, buf, kinds * ctas * 4) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(kinds, ctas, 4)
    assert a[1, 0, 0] > 0, f"rank {r}: P2P path not active"
print("ok", P, G)
