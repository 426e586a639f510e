"""Generate tests/golden/*.npz by running the REFERENCE itself (oracle/_ref,
compiled from /root/reference/proj/core/src by oracle/Makefile).

Run in the dev container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin the oracle restatement and the CUDA path on machines without
the reference (the GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Oracle, OrcState, Reference  # noqa: E402


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def record(ref, name, P, n, k, ts, inputs_at, tau, tau_prime, bucket):
    states = [OrcState.fresh(tau, tau_prime, bucket) for _ in range(P)]
    out = {"P": P, "n": n, "k": k, "ts": np.array(ts), "tau": tau, "tau_prime": tau_prime, "bucket": bucket}
    for t in ts:
        ins = [f32(inputs_at(t, r)) for r in range(P)]
        led = np.zeros((P, 6, 4), np.uint64)
        rc, res = ref.ok_sparse_allreduce(ins, states, t, k, led)
        assert rc == 0
        out[f"in_t{t}"] = np.stack(ins)
        out[f"u_idx_t{t}"] = res["u_idx"]
        out[f"u_val_t{t}"] = res["u_val"]
        for r in range(P):
            out[f"ix_t{t}_r{r}"] = res["indexes"][r]
        out[f"sel_t{t}"] = np.array(res["local_selected"], np.uint64)
        out[f"ledger_t{t}"] = led
        out[f"state_t{t}"] = np.stack([np.frombuffer(bytes(s), np.uint8) for s in states])
    np.savez_compressed(os.path.join(HERE, name), **out)


def main():
    ref = Reference()
    orc = Oracle()
    # acceptance.cpp criterion 1 instances (tau = tau' = 1, t = 1)
    for m in (0, 1, 2, 7, 8, 17):
        P = [2, 4, 8][m % 3]
        n = [64, 1000][(m // 3) % 2]
        k = [4, 16, 32][(m // 6) % 3]
        seed = 1000 + m
        record(ref, f"c1_m{m}.npz", P, n, k, [1], lambda t, r: orc.random_dense(seed * 8 + r, n), 1, 1, 4)
    # test_oktopk.cpp:277-330 (t = 1, n = 64, k = 6, seeds 2026 + 11r)
    for P in (2, 4):
        record(ref, f"t1_P{P}.npz", P, 64, 6, [1], lambda t, r: orc.random_dense(2026 + 11 * r, 64), 64, 32, 4)
    # drift trajectory: refreshes (tau = 8, tau' = 4), bucket 3, learned cuts
    record(ref, "drift_P4.npz", 4, 3000, 30, list(range(1, 13)), lambda t, r: ref.drift_f32(t, 5, 3000, r + 1),
           8, 4, 3)
    # skewed balance (all heavy mass in region 0)
    def skew(t, r):
        g = f32(orc.random_dense(50 + r + 10 * t, 2048)) * 1e-3
        g[:256] += 1.0 + 0.001 * r
        return g
    record(ref, "skew_P4.npz", 4, 2048, 64, [1, 2, 3], skew, 2, 1, 4)
    # topka_allreduce (collectives.cpp:152-159; test_collectives.cpp:167-190)
    os.makedirs(os.path.join(HERE, "topka"), exist_ok=True)
    rng = np.random.default_rng(77)
    topka = {
        "int_P4": (4, 200, 12, [orc.random_int_dense(900 + r, 200, 1000) for r in range(4)]),
        "f32_P2": (2, 1000, 37, [f32(orc.random_dense(300 + r, 1000)) for r in range(2)]),
        "ties_P8": (8, 512, 40, [rng.choice([-1.0, 1.0, 0.5, -0.5, 0.0, 0.25], 512) for _ in range(8)]),
        "kn_P2": (2, 64, 64, [f32(orc.random_dense(400 + r, 64)) for r in range(2)]),
        "k1_P1": (1, 300, 1, [f32(orc.random_dense(500, 300))]),
    }
    for name, (P, n, k, ins) in topka.items():
        ui, uv = ref.topka_allreduce(ins, k)
        np.savez_compressed(os.path.join(HERE, "topka", name + ".npz"), P=P, n=n, k=k, inputs=np.stack(ins),
                            u_idx=ui, u_val=uv)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
