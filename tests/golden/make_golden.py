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
    # gtopk / topkdsa / gaussiank (collectives.cpp:184-352; test_collectives.cpp:192-350)
    os.makedirs(os.path.join(HERE, "baselines"), exist_ok=True)
    rng = np.random.default_rng(78)
    base = {
        "gtopk_P2": ("gtopk", 2, 150, 8, True, [f32(orc.random_dense(4400 + 13 * r, 150)) for r in range(2)]),
        "gtopk_P8": ("gtopk", 8, 150, 8, True, [f32(orc.random_dense(4400 + 13 * r, 150)) for r in range(8)]),
        "gtopk_ties_P4": ("gtopk", 4, 400, 30, True, [rng.choice([-1.0, 1.0, 0.5, -0.5, 0.0], 400) for _ in range(4)]),
        "topkdsa_int_P4": ("topkdsa", 4, 120, 10, True, [orc.random_int_dense(7100 + r, 120, 50) for r in range(4)]),
        "topkdsa_cross_P4": ("topkdsa", 4, 64, 24, True,
                             [np.abs(orc.random_int_dense(8200 + 3 * r, 64, 9)) + 1.0 for r in range(4)]),
        "topkdsa_f32_P8": ("topkdsa", 8, 2000, 300, True, [f32(orc.random_dense(9100 + r, 2000)) for r in range(8)]),
        "topkdsa_cancel_P2": ("topkdsa", 2, 64, 40, True,
                              [np.where(np.arange(64) % 3 == 0, 1.0, 0.5) * s for s in (1.0, -1.0)]),
        "gaussiank_int_P4": ("gaussiank", 4, 300, 20, True, [orc.random_int_dense(6600 + r, 300, 500) for r in range(4)]),
        "gaussiank_f32_P2": ("gaussiank", 2, 4000, 40, True, [f32(orc.random_dense(6700 + r, 4000)) for r in range(2)]),
        "gaussiank_raw_P2": ("gaussiank", 2, 4000, 40, False, [f32(orc.random_dense(6800 + r, 4000)) for r in range(2)]),
    }
    for name, (which, P, n, k, sc, ins) in base.items():
        led = np.zeros((P, 6, 4), np.uint64)
        ui, uv = ref.baseline(which, ins, k, sc, led)
        th = np.array([ref.gaussian_threshold(x, k, sc) for x in ins]) if which == "gaussiank" else np.zeros(0)
        np.savez_compressed(os.path.join(HERE, "baselines", name + ".npz"), which=which, P=P, n=n, k=k,
                            scale=sc, inputs=np.stack(ins), u_idx=ui, u_val=uv, ledger=led, th=th)
    # dense_allreduce (collectives.cpp:89-150; test_collectives.cpp dense cases)
    os.makedirs(os.path.join(HERE, "dense"), exist_ok=True)
    for name, P, n in (("P2_n9", 2, 9), ("P4_n1001", 4, 1001), ("P8_n4096", 8, 4096), ("P8_n5", 8, 5)):
        ins = [f32(orc.random_dense(3100 + 7 * r, n) * (1.0 + 1000.0 * (r % 3))) for r in range(P)]
        led = np.zeros((P, 6, 4), np.uint64)
        out = ref.dense_allreduce(ins, led)
        np.savez_compressed(os.path.join(HERE, "dense", name + ".npz"), P=P, n=n, inputs=np.stack(ins), out=out,
                            ledger=led)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
