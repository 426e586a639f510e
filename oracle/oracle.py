"""ctypes bindings of the oracle libraries (test infrastructure only)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import (POINTER, Structure, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8,
                    c_size_t, c_uint32, c_uint64, c_void_p)
from typing import List, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "_build", "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libokref.so")
MAX_P = 8
PHASES = 6


class OrcState(Structure):
    """orc_state / okref_state / okt_state share this layout."""
    _fields_ = [
        ("local_th", c_double), ("global_th", c_double),
        ("tau", c_uint32), ("tau_prime", c_uint32),
        ("last_local_eval", c_int64), ("last_global_eval", c_int64),
        ("regions", c_int32), ("bucket_size", c_uint32),
        ("cuts", c_uint64 * (MAX_P + 1)), ("t", c_int64),
    ]

    @classmethod
    def fresh(cls, tau: int = 64, tau_prime: int = 32, bucket: int = 4) -> "OrcState":
        s = cls()
        s.tau, s.tau_prime, s.bucket_size = tau, tau_prime, bucket
        s.last_local_eval = s.last_global_eval = -1
        s.regions = -1
        return s

    def cuts_list(self) -> List[int]:
        return [int(self.cuts[i]) for i in range(self.regions + 1)] if self.regions >= 0 else []


class Counters(Structure):
    _fields_ = [("words_sent", c_uint64), ("words_recv", c_uint64), ("msgs_sent", c_uint64),
                ("msgs_recv", c_uint64)]


def build() -> None:
    """Compile liborc.so (and libokref.so where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def orc_available() -> bool:
    return os.path.exists(ORC_PATH)


def have_reference() -> bool:
    return os.path.exists(REF_PATH)


def _ptrs(arrs, ctype):
    return (POINTER(ctype) * len(arrs))(*[a.ctypes.data_as(POINTER(ctype)) for a in arrs])


class _Common:
    """Shared ok_sparse_allreduce driver for the restatement and the reference."""
    _fn_allreduce = None
    _fn_wire_enc = None
    _fn_wire_dec = None

    def wire_encode(self, idx: np.ndarray, val: np.ndarray) -> bytes:
        """wire_encode (sparse.cpp:275-285): [nnz u32][idx u32][f32 values]."""
        idx = np.ascontiguousarray(idx, dtype=np.uint32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        out = np.zeros(4 + 8 * idx.size, np.uint8)
        getattr(self.L, self._fn_wire_enc)(*self._wire_enc_args(idx, val, out))
        return out.tobytes()

    def wire_decode(self, b: bytes, n: int):
        """wire_decode (sparse.cpp:287-310): (indices, values), or None for a
        malformed image (DecodeError)."""
        buf = np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8)
        cap = max(1, len(b) // 4)
        idx = np.zeros(cap, np.uint32)
        val = np.zeros(cap, np.float64)
        nnz = c_size_t(0)
        rc = getattr(self.L, self._fn_wire_dec)(buf.ctypes.data_as(POINTER(c_uint8)), c_size_t(len(b)), c_size_t(n),
                                                 idx.ctypes.data_as(POINTER(c_uint32)),
                                                 val.ctypes.data_as(POINTER(c_double)), ctypes.byref(nnz))
        if rc:
            return None
        return idx[:nnz.value].copy(), val[:nnz.value].copy()

    def ok_sparse_allreduce(self, inputs: Sequence[np.ndarray], states: Sequence[OrcState], t: int, k: int,
                            ledger: np.ndarray = None):
        P = len(inputs)
        n = int(inputs[0].size)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        st = (OrcState * P)(*states)
        led = (Counters * (P * PHASES))()
        cap = max(n, 1)
        u_idx = np.zeros(cap, np.uint32)
        u_val = np.zeros(cap, np.float64)
        U = c_size_t()
        ix = [np.zeros(cap, np.uint32) for _ in range(P)]
        nix = (c_size_t * P)()
        sel = (c_size_t * P)()
        rc = self._call(P, _ptrs(g, c_double), n, t, k, st, led, u_idx, u_val, U, _ptrs(ix, c_uint32), nix, sel)
        for r in range(P):
            ctypes.memmove(ctypes.addressof(states[r]), ctypes.addressof(st[r]), ctypes.sizeof(OrcState))
        if ledger is not None:
            for r in range(P):
                for ph in range(PHASES):
                    c = led[r * PHASES + ph]
                    ledger[r, ph] += np.array((c.words_sent, c.words_recv, c.msgs_sent, c.msgs_recv), dtype=ledger.dtype)
        if rc:
            return rc, None
        U = U.value
        return 0, dict(u_idx=u_idx[:U].copy(), u_val=u_val[:U].copy(),
                       indexes=[ix[r][:nix[r]].copy() for r in range(P)],
                       local_selected=[int(sel[r]) for r in range(P)])


class Oracle(_Common):
    """The plain-C restatement (okt_oracle.c)."""

    @staticmethod
    def _wire_enc_args(idx, val, out):
        return (idx.ctypes.data_as(POINTER(c_uint32)), val.ctypes.data_as(POINTER(c_double)), c_size_t(idx.size),
                out.ctypes.data_as(POINTER(c_uint8)))

    def __init__(self, path: str = ORC_PATH):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        self.L = L
        L.orc_kth_largest_mag.restype = c_double
        L.orc_kth_largest_mag.argtypes = [POINTER(c_double), c_size_t, c_size_t]
        L.orc_select.restype = c_size_t
        L.orc_select.argtypes = [POINTER(c_double), c_size_t, c_double, POINTER(c_uint32), POINTER(c_double)]
        L.orc_sparse_sum.restype = c_size_t
        L.orc_topk_exact.restype = c_size_t
        L.orc_topk_exact.argtypes = [POINTER(c_double), c_size_t, c_size_t, POINTER(c_uint32), POINTER(c_double)]
        L.orc_topka_allreduce.restype = c_size_t
        L.orc_gtopk_allreduce.restype = c_size_t
        L.orc_topkdsa_allreduce.restype = c_size_t
        L.orc_gaussiank_allreduce.restype = c_size_t
        L.orc_dense_allreduce.restype = None
        L.orc_gaussian_threshold.restype = c_double
        L.orc_gaussian_threshold.argtypes = [POINTER(c_double), c_size_t, c_size_t, c_int]
        L.orc_space_repartition.restype = None
        L.orc_ok_sparse_allreduce.restype = c_int
        L.orc_sgd_step.restype = c_int
        L.orc_random_dense.restype = None
        L.orc_random_dense.argtypes = [c_uint64, c_size_t, POINTER(c_double)]
        L.orc_random_int_dense.restype = None
        L.orc_random_int_dense.argtypes = [c_uint64, c_size_t, c_int, POINTER(c_double)]
        L.orc_drift.restype = c_int
        L.orc_drift.argtypes = [c_int64, c_uint64, c_size_t, c_uint64, c_int, POINTER(c_double)]
        L.orc_equal_slice_ends.restype = None
        L.orc_equal_slice_ends.argtypes = [c_uint64, c_int, POINTER(c_uint64)]
        L.orc_wire_encode.restype = None
        L.orc_wire_encode.argtypes = [POINTER(c_uint32), POINTER(c_double), c_size_t, POINTER(c_uint8)]
        L.orc_wire_decode.restype = c_int
        L.orc_wire_decode.argtypes = [POINTER(c_uint8), c_size_t, c_size_t, POINTER(c_uint32), POINTER(c_double),
                                      POINTER(c_size_t)]
        self._fn_wire_enc, self._fn_wire_dec = "orc_wire_encode", "orc_wire_decode"

    def _call(self, P, g, n, t, k, st, led, u_idx, u_val, U, ix, nix, sel):
        return self.L.orc_ok_sparse_allreduce(
            c_int(P), st, g, c_size_t(n), c_int64(t), c_size_t(k), led,
            u_idx.ctypes.data_as(POINTER(c_uint32)), u_val.ctypes.data_as(POINTER(c_double)), ctypes.byref(U),
            ix, nix, sel)

    # generators
    def random_dense(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.L.orc_random_dense(seed, n, out.ctypes.data_as(POINTER(c_double)))
        return out

    def random_int_dense(self, seed: int, n: int, hi: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.L.orc_random_int_dense(seed, n, hi, out.ctypes.data_as(POINTER(c_double)))
        return out

    def drift(self, t: int, seed: int, n: int, rank_key: int = 0, fixed_positions: bool = False) -> np.ndarray:
        out = np.empty(n, np.float64)
        rc = self.L.orc_drift(t, seed, n, rank_key, int(fixed_positions), out.ctypes.data_as(POINTER(c_double)))
        if rc:
            raise ValueError("drift: t must be >= 1")
        return out

    # primitives
    def kth_largest_mag(self, v: np.ndarray, k: int) -> float:
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.L.orc_kth_largest_mag(v.ctypes.data_as(POINTER(c_double)), v.size, k)

    def select(self, g: np.ndarray, th: float):
        g = np.ascontiguousarray(g, dtype=np.float64)
        idx = np.empty(max(g.size, 1), np.uint32)
        val = np.empty(max(g.size, 1), np.float64)
        m = self.L.orc_select(g.ctypes.data_as(POINTER(c_double)), g.size, th,
                              idx.ctypes.data_as(POINTER(c_uint32)), val.ctypes.data_as(POINTER(c_double)))
        return idx[:m].copy(), val[:m].copy()

    def sparse_sum(self, parts: Sequence[tuple]):
        P = len(parts)
        idx = [np.ascontiguousarray(p[0], dtype=np.uint32) for p in parts]
        val = [np.ascontiguousarray(p[1], dtype=np.float64) for p in parts]
        nnz = (c_size_t * P)(*[i.size for i in idx])
        tot = max(sum(i.size for i in idx), 1)
        oi = np.empty(tot, np.uint32)
        ov = np.empty(tot, np.float64)
        m = self.L.orc_sparse_sum(c_int(P), _ptrs(idx, c_uint32), _ptrs(val, c_double), nnz,
                                  oi.ctypes.data_as(POINTER(c_uint32)), ov.ctypes.data_as(POINTER(c_double)))
        return oi[:m].copy(), ov[:m].copy()

    def topk_exact(self, g: np.ndarray, k: int):
        g = np.ascontiguousarray(g, dtype=np.float64)
        idx = np.empty(max(k, 1), np.uint32)
        val = np.empty(max(k, 1), np.float64)
        m = self.L.orc_topk_exact(g.ctypes.data_as(POINTER(c_double)), g.size, k,
                                  idx.ctypes.data_as(POINTER(c_uint32)), val.ctypes.data_as(POINTER(c_double)))
        return idx[:m].copy(), val[:m].copy()

    def topka_allreduce(self, inputs: Sequence[np.ndarray], k: int):
        P = len(inputs)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        oi = np.empty(max(P * k, 1), np.uint32)
        ov = np.empty(max(P * k, 1), np.float64)
        m = self.L.orc_topka_allreduce(c_int(P), _ptrs(g, c_double), c_size_t(g[0].size), c_size_t(k),
                                       oi.ctypes.data_as(POINTER(c_uint32)), ov.ctypes.data_as(POINTER(c_double)))
        return oi[:m].copy(), ov[:m].copy()

    def baseline(self, which: str, inputs: Sequence[np.ndarray], k: int, scale_to_floor: bool = True,
                 ledger: np.ndarray = None):
        """gtopk / topkdsa / gaussiank allreduce of P dense inputs (rank 0's result)."""
        P = len(inputs)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        n = g[0].size
        cap = max(P * n, 1)
        oi = np.empty(cap, np.uint32)
        ov = np.empty(cap, np.float64)
        led = ledger if ledger is not None else np.zeros((P, 6, 4), np.uint64)
        lp = led.ctypes.data_as(POINTER(Counters))
        args = (c_int(P), _ptrs(g, c_double), c_size_t(n), c_size_t(k))
        outs = (oi.ctypes.data_as(POINTER(c_uint32)), ov.ctypes.data_as(POINTER(c_double)), lp)
        if which == "gtopk":
            m = self.L.orc_gtopk_allreduce(*args, *outs)
        elif which == "topkdsa":
            m = self.L.orc_topkdsa_allreduce(*args, *outs)
        elif which == "gaussiank":
            m = self.L.orc_gaussiank_allreduce(*args, c_int(int(scale_to_floor)), *outs)
        else:
            raise ValueError(which)
        return oi[:m].copy(), ov[:m].copy()

    def dense_allreduce(self, inputs: Sequence[np.ndarray], ledger: np.ndarray = None) -> np.ndarray:
        P = len(inputs)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        out = np.empty(max(g[0].size, 1), np.float64)
        led = ledger if ledger is not None else np.zeros((P, 6, 4), np.uint64)
        self.L.orc_dense_allreduce(c_int(P), _ptrs(g, c_double), c_size_t(g[0].size),
                                   out.ctypes.data_as(POINTER(c_double)), led.ctypes.data_as(POINTER(Counters)))
        return out[:g[0].size].copy()

    def gaussian_threshold(self, g: np.ndarray, k: int, scale_to_floor: bool = True) -> float:
        g = np.ascontiguousarray(g, dtype=np.float64)
        return self.L.orc_gaussian_threshold(g.ctypes.data_as(POINTER(c_double)), g.size, k, int(scale_to_floor))

    def space_repartition(self, sels: Sequence[np.ndarray], n: int, ledger: np.ndarray = None) -> List[int]:
        P = len(sels)
        s = [np.ascontiguousarray(x, dtype=np.uint32) for x in sels]
        m = (c_size_t * P)(*[x.size for x in s])
        cuts = (c_uint64 * (P + 1))()
        led = (Counters * (P * PHASES))()
        self.L.orc_space_repartition(c_int(P), _ptrs(s, c_uint32), m, c_uint64(n), cuts, led)
        if ledger is not None:
            for r in range(P):
                for ph in range(PHASES):
                    c = led[r * PHASES + ph]
                    ledger[r, ph] += np.array((c.words_sent, c.words_recv, c.msgs_sent, c.msgs_recv), dtype=ledger.dtype)
        return [int(c) for c in cuts]

    def equal_slice_ends(self, n: int, P: int) -> List[int]:
        e = (c_uint64 * (P + 1))()
        self.L.orc_equal_slice_ends(n, P, e)
        return [int(x) for x in e]

    def sgd_step(self, grads, eps, ws, states, alpha: float, t: int, k: int, ledger: np.ndarray = None):
        """In-place on eps / ws (lists of float64 arrays)."""
        P = len(grads)
        n = int(grads[0].size)
        st = (OrcState * P)(*states)
        led = (Counters * (P * PHASES))()
        u_idx = np.zeros(max(n, 1), np.uint32)
        u_val = np.zeros(max(n, 1), np.float64)
        U = c_size_t()
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in grads]
        rc = self.L.orc_sgd_step(c_int(P), st, _ptrs(g, c_double), _ptrs(eps, c_double), _ptrs(ws, c_double),
                                 c_size_t(n), c_double(alpha), c_int64(t), c_size_t(k), led,
                                 u_idx.ctypes.data_as(POINTER(c_uint32)), u_val.ctypes.data_as(POINTER(c_double)),
                                 ctypes.byref(U))
        for r in range(P):
            ctypes.memmove(ctypes.addressof(states[r]), ctypes.addressof(st[r]), ctypes.sizeof(OrcState))
        if ledger is not None:
            for r in range(P):
                for ph in range(PHASES):
                    c = led[r * PHASES + ph]
                    ledger[r, ph] += np.array((c.words_sent, c.words_recv, c.msgs_sent, c.msgs_recv), dtype=ledger.dtype)
        return rc, u_idx[:U.value].copy(), u_val[:U.value].copy()


class Reference(_Common):
    """The reference implementation itself (oracle/_ref/libokref.so)."""

    @staticmethod
    def _wire_enc_args(idx, val, out):
        n = int(idx.max()) + 1 if idx.size else 1
        return (idx.ctypes.data_as(POINTER(c_uint32)), val.ctypes.data_as(POINTER(c_double)), c_size_t(idx.size),
                c_size_t(n), out.ctypes.data_as(POINTER(c_uint8)))

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        L = ctypes.CDLL(path)
        self.L = L
        L.okref_allreduce.restype = c_int
        L.okref_topka.restype = c_int
        L.okref_baseline.restype = c_int
        L.okref_dense.restype = c_int
        L.okref_gaussian_threshold.restype = c_double
        L.okref_gaussian_threshold.argtypes = [POINTER(c_double), c_size_t, c_size_t, c_int]
        L.okref_th_re_evaluate_dense.restype = c_double
        L.okref_th_re_evaluate_dense.argtypes = [POINTER(c_double), c_size_t, c_size_t]
        L.okref_drift_f32.restype = None
        L.okref_drift_f32.argtypes = [c_int64, c_uint64, c_size_t, c_uint64, POINTER(c_double)]
        L.okref_wire_encode.restype = c_int
        L.okref_wire_encode.argtypes = [POINTER(c_uint32), POINTER(c_double), c_size_t, c_size_t, POINTER(c_uint8)]
        L.okref_wire_decode.restype = c_int
        L.okref_wire_decode.argtypes = [POINTER(c_uint8), c_size_t, c_size_t, POINTER(c_uint32), POINTER(c_double),
                                        POINTER(c_size_t)]
        self._fn_wire_enc, self._fn_wire_dec = "okref_wire_encode", "okref_wire_decode"
        L.okref_bench_sgd.restype = c_int
        L.okref_bench_sgd.argtypes = [c_int, c_size_t, c_size_t, c_int, c_int, c_uint32, c_uint32, c_uint32,
                                      c_double, c_uint64, c_int, POINTER(c_double), c_char_p, c_size_t]
        self.err = ctypes.create_string_buffer(512)

    def _call(self, P, g, n, t, k, st, led, u_idx, u_val, U, ix, nix, sel):
        return self.L.okref_allreduce(
            c_int(P), g, c_size_t(n), c_int64(t), c_size_t(k), st, led,
            u_idx.ctypes.data_as(POINTER(c_uint32)), u_val.ctypes.data_as(POINTER(c_double)), ctypes.byref(U),
            ix, nix, sel, self.err, c_size_t(512))

    def topka_allreduce(self, inputs: Sequence[np.ndarray], k: int):
        P = len(inputs)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        oi = np.empty(max(P * k, 1), np.uint32)
        ov = np.empty(max(P * k, 1), np.float64)
        U = c_size_t(0)
        rc = self.L.okref_topka(c_int(P), _ptrs(g, c_double), c_size_t(g[0].size), c_size_t(k),
                                oi.ctypes.data_as(POINTER(c_uint32)), ov.ctypes.data_as(POINTER(c_double)),
                                ctypes.byref(U), self.err, c_size_t(512))
        if rc:
            raise RuntimeError(f"okref_topka rc={rc}: {self.err.value.decode(errors='replace')}")
        return oi[:U.value].copy(), ov[:U.value].copy()

    def baseline(self, which: str, inputs: Sequence[np.ndarray], k: int, scale_to_floor: bool = True,
                 ledger: np.ndarray = None):
        P = len(inputs)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        n = g[0].size
        cap = max(P * n, 1)
        oi = np.empty(cap, np.uint32)
        ov = np.empty(cap, np.float64)
        U = c_size_t(0)
        led = ledger if ledger is not None else np.zeros((P, 6, 4), np.uint64)
        code = {"gtopk": 0, "topkdsa": 1, "gaussiank": 2 if scale_to_floor else 3}[which]
        rc = self.L.okref_baseline(c_int(code), c_int(P), _ptrs(g, c_double), c_size_t(n), c_size_t(k),
                                   oi.ctypes.data_as(POINTER(c_uint32)), ov.ctypes.data_as(POINTER(c_double)),
                                   ctypes.byref(U), led.ctypes.data_as(POINTER(Counters)), self.err, c_size_t(512))
        if rc:
            raise RuntimeError(f"okref_baseline rc={rc}: {self.err.value.decode(errors='replace')}")
        return oi[:U.value].copy(), ov[:U.value].copy()

    def dense_allreduce(self, inputs: Sequence[np.ndarray], ledger: np.ndarray = None) -> np.ndarray:
        P = len(inputs)
        g = [np.ascontiguousarray(x, dtype=np.float64) for x in inputs]
        out = np.empty(max(g[0].size, 1), np.float64)
        led = ledger if ledger is not None else np.zeros((P, 6, 4), np.uint64)
        rc = self.L.okref_dense(c_int(P), _ptrs(g, c_double), c_size_t(g[0].size),
                                out.ctypes.data_as(POINTER(c_double)), led.ctypes.data_as(POINTER(Counters)),
                                self.err, c_size_t(512))
        if rc:
            raise RuntimeError(f"okref_dense rc={rc}: {self.err.value.decode(errors='replace')}")
        return out[:g[0].size].copy()

    def gaussian_threshold(self, g: np.ndarray, k: int, scale_to_floor: bool = True) -> float:
        g = np.ascontiguousarray(g, dtype=np.float64)
        return self.L.okref_gaussian_threshold(g.ctypes.data_as(POINTER(c_double)), g.size, k, int(scale_to_floor))

    def th_re_evaluate(self, g: np.ndarray, k: int) -> float:
        g = np.ascontiguousarray(g, dtype=np.float64)
        return self.L.okref_th_re_evaluate_dense(g.ctypes.data_as(POINTER(c_double)), g.size, k)

    def drift_f32(self, t: int, seed: int, n: int, rank_key: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.L.okref_drift_f32(t, seed, n, rank_key, out.ctypes.data_as(POINTER(c_double)))
        return out

    def bench_sgd(self, P: int, n: int, k: int, warmup: int, iters: int, tau: int = 64, tau_prime: int = 32,
                  bucket: int = 4, alpha: float = 1.0, seed: int = 1, pin: bool = True) -> np.ndarray:
        ms = np.zeros(iters, np.float64)
        rc = self.L.okref_bench_sgd(P, n, k, warmup, iters, tau, tau_prime, bucket, alpha, seed, int(pin),
                                    ms.ctypes.data_as(POINTER(c_double)), self.err, 512)
        if rc:
            raise RuntimeError(f"reference bench failed ({rc}): {self.err.value.decode()}")
        return ms
