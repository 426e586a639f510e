"""ctypes binding of the in-tree C-ABI library ``libokt.so`` (include/okt.h).

The product path is the CUDA library; this module only declares its
signatures.  There is no fallback: if the library is missing the import of the
hot-path API fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int,
                    c_int32, c_int64, c_size_t, c_uint32, c_uint64, c_void_p)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OKT_LIB_PATH") or os.path.join(HERE, "libokt.so")  # (override: diagnostics A/B builds)

OKT_MAX_WORLD = 8
OKT_T_COUNT = 9
TIMER_NAMES = ("select", "threshold", "split", "merge", "global", "allgather",
               "apply", "step", "k1")

# Every symbol include/okt.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "okt_abi_version", "okt_status_string", "okt_last_error",
    "okt_world_create_local", "okt_world_close", "okt_world_destroy",
    "okt_comm_init_local", "okt_nccl_unique_id", "okt_comm_init_nccl",
    "okt_comm_destroy", "okt_comm_info", "okt_comm_reserve",
    "okt_get_state", "okt_set_state", "okt_set_params", "okt_ledger",
    "okt_ledger_reset", "okt_sparse_allreduce", "okt_residual_reset",
    "okt_residual", "okt_sgd_step", "okt_sparse_allreduce_host",
    "okt_sparse_allreduce_async", "okt_sgd_step_async", "okt_step_wait", "okt_device_barrier",
    "okt_sgd_step_host", "okt_memcpy_h2d", "okt_memcpy_d2h",
    "okt_th_re_evaluate_dense", "okt_th_re_evaluate_sparse",
    "okt_select_by_threshold", "okt_space_repartition",
    "okt_split_and_reduce", "okt_balance_and_allgatherv", "okt_topka_allreduce", "okt_gtopk_allreduce", "okt_dense_allreduce",
    "okt_topkdsa_allreduce", "okt_gaussiank_threshold", "okt_gaussiank_allreduce",
    "okt_set_profiling", "okt_phase_times", "okt_phase_bytes", "okt_reset_phase_times",
    "okt_kernel_launches", "okt_debug_p2p_trace", "okt_wire_encode", "okt_wire_decode", "okt_gen_random_dense", "okt_gen_drift",
    "okt_plan_cuts", "okt_plan_balance", "okt_plan_ledger",
)


class OktState(Structure):
    _fields_ = [
        ("local_th", c_double),
        ("global_th", c_double),
        ("tau", c_uint32),
        ("tau_prime", c_uint32),
        ("last_local_eval", c_int64),
        ("last_global_eval", c_int64),
        ("regions", c_int32),
        ("bucket_size", c_uint32),
        ("cuts", c_uint64 * (OKT_MAX_WORLD + 1)),
        ("t", c_int64),
    ]


class OktCounters(Structure):
    _fields_ = [(n, c_uint64) for n in ("words_sent", "words_recv", "msgs_sent",
                                         "msgs_recv", "bytes_sent", "bytes_recv")]


class OktSparse(Structure):
    _fields_ = [("d_idx", c_void_p), ("d_val", c_void_p), ("nnz", c_uint64),
                ("n", c_uint64)]


class OktPiece(Structure):
    _fields_ = [("peer", c_int32), ("begin", c_uint64), ("end", c_uint64)]


class OktResult(Structure):
    _fields_ = [("u", OktSparse), ("d_indexes", c_void_p), ("n_indexes", c_uint64),
                ("local_selected", c_uint64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libokt.so (once).  Raises ImportError when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; g.build()\"`"
            " (the CUDA library is the only implementation; there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P = POINTER
    sig = {
        "okt_abi_version": (c_int, []),
        "okt_status_string": (c_char_p, [c_int]),
        "okt_last_error": (c_char_p, []),
        "okt_world_create_local": (c_int, [P(c_void_p), c_int, P(c_int)]),
        "okt_world_close": (c_int, [c_void_p]),
        "okt_world_destroy": (c_int, [c_void_p]),
        "okt_comm_init_local": (c_int, [P(c_void_p), c_void_p, c_int]),
        "okt_nccl_unique_id": (c_int, [c_void_p, c_size_t]),
        "okt_comm_init_nccl": (c_int, [P(c_void_p), c_int, c_int, c_int, c_void_p, c_size_t]),
        "okt_comm_destroy": (c_int, [c_void_p]),
        "okt_comm_info": (c_int, [c_void_p, P(c_int), P(c_int), P(c_int)]),
        "okt_comm_reserve": (c_int, [c_void_p, c_size_t]),
        "okt_get_state": (c_int, [c_void_p, P(OktState)]),
        "okt_set_state": (c_int, [c_void_p, P(OktState)]),
        "okt_set_params": (c_int, [c_void_p, c_uint32, c_uint32, c_uint32]),
        "okt_ledger": (c_int, [c_void_p, c_int, P(OktCounters)]),
        "okt_ledger_reset": (c_int, [c_void_p]),
        "okt_sparse_allreduce": (c_int, [c_void_p, c_void_p, c_size_t, c_int64, c_size_t,
                                         P(OktResult), c_void_p]),
        "okt_sparse_allreduce_async": (c_int, [c_void_p, c_void_p, c_size_t, c_int64, c_size_t, c_void_p]),
        "okt_sgd_step_async": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_double, c_int64, c_size_t,
                                       c_void_p]),
        "okt_step_wait": (c_int, [c_void_p, P(OktResult)]),
        "okt_device_barrier": (c_int, [c_void_p, c_void_p]),
        "okt_residual_reset": (c_int, [c_void_p, c_size_t, c_void_p, c_void_p]),
        "okt_residual": (c_int, [c_void_p, P(c_void_p), P(c_size_t)]),
        "okt_sgd_step": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_double, c_int64,
                                 c_size_t, P(OktResult), c_void_p]),
        "okt_sparse_allreduce_host": (c_int, [c_void_p, c_void_p, c_size_t, c_int64, c_size_t,
                                              c_void_p, c_void_p, c_void_p, c_size_t,
                                              P(OktResult), c_void_p]),
        "okt_sgd_step_host": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_double, c_int64,
                                      c_size_t, c_void_p, c_void_p, c_size_t, P(OktResult),
                                      c_void_p]),
        "okt_memcpy_h2d": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
        "okt_memcpy_d2h": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
        "okt_th_re_evaluate_dense": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t,
                                             P(c_double), c_void_p]),
        "okt_th_re_evaluate_sparse": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t,
                                              P(c_double), c_void_p]),
        "okt_topka_allreduce": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]),
        "okt_dense_allreduce": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
        "okt_gtopk_allreduce": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]),
        "okt_topkdsa_allreduce": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]),
        "okt_gaussiank_threshold": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t, c_int, c_void_p, c_void_p]),
        "okt_gaussiank_allreduce": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t, c_int, c_void_p, c_void_p]),
        "okt_select_by_threshold": (c_int, [c_void_p, c_void_p, c_size_t, c_double,
                                            P(OktSparse), c_void_p]),
        "okt_space_repartition": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t,
                                          P(c_uint64), c_void_p]),
        "okt_split_and_reduce": (c_int, [c_void_p, c_void_p, c_size_t, c_double, P(c_uint64),
                                         c_uint32, P(OktSparse), P(OktSparse), c_void_p]),
        "okt_balance_and_allgatherv": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_size_t,
                                               c_double, P(OktSparse), c_void_p]),
        "okt_set_profiling": (c_int, [c_void_p, c_int]),
        "okt_phase_times": (c_int, [c_void_p, P(c_double), P(c_uint64)]),
        "okt_phase_bytes": (c_int, [c_void_p, P(c_double)]),
        "okt_reset_phase_times": (c_int, [c_void_p]),
        "okt_kernel_launches": (c_int, [c_void_p, P(c_uint64)]),
        "okt_wire_encode": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
        "okt_wire_decode": (c_int, [c_void_p, c_size_t, c_size_t, c_void_p, c_void_p, c_size_t, P(c_size_t),
                                    c_void_p]),
        "okt_debug_p2p_trace": (c_int, [c_void_p, P(c_uint64), c_size_t]),
        "okt_gen_random_dense": (c_int, [c_void_p, c_size_t, c_uint64, c_void_p]),
        "okt_gen_drift": (c_int, [c_void_p, c_size_t, c_int64, c_uint64, c_uint64, c_int,
                                  c_void_p]),
        "okt_plan_cuts": (c_int, [P(c_uint64), c_int, c_uint64, P(c_uint64)]),
        "okt_plan_balance": (c_int, [c_int, c_int, P(c_uint64), P(c_int), P(OktPiece), P(c_int),
                                     P(OktPiece), P(c_int), P(OktPiece), P(c_uint64), P(c_uint64)]),
        "okt_plan_ledger": (c_int, [c_int, c_int, c_int, P(c_uint64), c_uint64, c_uint32,
                                    P(OktCounters)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


__all__ = ["lib", "LIB_PATH", "EXPORTS", "OktState", "OktCounters", "OktSparse", "OktPiece",
           "OktResult", "OKT_MAX_WORLD", "OKT_T_COUNT", "TIMER_NAMES", "c_float"]
