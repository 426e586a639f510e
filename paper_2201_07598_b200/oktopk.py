"""Host-side mirror of the reference's Ok-Topk interface over the C-ABI.

Names, argument meaning and error behaviour follow the reference
(``proj/core/include/oklab/{oktopk,sparse,transport,trainer,errors}.hpp``) so
parity tests read like ``proj/tests/test_oktopk.cpp``:

    w = World(4)
    got = run_ranks(w, lambda ctx: ok_sparse_allreduce(ctx, OkState(), g[ctx.rank], 1, k))
    w.ledger.at(0, Phase.split).msgs_sent

Every computation runs in ``libokt.so`` (hand-written sm_100a kernels); this
module only moves arguments across the boundary.  Dense inputs may be numpy
arrays (copied to the rank's GPU as fp32) or CUDA float32 torch tensors.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import OktCounters, OktResult, OktSparse, OktState


# ---- errors (proj/core/include/oklab/errors.hpp) --------------------------------
class OkError(RuntimeError):
    pass


class TransportError(OkError):
    pass


class ProtocolError(OkError):
    pass


class DecodeError(OkError):
    pass


class NumericError(OkError):
    pass


class ConfigError(OkError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class CudaError(OkError):
    pass


_ERRORS = {1: InvalidArgument, 2: NumericError, 3: ProtocolError, 4: TransportError,
           5: ConfigError, 6: CudaError, 7: CudaError, 8: OkError, 9: DecodeError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.lib().okt_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, OkError)(msg)


# ---- types ---------------------------------------------------------------------
class Phase(IntEnum):
    """oklab::Phase (transport.hpp:15-22)."""
    split = 0
    balance = 1
    allgatherv = 2
    consensus = 3
    dense = 4
    gather = 5


@dataclass
class SparseGrad:
    """oklab::SparseGrad (sparse.hpp:34-49): strictly increasing u32 indices."""
    n: int = 0
    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    def nnz(self) -> int:
        return int(self.indices.size)

    def empty(self) -> bool:
        return self.indices.size == 0

    def valid(self) -> bool:
        if self.indices.size != self.values.size:
            return False
        if self.indices.size and int(self.indices.max()) >= self.n:
            return False
        return bool(np.all(np.diff(self.indices.astype(np.int64)) > 0))

    def as_map(self) -> dict:
        return {int(i): float(v) for i, v in zip(self.indices, self.values)}

    def __eq__(self, other) -> bool:  # same_sparse (test_util.hpp:155-157)
        return (isinstance(other, SparseGrad) and self.n == other.n
                and np.array_equal(self.indices, other.indices)
                and np.array_equal(self.values, other.values))


@dataclass
class ThresholdState:
    """oklab::ThresholdState (sparse.hpp:56-63)."""
    local_th: float = 0.0
    global_th: float = 0.0
    tau: int = 64
    tau_prime: int = 32
    last_local_eval: int = -1
    last_global_eval: int = -1


@dataclass
class RegionBoundaries:
    """oklab::RegionBoundaries (oktopk.hpp:16-22)."""
    cuts: List[int] = field(default_factory=list)

    def regions(self) -> int:
        return len(self.cuts) - 1


@dataclass
class OkState:
    """oklab::OkState (oktopk.hpp:30-35)."""
    th: ThresholdState = field(default_factory=ThresholdState)
    bounds: RegionBoundaries = field(default_factory=RegionBoundaries)
    t: int = 0
    bucket_size: int = 4

    def _to_c(self) -> OktState:
        s = OktState()
        s.local_th, s.global_th = self.th.local_th, self.th.global_th
        s.tau, s.tau_prime = self.th.tau, self.th.tau_prime
        s.last_local_eval, s.last_global_eval = self.th.last_local_eval, self.th.last_global_eval
        s.regions = len(self.bounds.cuts) - 1 if self.bounds.cuts else -1
        for i, c in enumerate(self.bounds.cuts[: _lib.OKT_MAX_WORLD + 1]):
            s.cuts[i] = c
        s.bucket_size = self.bucket_size
        s.t = self.t
        return s

    def _from_c(self, s: OktState) -> None:
        self.th.local_th, self.th.global_th = s.local_th, s.global_th
        self.th.tau, self.th.tau_prime = s.tau, s.tau_prime
        self.th.last_local_eval, self.th.last_global_eval = s.last_local_eval, s.last_global_eval
        self.bounds.cuts = [int(s.cuts[i]) for i in range(s.regions + 1)] if s.regions >= 0 else []
        self.bucket_size = s.bucket_size
        self.t = s.t


@dataclass
class OkAllreduceResult:
    """oklab::OkAllreduceResult (oktopk.hpp:95-99)."""
    u: SparseGrad
    indexes: np.ndarray
    local_selected: int


@dataclass
class SplitReduceResult:
    """oklab::SplitReduceResult (oktopk.hpp:61-64)."""
    region_reduced: SparseGrad
    local_topk_indexes: np.ndarray


# ---- worlds, contexts, ledgers ----------------------------------------------------
class WorkerCtx:
    """oklab::WorkerCtx (transport.hpp:111-122): one rank's comm handle."""

    def __init__(self, comm: int, rank: int, world: int, device: int):
        self.comm = ctypes.c_void_p(comm)
        self.rank = rank
        self.world = world
        self.device = device
        self._bound_residual = None


class TrafficLedger:
    """Read-only view of the per-rank ledgers (transport.hpp:52-83)."""

    def __init__(self, ctxs: Sequence[WorkerCtx]):
        self._ctxs = list(ctxs)

    def at(self, rank: int, phase: Phase) -> OktCounters:
        c = OktCounters()
        _check(_lib.lib().okt_ledger(self._ctxs[rank].comm, int(phase), ctypes.byref(c)))
        return c

    def words_recv(self, rank: int, phases: Sequence[Phase]) -> int:
        return sum(self.at(rank, p).words_recv for p in phases)

    def words_sent(self, rank: int, phases: Sequence[Phase]) -> int:
        return sum(self.at(rank, p).words_sent for p in phases)

    def total_sent(self, phase: Phase) -> int:
        return sum(self.at(r, phase).words_sent for r in range(len(self._ctxs)))

    def total_recv(self, phase: Phase) -> int:
        return sum(self.at(r, phase).words_recv for r in range(len(self._ctxs)))

    def reset(self) -> None:
        for c in self._ctxs:
            _check(_lib.lib().okt_ledger_reset(c.comm))


class World:
    """P ranks as host threads of this process (test_util.hpp:22-32).

    ``devices[r]`` is rank r's GPU; by default every rank shares the current
    device (exchanges are then HBM copies; on several GPUs they are NVLink
    peer copies).
    """

    def __init__(self, P: int, devices: Optional[Sequence[int]] = None):
        L = _lib.lib()
        self.P = P
        self._w = ctypes.c_void_p()
        if devices is None:
            import torch
            devices = [torch.cuda.current_device()] * P
        self.devices = list(devices)
        arr = (ctypes.c_int * P)(*self.devices)
        _check(L.okt_world_create_local(ctypes.byref(self._w), P, arr))
        self._ctxs = []
        for r in range(P):
            c = ctypes.c_void_p()
            _check(L.okt_comm_init_local(ctypes.byref(c), self._w, r))
            self._ctxs.append(WorkerCtx(c.value, r, P, self.devices[r]))
        self.ledger = TrafficLedger(self._ctxs)

    def ctx(self, rank: int) -> WorkerCtx:
        return self._ctxs[rank]

    def close(self) -> None:
        _lib.lib().okt_world_close(self._w)

    def destroy(self) -> None:
        L = _lib.lib()
        for c in self._ctxs:
            L.okt_comm_destroy(c.comm)
        self._ctxs = []
        if self._w:
            L.okt_world_destroy(self._w)
            self._w = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def run_ranks(world: World, body: Callable[[WorkerCtx], object]) -> list:
    """test_util.hpp:38-76: one thread per rank; on failure the world is closed
    and the first non-TransportError (the root cause) is re-raised."""
    out = [None] * world.P
    errs: list = [None] * world.P

    def work(r: int) -> None:
        try:
            import torch
            torch.cuda.set_device(world.devices[r])
            out[r] = body(world.ctx(r))
        except BaseException as e:  # noqa: BLE001 - rethrown below
            errs[r] = e
            world.close()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world.P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = next((e for e in errs if e is not None), None)
    root = next((e for e in errs if e is not None and not isinstance(e, TransportError)), None)
    if root is not None:
        raise root
    if first is not None:
        raise first
    return out


# ---- data movement helpers ----------------------------------------------------------
def _device_f32(g, device: int):
    """numpy / list / torch tensor -> contiguous float32 CUDA tensor on `device`."""
    import torch
    if isinstance(g, torch.Tensor):
        t = g
        if t.dtype != torch.float32:
            t = t.float()
        if t.device.type != "cuda" or t.device.index != device:
            t = t.to(f"cuda:{device}")
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(g, dtype=np.float64).astype(np.float32))
    return torch.from_numpy(a).to(f"cuda:{device}")


def _d2h(ptr, count: int, dtype) -> np.ndarray:
    out = np.empty(count, dtype=dtype)
    if count:
        _check(_lib.lib().okt_memcpy_d2h(out.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ptr),
                                         out.nbytes, None))
    return out


def _sparse_from(s: OktSparse, n: Optional[int] = None) -> SparseGrad:
    return SparseGrad(int(s.n if n is None else n), _d2h(s.d_idx, int(s.nnz), np.uint32),
                      _d2h(s.d_val, int(s.nnz), np.float64))


_scratch_lock = threading.Lock()
_scratch: dict = {}


def _scratch_ctx() -> WorkerCtx:
    """A single-rank world on the current device for the ctx-free entry points
    (th_re_evaluate, select_by_threshold), one per host thread."""
    import torch
    key = (threading.get_ident(), torch.cuda.current_device())
    with _scratch_lock:
        w = _scratch.get(key)
        if w is None:
            w = World(1, [torch.cuda.current_device()])
            _scratch[key] = w
    return w.ctx(0)


# ---- the reference's entry points ---------------------------------------------------
def th_re_evaluate(g, k: int, ctx: Optional[WorkerCtx] = None) -> float:
    """oktopk.cpp:12-26.  Dense input (numpy / tensor) or a SparseGrad."""
    ctx = ctx or _scratch_ctx()
    th = ctypes.c_double()
    L = _lib.lib()
    if isinstance(g, SparseGrad):
        if k < 1 and g.nnz():
            raise InvalidArgument("th_re_evaluate: k must be >= 1")
        import torch
        v = torch.from_numpy(np.ascontiguousarray(g.values, dtype=np.float64)).to(f"cuda:{ctx.device}")
        _check(L.okt_th_re_evaluate_sparse(ctx.comm, ctypes.c_void_p(v.data_ptr()), g.nnz(), max(k, 0),
                                           ctypes.byref(th), None))
    else:
        d = _device_f32(g, ctx.device)
        _check(L.okt_th_re_evaluate_dense(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(k, 0),
                                          ctypes.byref(th), None))
    return th.value


def select_by_threshold(g, th: float, ctx: Optional[WorkerCtx] = None) -> SparseGrad:
    """sparse.cpp:94-106 (dense input)."""
    ctx = ctx or _scratch_ctx()
    d = _device_f32(g, ctx.device)
    s = OktSparse()
    _check(_lib.lib().okt_select_by_threshold(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(),
                                              float(th), ctypes.byref(s), None))
    return _sparse_from(s, d.numel())


def space_repartition(ctx: WorkerCtx, selected: SparseGrad) -> RegionBoundaries:
    """oktopk.cpp:28-61 on an already-selected coordinate set."""
    import torch
    idx = torch.from_numpy(np.ascontiguousarray(selected.indices.astype(np.int32))).to(f"cuda:{ctx.device}")
    cuts = (ctypes.c_uint64 * (ctx.world + 1))()
    _check(_lib.lib().okt_space_repartition(ctx.comm, ctypes.c_void_p(idx.data_ptr()), selected.nnz(),
                                            selected.n, cuts, None))
    return RegionBoundaries([int(c) for c in cuts])


def split_and_reduce(ctx: WorkerCtx, g, local_th: float, bounds: RegionBoundaries,
                     bucket_size: int) -> SplitReduceResult:
    """oktopk.cpp:95-163."""
    if bounds.regions() != ctx.world:
        raise InvalidArgument("split_and_reduce: boundaries do not match P")
    d = _device_f32(g, ctx.device)
    cuts = (ctypes.c_uint64 * (ctx.world + 1))(*bounds.cuts)
    region, local = OktSparse(), OktSparse()
    _check(_lib.lib().okt_split_and_reduce(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), float(local_th),
                                           cuts, bucket_size, ctypes.byref(region), ctypes.byref(local), None))
    return SplitReduceResult(_sparse_from(region), _d2h(local.d_idx, int(local.nnz), np.uint32))


def balance_and_allgatherv(ctx: WorkerCtx, region: SparseGrad, global_th: float) -> SparseGrad:
    """oktopk.cpp:165-244."""
    import torch
    dev = f"cuda:{ctx.device}"
    idx = torch.from_numpy(np.ascontiguousarray(region.indices.astype(np.int32))).to(dev)
    val = torch.from_numpy(np.ascontiguousarray(region.values, dtype=np.float64)).to(dev)
    u = OktSparse()
    _check(_lib.lib().okt_balance_and_allgatherv(ctx.comm, ctypes.c_void_p(idx.data_ptr()),
                                                 ctypes.c_void_p(val.data_ptr()), region.nnz(), region.n,
                                                 float(global_th), ctypes.byref(u), None))
    return _sparse_from(u, region.n)


def topka_allreduce(ctx: WorkerCtx, g, k: int) -> SparseGrad:
    """Table-1 baseline TopkA (collectives.cpp:152-159): exact local top-k,
    sparse_allgatherv, stride-doubling sparse_sum — all on the GPU."""
    d = _device_f32(g, ctx.device)
    s = OktSparse()
    _check(_lib.lib().okt_topka_allreduce(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(int(k), 0),
                                          ctypes.byref(s), None))
    return _sparse_from(s, d.numel())


def dense_allreduce(ctx: WorkerCtx, g) -> np.ndarray:
    """Dense fp64 recursive-halving allreduce (collectives.cpp:89-150) of the
    fp32 gradient; returns the summed vector (float64, host)."""
    d = _device_f32(g, ctx.device)
    p = ctypes.c_void_p()
    _check(_lib.lib().okt_dense_allreduce(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), ctypes.byref(p), None))
    return _d2h(p.value, d.numel(), np.float64)


def gtopk_allreduce(ctx: WorkerCtx, g, k: int) -> SparseGrad:
    """Table-1 baseline gTopk (collectives.cpp:300-325)."""
    d = _device_f32(g, ctx.device)
    s = OktSparse()
    _check(_lib.lib().okt_gtopk_allreduce(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(int(k), 0),
                                          ctypes.byref(s), None))
    return _sparse_from(s, d.numel())


def topkdsa_allreduce(ctx: WorkerCtx, g, k: int) -> SparseGrad:
    """Table-1 baseline TopkDSA (collectives.cpp:184-297): reduce-scatter with the
    COO -> dense-window switch, then allgatherv of the owned segments."""
    d = _device_f32(g, ctx.device)
    s = OktSparse()
    _check(_lib.lib().okt_topkdsa_allreduce(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(int(k), 0),
                                            ctypes.byref(s), None))
    return _sparse_from(s, d.numel())


def gaussiank_allreduce(ctx: WorkerCtx, g, k: int, scale_to_floor: bool = True) -> SparseGrad:
    """Table-1 baseline Gaussiank (collectives.cpp:342-352; GaussiankOptions)."""
    d = _device_f32(g, ctx.device)
    s = OktSparse()
    _check(_lib.lib().okt_gaussiank_allreduce(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(int(k), 0),
                                              int(bool(scale_to_floor)), ctypes.byref(s), None))
    return _sparse_from(s, d.numel())


def gaussian_threshold(g, k: int, ctx: Optional[WorkerCtx] = None) -> float:
    """sparse.cpp:167-188 (fp64 moments by a tree reduction: within a few ulp)."""
    ctx = ctx or _scratch_ctx()
    d = _device_f32(g, ctx.device)
    th = ctypes.c_double()
    _check(_lib.lib().okt_gaussiank_threshold(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(int(k), 0), 0,
                                              ctypes.byref(th), None))
    return th.value


def gaussiank_scaled_threshold(g, k: int, ctx: Optional[WorkerCtx] = None) -> float:
    """collectives.cpp:327-340."""
    ctx = ctx or _scratch_ctx()
    d = _device_f32(g, ctx.device)
    th = ctypes.c_double()
    _check(_lib.lib().okt_gaussiank_threshold(ctx.comm, ctypes.c_void_p(d.data_ptr()), d.numel(), max(int(k), 0), 1,
                                              ctypes.byref(th), None))
    return th.value


def wire_encode(s: SparseGrad, device: int = 0) -> bytes:
    """oklab::wire_encode (sparse.hpp:126, sparse.cpp:275-285) on the device:
    [nnz u32][indices u32 x nnz][values f32 x nnz], little endian."""
    import torch
    nnz = s.nnz()
    idx = torch.from_numpy(np.ascontiguousarray(s.indices, dtype=np.uint32).view(np.int32)).to(f"cuda:{device}")
    val = torch.from_numpy(np.ascontiguousarray(s.values, dtype=np.float64)).to(f"cuda:{device}")
    out = torch.empty(1 + 2 * nnz, dtype=torch.int32, device=f"cuda:{device}")
    with torch.cuda.device(device):
        _check(_lib.lib().okt_wire_encode(ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(val.data_ptr()), nnz,
                                          ctypes.c_void_p(out.data_ptr()), None))
    return out.cpu().numpy().view(np.uint8).tobytes()


def wire_decode(b: bytes, n: int, device: int = 0) -> SparseGrad:
    """oklab::wire_decode (sparse.hpp:131, sparse.cpp:287-310) on the device;
    a malformed image raises DecodeError."""
    import torch
    raw = np.frombuffer(bytes(b) + b"\0" * (-len(b) % 4), np.uint8).view(np.int32)
    img = torch.from_numpy(raw.copy()).to(f"cuda:{device}") if raw.size else torch.zeros(1, dtype=torch.int32,
                                                                                            device=f"cuda:{device}")
    cap = max(1, (len(b) - 4) // 8) if len(b) >= 4 else 1
    idx = torch.empty(cap, dtype=torch.int32, device=f"cuda:{device}")
    val = torch.empty(cap, dtype=torch.float64, device=f"cuda:{device}")
    nnz = ctypes.c_size_t(0)
    with torch.cuda.device(device):
        _check(_lib.lib().okt_wire_decode(ctypes.c_void_p(img.data_ptr()), len(b), n, ctypes.c_void_p(idx.data_ptr()),
                                          ctypes.c_void_p(val.data_ptr()), cap, ctypes.byref(nnz), None))
    m = nnz.value
    return SparseGrad(n, idx[:m].cpu().numpy().view(np.uint32).copy(), val[:m].cpu().numpy().copy())


def ok_sparse_allreduce(ctx: WorkerCtx, state: OkState, g, t: int, k: int) -> OkAllreduceResult:
    """oktopk.cpp:246-307.  `state` is read before and written back after the
    call, as the reference mutates its OkState in place."""
    L = _lib.lib()
    d = _device_f32(g, ctx.device) if (not hasattr(g, "__len__") or len(g)) else None
    cs = state._to_c()
    _check(L.okt_set_state(ctx.comm, ctypes.byref(cs)))
    res = OktResult()
    n = 0 if d is None else d.numel()
    ptr = ctypes.c_void_p(d.data_ptr()) if d is not None else ctypes.c_void_p()
    _check(L.okt_sparse_allreduce(ctx.comm, ptr, n, int(t), max(int(k), 0), ctypes.byref(res), None))
    _check(L.okt_get_state(ctx.comm, ctypes.byref(cs)))
    state._from_c(cs)
    return OkAllreduceResult(_sparse_from(res.u, n), _d2h(res.d_indexes, int(res.n_indexes), np.uint32),
                             int(res.local_selected))


# ---- error-feedback SGD step (trainer.hpp:146-152) ------------------------------------
@dataclass
class LrSchedule:
    alpha: float = 0.05
    inv_sqrt_decay: bool = False

    def at(self, t: int) -> float:
        return self.alpha / np.sqrt(t) if self.inv_sqrt_decay else self.alpha


class ModelState:
    """oklab::ModelState: w lives on the rank's GPU (fp32)."""

    def __init__(self, w, device: int, lr: Optional[LrSchedule] = None):
        self.w = _device_f32(w, device).clone()
        self.t = 0
        self.lr = lr or LrSchedule()


class Residual:
    """oklab::Residual; the live buffer is owned by the comm (okt_residual)."""

    def __init__(self, n: int, eps=None):
        self.n = n
        self.init = None if eps is None else np.asarray(eps, dtype=np.float64)

    def eps(self, ctx: WorkerCtx) -> np.ndarray:
        p, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(_lib.lib().okt_residual(ctx.comm, ctypes.byref(p), ctypes.byref(n)))
        return _d2h(p.value, n.value, np.float32).astype(np.float64)


def oktopk_sgd_step(ctx: WorkerCtx, model: ModelState, residual: Residual, grad, k: int,
                    ok: OkState) -> OkAllreduceResult:
    """trainer.cpp:466-488 with the problem's gradient passed in: acc = eps +
    alpha*grad; ok_sparse_allreduce(acc); eps = acc zeroed at indexes;
    w -= u / P."""
    L = _lib.lib()
    if ctx._bound_residual is not residual:
        init = None
        if residual.init is not None:
            init = _device_f32(residual.init, ctx.device)
        _check(L.okt_residual_reset(ctx.comm, residual.n,
                                    ctypes.c_void_p(init.data_ptr()) if init is not None else ctypes.c_void_p(),
                                    None))
        ctx._bound_residual = residual
    d = _device_f32(grad, ctx.device)
    t = model.t + 1
    cs = ok._to_c()
    _check(L.okt_set_state(ctx.comm, ctypes.byref(cs)))
    res = OktResult()
    _check(L.okt_sgd_step(ctx.comm, ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(model.w.data_ptr()),
                          d.numel(), float(model.lr.at(t)), t, int(k), ctypes.byref(res), None))
    _check(L.okt_get_state(ctx.comm, ctypes.byref(cs)))
    ok._from_c(cs)
    model.t = t
    return OkAllreduceResult(_sparse_from(res.u, d.numel()), _d2h(res.d_indexes, int(res.n_indexes), np.uint32),
                             int(res.local_selected))


# ---- instrumentation -------------------------------------------------------------------
def kernel_launches(ctx: WorkerCtx) -> int:
    v = ctypes.c_uint64()
    _check(_lib.lib().okt_kernel_launches(ctx.comm, ctypes.byref(v)))
    return v.value


def set_profiling(ctx: WorkerCtx, on: bool) -> None:
    _check(_lib.lib().okt_set_profiling(ctx.comm, 1 if on else 0))


def phase_times(ctx: WorkerCtx) -> dict:
    ms = (ctypes.c_double * _lib.OKT_T_COUNT)()
    calls = (ctypes.c_uint64 * _lib.OKT_T_COUNT)()
    _check(_lib.lib().okt_phase_times(ctx.comm, ms, calls))
    return {name: (ms[i], int(calls[i])) for i, name in enumerate(_lib.TIMER_NAMES)}
