#!/usr/bin/env python3
"""Ok-Topk sparse-allreduce benchmark (BASELINE.json metric) on B200.

One step = one Ok-Topk error-feedback SGD iteration through the C-ABI
(okt_sgd_step_async + okt_step_wait: acc = eps + alpha*g fused with threshold
selection, split and reduce, global threshold, balance + allgatherv, residual
/ model scatter; the per-step CUDA events bracket the enqueue, the wait comes
after the end event) on a
VGG-16-sized fp32 gradient (n = 14,728,266, density 1%, BASELINE.json
configs[1]), tau = 64, tau' = 32, bucket 4 — refresh iterations included in
the timed window in their natural 1-in-32 proportion.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl okt|reference]

N > 1 runs under torchrun, one process per GPU; the data path is the library's
own NCCL communicator (NVLink), torch.distributed (gloo) is only plumbing for
the id broadcast, barriers and the max-over-ranks reduction.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

VGG_N = 14_728_266


def k_for(n: int, density: float) -> int:
    """ExperimentConfig::k (harness.cpp:82-86)."""
    raw = density * float(n) * (1.0 - 1e-12)
    return max(1, min(n, int(math.ceil(raw))))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="okt", choices=["okt", "reference"])
    # (--elements: under torchrun an abbreviation-like "--n" is taken by the launcher)
    ap.add_argument("--n", "--elements", dest="n", type=int, default=VGG_N)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--tau", type=int, default=64)
    ap.add_argument("--tau-prime", type=int, default=32)
    ap.add_argument("--bucket", type=int, default=4)
    ap.add_argument("--ring", type=int, default=8, help="distinct gradient snapshots cycled per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=32)
    ap.add_argument("--trace", default="", help="directory: dump a CUPTI timeline (torch.profiler) of 16 steps")
    ap.add_argument("--no-l2-flush", action="store_true", help="diagnostics only: skip the L2 flush between steps")
    ap.add_argument("--p2p-trace", default="",
                    help="directory: dump per-CTA globaltimer stamps of the last device-driven (P2P) step")
    a = ap.parse_args()
    if a.p2p_trace:
        os.environ["OKT_P2P_TRACE"] = "1"  # read when the comm maps its peers
    return a


def dump_p2p_trace(L, comm, rank, outdir):
    """Per-kernel spans of the last P2P step from the CTAs' %globaltimer stamps
    (okt_debug_p2p_trace), relative to the first K1 CTA start."""
    import numpy as np
    kinds, ctas = 7, 2048
    buf = (ctypes.c_uint64 * (kinds * ctas * 4))()
    if L.okt_debug_p2p_trace(comm, buf, kinds * ctas * 4):
        return
    a = np.frombuffer(buf, dtype=np.uint64).reshape(kinds, ctas, 4).astype(np.int64)
    used = a[:, :, 0] > 0
    t0 = a[0, :, 0][used[0]].min() if used[0].any() else 0
    out = {}
    for k, nm in enumerate(["k1", "merge", "compact", "pull0", "pull1", "publish_l", "publish_sur"]):
        u = used[k]
        if not u.any():
            continue
        st, wt, en = a[k, u, 0] - t0, a[k, u, 1] - t0, a[k, u, 2] - t0
        wt = wt[a[k, u, 1] > 0]
        en = en[a[k, u, 2] > 0]
        out[nm] = {"ctas": int(u.sum()), "start_min_us": float(st.min()) / 1e3, "start_max_us": float(st.max()) / 1e3,
                   "waited_min_us": float(wt.min()) / 1e3 if wt.size else None,
                   "waited_max_us": float(wt.max()) / 1e3 if wt.size else None,
                   "end_med_us": float(np.median(en)) / 1e3 if en.size else None,
                   "end_max_us": float(en.max()) / 1e3 if en.size else None}
    os.makedirs(outdir, exist_ok=True)
    np.save(os.path.join(outdir, f"p2p_trace_rank{rank}.npy"), a)
    with open(os.path.join(outdir, f"p2p_trace_rank{rank}.json"), "w") as f:
        json.dump(out, f, indent=1)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, P):
    return {"workload": "vgg16-sized fp32 gradient, Ok-Topk EF-SGD step" if args.n == VGG_N
            else f"n={args.n} fp32 gradient, Ok-Topk EF-SGD step",
            "n": args.n, "density": args.density, "k": k_for(args.n, args.density), "P": P,
            "tau": args.tau, "tau_prime": args.tau_prime, "bucket": args.bucket,
            "inputs": f"drifting_gradient_process(t, seed=1, rank_key=r+1), ring of {args.ring} snapshots",
            "parallelism": f"dp{P} (one process per GPU, NCCL/NVLink)" if P > 1 else "single GPU",
            "rank_alignment": "device barrier (okt_device_barrier, NVLink flags) before each timed step, "
                              "outside the events" if P > 1 else None,
            "l2": "not flushed (diagnostic run)" if args.no_l2_flush else
            "flushed before every timed step, outside the events: 256 MiB write, then a 256 MiB read sweep "
            "(clean L2: no write-back of the flush buffer inside the step)"}


# ---- clocks ----------------------------------------------------------------------
class Clocks:
    """Samples SM clock and throttle reasons through NVML on a background
    thread while the measured region runs (nvidia-smi's 200 ms polling is too
    coarse for a region this short)."""

    HW = 0x0000000000000008          # hw_slowdown
    HW_THERMAL = 0x0000000000000040
    SW_THERMAL = 0x0000000000000020
    SW_POWER = 0x0000000000000004

    def __init__(self, gpu: int):
        import threading
        self.gpu = gpu
        self.samples, self.reasons, self.mx = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, nm in ((self.HW, "hw_slowdown"), (self.HW_THERMAL, "hw_thermal_slowdown"),
                                (self.SW_THERMAL, "sw_thermal_slowdown"), (self.SW_POWER, "sw_power_cap")):
                    if r & bit:
                        self.reasons.add(nm)
                self._stop.wait(0.002)
        except Exception as e:  # pragma: no cover - reported in the JSON
            self.reasons.add(f"nvml unavailable: {e}")

    def start(self):
        import threading
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=5)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---- reference arm -------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0  # rank 0 alone times the reference's CPU path with P = N threads
    P = max(args.gpus, world)
    k = k_for(args.n, args.density)
    line = {"metric": "Ok-Topk sparse allreduce ms/iter", "unit": "ms/iter", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(args, P)}
    try:
        from oracle import Reference
        ref = Reference()
    except Exception as e:  # the reference .so is built in the dev container and travels
        line["unavailable"] = f"oracle/_ref/libokref.so not loadable: {e}"
        print(json.dumps(line))
        return 0
    steps = args.steps
    t0 = time.time()
    ms = ref.bench_sgd(P, args.n, k, args.warmup, steps, args.tau, args.tau_prime, args.bucket, 1.0, 1, True)
    wall = time.time() - t0
    v = float(ms.mean())
    line.update({"value": v, "ms_per_step": v,
                 "cpu_baseline": {"value": v, "unit": "ms/iter", "cores": P, "kind": "reference",
                                  "sample": f"{steps} timed iterations after {args.warmup} warm-up, "
                                            f"P={P} rank threads (InprocTransport), one core each",
                                  "cpu": _cpu_model(), "nproc": os.cpu_count(), "wall_s": round(wall, 1)},
                 "e2e": {"value": v, "unit": "ms/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                 "ms_min": float(ms.min()), "ms_max": float(ms.max())})
    print(json.dumps(line))
    return 0


def _cpu_model() -> str:
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class L2Flush:
    """Evicts L2 between timed steps: a write of a buffer larger than L2, then
    a read sweep of another one, so the step starts with L2 holding neither its
    inputs nor dirty lines whose write-back it would pay for."""

    def __init__(self, nbytes: int):
        import torch
        self.w = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.r = torch.zeros(nbytes // 8, dtype=torch.int64, device="cuda")

    def fill_(self, v: int):
        self.w.fill_(v)
        self.r.sum()


def trace_steps(args, rank, stream, step, t0, step_async=None, wait=None, flush=None):
    """CUPTI timeline of 16 steps: per-kernel device time and the idle gaps
    between them (host launch / sync latency), written next to a chrome trace."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    os.makedirs(args.trace, exist_ok=True)
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for i in range(16):
            if step_async is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(i & 0xff)
                step_async(t0 + 1 + i)
                wait()
            else:
                step(t0 + 1 + i)
        torch.cuda.synchronize()
    prof.export_chrome_trace(os.path.join(args.trace, f"trace_rank{rank}.json"))
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    per = {}
    for e in ev:
        d = per.setdefault(e.name[:60], [0, 0.0])
        d[0] += 1
        d[1] += e.time_range.elapsed_us()
    span = (ev[-1].time_range.end - ev[0].time_range.start) if ev else 0
    busy = sum(e.time_range.elapsed_us() for e in ev)
    with open(os.path.join(args.trace, f"summary_rank{rank}.txt"), "w") as f:
        f.write(f"16 steps: device span {span:.1f} us, kernel+copy busy {busy:.1f} us\n")
        for k, (c, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{c:5d} {us / 16:9.2f} us/step  {k}\n")


# ---- our arm ------------------------------------------------------------------------
def bind_to_gpu_cpus(gpu: int) -> str:
    """Pin this rank to the CPU cores local to its GPU (NVML's affinity mask),
    so its pinned host buffers are first-touched on the GPU's NUMA node — the
    usual one-process-per-GPU deployment.  Returns a description for the JSON."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return f"bound to the GPU-local cores ({len(cpus)} of {os.cpu_count()})"
    except Exception as e:  # no NVML affinity: leave the scheduler's placement
        return f"unbound ({type(e).__name__})"
    return "unbound"


def run_okt(args):
    import torch
    import torch.distributed as dist

    from paper_2201_07598_b200 import lib
    from paper_2201_07598_b200._lib import OktResult

    rank, world, local = dist_env()
    P = world
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    affinity = bind_to_gpu_cpus(local)
    L = lib()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    # ---- comm: NCCL over NVLink for P > 1, a local single-rank world for P = 1
    comm = ctypes.c_void_p()
    if P > 1:
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            assert L.okt_nccl_unique_id(uid, 128) == 0
        obj = [bytes(uid)] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        ctypes.memmove(uid, obj[0], 128)
        rc = L.okt_comm_init_nccl(ctypes.byref(comm), rank, P, local, uid, 128)
    else:
        w = ctypes.c_void_p()
        dev = (ctypes.c_int * 1)(local)
        rc = L.okt_world_create_local(ctypes.byref(w), 1, dev)
        rc = rc or L.okt_comm_init_local(ctypes.byref(comm), w, 0)
    if rc:
        raise SystemExit(f"comm init failed: {L.okt_last_error().decode()}")
    n, k = args.n, k_for(args.n, args.density)
    assert L.okt_set_params(comm, args.tau, args.tau_prime, args.bucket) == 0
    assert L.okt_comm_reserve(comm, n) == 0
    stream = torch.cuda.Stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    # ---- inputs: a ring of drift snapshots per rank, generated on the device
    ring = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(args.ring)]
    for i, buf in enumerate(ring):
        assert L.okt_gen_drift(ctypes.c_void_p(buf.data_ptr()), n, i + 1, 1, rank + 1, 0, sp) == 0
    wmodel = torch.zeros(n, dtype=torch.float32, device="cuda")
    assert L.okt_residual_reset(comm, n, None, sp) == 0
    flush = L2Flush(1 << 20 if args.no_l2_flush else 256 << 20)
    res = OktResult()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def step(t):
        g = ring[(t - 1) % args.ring]
        rc = L.okt_sgd_step(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(wmodel.data_ptr()), n, 1.0, t, k,
                            ctypes.byref(res), sp)
        if rc:
            raise SystemExit(f"okt_sgd_step failed: {L.okt_last_error().decode()}")

    def step_async(t):
        g = ring[(t - 1) % args.ring]
        rc = L.okt_sgd_step_async(comm, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(wmodel.data_ptr()), n,
                                  1.0, t, k, sp)
        if rc:
            raise SystemExit(f"okt_sgd_step_async failed: {L.okt_last_error().decode()}")

    def wait():
        rc = L.okt_step_wait(comm, ctypes.byref(res))
        if rc:
            raise SystemExit(f"okt_step_wait failed: {L.okt_last_error().decode()}")

    # ---- warm-up
    t = 0
    for _ in range(args.warmup):
        t += 1
        step(t)
    barrier()
    if args.trace:
        trace_steps(args, rank, stream, step, t, step_async, wait, flush)
        t += 16
    # ---- timed device-resident run (no profiling events inside the steps)
    launches0 = ctypes.c_uint64()
    L.okt_kernel_launches(comm, ctypes.byref(launches0))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = Clocks(local)
    clocks.start()
    barrier()
    U_sum, m_sum = 0, 0
    t_first = t + 1
    wall0 = time.perf_counter()
    for i in range(args.steps):
        t += 1
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xff)  # evict L2 between timed steps (outside the events)
        if world > 1:
            # align the ranks' GPUs (device barrier over NVLink, outside the
            # events): the step is timed without the host loop's launch skew
            L.okt_device_barrier(comm, ctypes.c_void_p(stream.cuda_stream))
        with torch.cuda.stream(stream):
            ev[i][0].record(stream)
        step_async(t)
        with torch.cuda.stream(stream):
            ev[i][1].record(stream)
        wait()
        U_sum += res.u.nnz
        m_sum += res.local_selected
    barrier()
    wall = time.perf_counter() - wall0
    launches1 = ctypes.c_uint64()
    L.okt_kernel_launches(comm, ctypes.byref(launches1))
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if args.p2p_trace:
        dump_p2p_trace(L, comm, rank, args.p2p_trace)
    # ---- the same timed loop again with the library's per-phase CUDA events
    # on its stream (phase breakdown + the K1 roofline)
    from paper_2201_07598_b200._lib import OKT_T_COUNT, TIMER_NAMES
    L.okt_set_profiling(comm, 1)
    L.okt_reset_phase_times(comm)
    barrier()
    for i in range(args.steps):
        t += 1
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xff)
        step_async(t)
        wait()
    barrier()
    ms_t = (ctypes.c_double * OKT_T_COUNT)()
    calls = (ctypes.c_uint64 * OKT_T_COUNT)()
    byts = (ctypes.c_double * OKT_T_COUNT)()
    L.okt_phase_times(comm, ms_t, calls)
    L.okt_phase_bytes(comm, byts)
    L.okt_set_profiling(comm, 0)
    phases = {nm: round(ms_t[i] / max(1, args.steps), 4) for i, nm in enumerate(TIMER_NAMES)}
    k1_ms, k1_bytes, k1_calls = ms_t[TIMER_NAMES.index("k1")], byts[TIMER_NAMES.index("k1")], calls[TIMER_NAMES.index("k1")]
    # ---- end-to-end through the synchronous host-buffer C-ABI call (the
    # reference's calling convention: H2D gradient, step, D2H u, all timed)
    hbuf = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(min(args.ring, 4))]
    for i, hb in enumerate(hbuf):
        hb.copy_(ring[i].cpu())
    cap = n
    h_uidx = torch.empty(cap, dtype=torch.int32).pin_memory()
    h_uval = torch.empty(cap, dtype=torch.float64).pin_memory()
    e2e_steps = max(4, min(args.steps, 32))
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
    # untimed warm-up of the host-buffer path (its device staging is allocated on first use)
    for i in range(2):
        t += 1
        if L.okt_sgd_step_host(comm, ctypes.c_void_p(hbuf[i % len(hbuf)].data_ptr()), ctypes.c_void_p(wmodel.data_ptr()),
                               n, 1.0, t, k, ctypes.c_void_p(h_uidx.data_ptr()), ctypes.c_void_p(h_uval.data_ptr()),
                               cap, ctypes.byref(res), sp):
            raise SystemExit(f"okt_sgd_step_host failed: {L.okt_last_error().decode()}")
    barrier()
    d2h = 0
    for i in range(e2e_steps):
        t += 1
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xff)
        if world > 1:
            barrier()  # hosts and GPUs aligned before each timed call (outside the events)
            L.okt_device_barrier(comm, ctypes.c_void_p(stream.cuda_stream))
        with torch.cuda.stream(stream):
            e2e_ev[i][0].record(stream)
        rc = L.okt_sgd_step_host(comm, ctypes.c_void_p(hbuf[i % len(hbuf)].data_ptr()),
                                 ctypes.c_void_p(wmodel.data_ptr()), n, 1.0, t, k,
                                 ctypes.c_void_p(h_uidx.data_ptr()), ctypes.c_void_p(h_uval.data_ptr()), cap,
                                 ctypes.byref(res), sp)
        if rc:
            raise SystemExit(f"okt_sgd_step_host failed: {L.okt_last_error().decode()}")
        with torch.cuda.stream(stream):
            e2e_ev[i][1].record(stream)
        d2h += 12 * res.u.nnz
    barrier()
    clk = clocks.stop()
    e2e_list = [a.elapsed_time(b) for a, b in e2e_ev]
    e2e_ms = sum(e2e_list) / e2e_steps
    if os.environ.get("OKT_BENCH_DEBUG"):
        print(f"[rank {rank}] e2e t0={t - e2e_steps + 1} ms={[round(x, 3) for x in e2e_list]}", file=sys.stderr)
    # ---- reference point: a dense NCCL allreduce of the same gradient
    dense_ms = None
    if world > 1:
        pg = dist.new_group(backend="nccl")
        dense = torch.empty(n, dtype=torch.float32, device="cuda")
        dense.copy_(ring[0])
        dev_ = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(16)]
        for i in range(4 + len(dev_)):
            flush.fill_(i & 0xff)
            barrier()
            if i >= 4:
                dev_[i - 4][0].record()
            dist.all_reduce(dense, group=pg)
            if i >= 4:
                dev_[i - 4][1].record()
        torch.cuda.synchronize()
        dense_ms = sum(a.elapsed_time(b) for a, b in dev_) / len(dev_)
    # ---- max over ranks
    mine = torch.tensor([total_ms, e2e_ms, wall, dense_ms or 0.0], dtype=torch.float64)
    per_step = torch.tensor(step_ms, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, wall, dense_ms = mine.tolist()
    # steady vs refresh iterations ((t - 1) % tau' == 0 re-evaluates the thresholds)
    refresh = [(t_first + i - 1) % args.tau_prime == 0 for i in range(args.steps)]
    st_ms = [v for v, r in zip(per_step.tolist(), refresh) if not r]
    rf_ms = [v for v, r in zip(per_step.tolist(), refresh) if r]
    ms_per_step = total_ms / args.steps
    achieved = k1_bytes / (k1_ms * 1e-3) / 1e9 if k1_ms > 0 else None
    peak = None
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        peak_src = "measured"
    except Exception:
        peak, peak_src = 6650.0, "fallback"
    line = None
    if rank == 0:
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))
            traffic = prof.get("bytes_per_launch")
        except Exception:
            pass
        line = {"metric": "Ok-Topk sparse allreduce ms/iter", "value": ms_per_step, "unit": "ms/iter",
                "n_gpus": P, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": workload(args, P),
                "e2e": {"value": e2e_ms, "unit": "ms/iter", "h2d_bytes_per_step": 4 * n,
                        "d2h_bytes_per_step": int(d2h / e2e_steps), "steps": e2e_steps,
                        "ms_min": min(e2e_list), "ms_median": statistics.median(e2e_list), "ms_max": max(e2e_list),
                        "path": "okt_sgd_step_host: gradient H2D from pinned host memory, step, u D2H", "cpu_affinity": affinity},
                "gpu_launches": int(launches1.value - launches0.value),
                "roofline": {"bound": "hbm", "kernel": "k1_kernel (fused residual accumulate + threshold select "
                                                         "+ chunk-local COO compaction; phase A of K1)",
                             "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                             "peak_source": peak_src,
                             "bytes_per_launch": k1_bytes / max(1, k1_calls),
                             "us_per_launch": 1e3 * k1_ms / max(1, k1_calls), "launches": int(k1_calls),
                             "bytes_formula": "12n + 8e per EF step (read g, eps; write eps; 8 B per staged "
                                              "entry e); refresh steps add a 4n + 8m select pass"},
                "phases_ms_per_step": phases,
                "steady_ms": statistics.mean(st_ms) if st_ms else None,
                "refresh_ms": statistics.mean(rf_ms) if rf_ms else None,
                "refresh_steps_timed": len(rf_ms),
                # dense-equivalent bandwidth, comparable to an allreduce's busBw
                "dense_equivalent_gbs": 2 * 4 * n * (P - 1) / P / (ms_per_step * 1e-3) / 1e9 if P > 1 else None,
                "avg_U": U_sum / args.steps, "avg_local_selected": m_sum / args.steps,
                "wall_ms_per_step": 1e3 * wall / args.steps,
                "dense_nccl_allreduce": None if world == 1 else {
                    "ms": dense_ms, "bytes": 4 * n,
                    "note": "reference point: torch.distributed NCCL all_reduce of the dense fp32 gradient, "
                            "device-timed, max over ranks (not the metric)"},
                "clocks": clk}
    # ---- CPU baseline (rank 0, N = 1 only): the reference itself, bounded sample
    if rank == 0 and P == 1 and not args.no_cpu_baseline:
        try:
            from oracle import Reference
            ref = Reference()
            t0 = time.time()
            ms = ref.bench_sgd(1, n, k, 1, args.cpu_iters, args.tau, args.tau_prime, args.bucket, 1.0, 1, True)
            line["cpu_baseline"] = {"value": float(ms.mean()), "unit": "ms/iter", "cores": 1, "kind": "reference",
                                    "sample": f"{args.cpu_iters} iterations t=2..{args.cpu_iters + 1} "
                                              f"(one tau' refresh) of the reference's EF-SGD step, same n/k/tau",
                                    "cpu": _cpu_model(), "wall_s": round(time.time() - t0, 1)}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    L.okt_comm_destroy(comm)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_okt(args)


if __name__ == "__main__":
    sys.exit(main())
