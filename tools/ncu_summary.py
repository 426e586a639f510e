#!/usr/bin/env python3
"""Summarise `ncu --page raw --csv` exports (one kernel launch each) into the
per-kernel evidence DESIGN.md §7 cites: duration, DRAM bytes read / written
and their rate against the measured HBM peak, algorithmic bytes (given) and
the achieved fraction, L1 sectors per request, occupancy, and the top warp
stall reasons.

    python tools/ncu_summary.py NAME=FILE_raw.csv[:ALGO_BYTES] ... > summary.json
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    names, units, vals = rows[0], rows[1], rows[2]
    return {n: (v, u) for n, u, v in zip(names, units, vals)}


def num(d, key, scale_units=True):
    if key not in d:
        return None
    v, u = d[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    if scale_units:
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u)
        if mult is not None:
            x *= mult
    return x


def main():
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    out = {"peak_hbm_gbs": peak, "kernels": {}}
    for arg in sys.argv[1:]:
        name, spec = arg.split("=", 1)
        path, _, algo = spec.partition(":")
        d = load(path)
        if d is None:
            out["kernels"][name] = {"missing": path}
            continue
        t = num(d, "gpu__time_duration.sum")
        rd = num(d, "dram__bytes_read.sum")
        wr = num(d, "dram__bytes_write.sum")
        e = {"kernel": d.get("Kernel Name", ("?",))[0][:120], "source": os.path.relpath(path, ROOT),
             "us": t * 1e6 if t else None, "dram_read_bytes": rd, "dram_write_bytes": wr}
        if t and rd is not None and wr is not None:
            e["dram_gbs"] = (rd + wr) / t / 1e9
            e["dram_frac_of_peak"] = e["dram_gbs"] / peak
        if algo and t:
            a = float(algo)
            e["algorithmic_bytes"] = a
            e["algorithmic_gbs"] = a / t / 1e9
            e["algorithmic_frac_of_peak"] = e["algorithmic_gbs"] / peak
        req = num(d, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", False)
        sec = num(d, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", False)
        if req and sec:
            e["ld_sectors_per_request"] = sec / req
        occ = num(d, "sm__warps_active.avg.pct_of_peak_sustained_active", False)
        if occ is not None:
            e["achieved_occupancy_pct"] = occ
        regs = num(d, "launch__registers_per_thread", False)
        if regs is not None:
            e["registers"] = regs
        stalls = {}
        for k, (v, u) in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        if stalls:
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
            e["top_stalls_per_issue"] = {k: round(v, 2) for k, v in top}
        out["kernels"][name] = e
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
