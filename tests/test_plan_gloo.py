"""CPU multi-rank coverage of the N > 1 host logic: world_size 2 and 4 gloo
process groups derive the space_repartition consensus and the balance +
allgatherv plan through libokt.so's planning entry points (the same code the
device orchestration runs), move the data with gloo send/recv, and must end
with the reference's results (oracle) and ledger counts."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, P, port, scenario, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=P)
        from oracle import Oracle
        from paper_2201_07598_b200 import _lib
        L = _lib.lib()
        orc = Oracle()
        out = {}
        if scenario == "cuts":
            n = 5000
            sels = []
            for r in range(P):
                g = orc.random_dense(400 + r, n)
                th = orc.kth_largest_mag(g, 50 + 7 * r)
                sels.append(orc.select(g, th)[0])
            mine = sels[rank]
            m = mine.size
            prop = [0] + [int(mine[(j * m) // P]) if m else j * n // P for j in range(1, P)] + [n]
            allp = [torch.zeros(P + 1, dtype=torch.int64) for _ in range(P)]
            dist.all_gather(allp, torch.tensor(prop, dtype=torch.int64))
            flat = (ctypes.c_uint64 * (P * (P + 1)))(*[int(x) for t in allp for x in t.tolist()])
            cuts = (ctypes.c_uint64 * (P + 1))()
            assert L.okt_plan_cuts(flat, P, n, cuts) == 0
            out["cuts"] = list(cuts)
            out["want"] = orc.space_repartition(sels, n)
            c = _lib.OktCounters()
            assert L.okt_plan_ledger(rank, P, 2, None, P + 1, 0, ctypes.byref(c)) == 0
            out["consensus_words"] = c.words_sent
        else:
            # survivors: skewed (everything at rank 0) or spread
            rng = np.random.default_rng(7)
            n = 10_000
            sizes = [120, 0, 0, 0][:P] if scenario == "skew" else [5 + 3 * r for r in range(P)]
            stream_idx = np.sort(rng.choice(n, size=sum(sizes), replace=False)).astype(np.int64)
            stream_val = rng.standard_normal(sum(sizes))
            off = np.concatenate([[0], np.cumsum(sizes)])
            my_idx = torch.from_numpy(stream_idx[off[rank]:off[rank + 1]].copy())
            my_val = torch.from_numpy(stream_val[off[rank]:off[rank + 1]].copy())
            got = [torch.zeros(1, dtype=torch.int64) for _ in range(P)]
            dist.all_gather(got, torch.tensor([my_idx.numel()], dtype=torch.int64))
            sz = (ctypes.c_uint64 * P)(*[int(t.item()) for t in got])
            bal = ctypes.c_int()
            sends = (_lib.OktPiece * P)()
            recvs = (_lib.OktPiece * P)()
            ns, nr = ctypes.c_int(), ctypes.c_int()
            own = _lib.OktPiece()
            poff = (ctypes.c_uint64 * P)()
            psz = (ctypes.c_uint64 * P)()
            assert L.okt_plan_balance(rank, P, sz, ctypes.byref(bal), sends, ctypes.byref(ns), recvs,
                                      ctypes.byref(nr), ctypes.byref(own), poff, psz) == 0
            total = sum(sz)
            u_idx = torch.full((total,), -1, dtype=torch.int64)
            u_val = torch.zeros(total, dtype=torch.float64)
            base = off[rank]
            if own.end > own.begin:
                u_idx[own.begin:own.end] = my_idx[own.begin - base:own.end - base]
                u_val[own.begin:own.end] = my_val[own.begin - base:own.end - base]
            reqs = []
            for i in range(ns.value):
                p = sends[i]
                reqs.append(dist.isend(my_idx[p.begin - base:p.end - base].clone(), p.peer))
                reqs.append(dist.isend(my_val[p.begin - base:p.end - base].clone(), p.peer))
            bufs = []
            for i in range(nr.value):
                p = recvs[i]
                bi = torch.empty(p.end - p.begin, dtype=torch.int64)
                bv = torch.empty(p.end - p.begin, dtype=torch.float64)
                reqs.append(dist.irecv(bi, p.peer))
                reqs.append(dist.irecv(bv, p.peer))
                bufs.append((p, bi, bv))
            for r_ in reqs:
                r_.wait()
            for p, bi, bv in bufs:
                u_idx[p.begin:p.end] = bi
                u_val[p.begin:p.end] = bv
            # allgatherv of the (balanced) parts straight into u
            reqs = []
            a, b = poff[rank], poff[rank] + psz[rank]
            for peer in range(P):
                if peer == rank:
                    continue
                reqs.append(dist.isend(u_idx[a:b].clone(), peer))
                reqs.append(dist.isend(u_val[a:b].clone(), peer))
            recv_bufs = []
            for peer in range(P):
                if peer == rank:
                    continue
                pa, pb = poff[peer], poff[peer] + psz[peer]
                bi = torch.empty(pb - pa, dtype=torch.int64)
                bv = torch.empty(pb - pa, dtype=torch.float64)
                reqs.append(dist.irecv(bi, peer))
                reqs.append(dist.irecv(bv, peer))
                recv_bufs.append((pa, pb, bi, bv))
            for r_ in reqs:
                r_.wait()
            for pa, pb, bi, bv in recv_bufs:
                u_idx[pa:pb] = bi
                u_val[pa:pb] = bv
            out["u_ok"] = bool(np.array_equal(u_idx.numpy(), stream_idx) and np.array_equal(u_val.numpy(), stream_val))
            out["balanced"] = bal.value
            cb, ca = _lib.OktCounters(), _lib.OktCounters()
            assert L.okt_plan_ledger(rank, P, 4, sz, 0, 0, ctypes.byref(cb)) == 0
            assert L.okt_plan_ledger(rank, P, 1, psz, 0, 0, ctypes.byref(ca)) == 0
            out["balance"] = (cb.words_sent, cb.msgs_sent, cb.words_recv, cb.msgs_recv)
            out["allgatherv_recv_words"] = ca.words_recv
            out["total"] = total
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def run(P, scenario):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, scenario, q)) for r in range(P)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(P):
        r, out, err = q.get(timeout=180)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("P", [2, 4])
def test_consensus_cuts_over_gloo(P):
    res = run(P, "cuts")
    for r in range(P):
        assert res[r]["cuts"] == res[0]["want"]
        assert res[r]["consensus_words"] == (P + 1) * (P.bit_length() - 1)


@pytest.mark.parametrize("P", [2, 4])
def test_spread_survivors_allgatherv_over_gloo(P):
    res = run(P, "spread")
    for r in range(P):
        assert res[r]["u_ok"] and res[r]["balanced"] == 0
        assert res[r]["balance"] == (0, 0, 0, 0)
        assert res[r]["allgatherv_recv_words"] == 2 * (res[r]["total"] - (5 + 3 * r))


def test_skewed_survivors_rebalance_over_gloo():
    # test_oktopk.cpp:249-275 with 120 survivors at rank 0 of 4: blocks of 30
    # move to ranks 1..3 (90 entries = 180 words in 3 messages).
    res = run(4, "skew")
    assert all(res[r]["u_ok"] and res[r]["balanced"] == 1 for r in range(4))
    assert res[0]["balance"] == (180, 3, 0, 0)
    for r in range(1, 4):
        assert res[r]["balance"] == (0, 0, 60, 1)
