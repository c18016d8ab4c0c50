"""Multi-process host logic of the multi-GPU path on CPU (gloo, world size 2).

Covered: the three exchanges of ProcessGroupComm (stats, histogram counts,
sparse runs, incompressible-count scan — host and device-tensor variants) and
the byte-OR assembly of rank parts (merge_parts).  The per-rank encoder is
emulated with the oracle (test infrastructure) restating K4's contract for an
element range: bits at their global positions, zero bits outside the range,
local exact values, local per-block prefix.  The assembled result must equal
the single-process oracle encode byte for byte.
"""

import os
import socket

import numpy as np
import pytest

import nmk_oracle as O
from paper_1703_02438_b200 import distributed as D
from paper_1703_02438_b200 import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def emulate_rank_part(enc, cur, e0, e1):
    """What K4 produces for [e0, e1) of the global stream (CPU stand-in)."""
    epb, bits, n = enc["epb"], enc["bits"], enc["n"]
    codes = enc["codes"].copy()
    b0, b1 = e0 // epb, (e1 - 1) // epb
    blocks = []
    for b in range(b0, b1 + 1):
        s, e = b * epb, min((b + 1) * epb, n)
        c = codes[s:e].copy()
        c[: max(e0 - s, 0)] = 0
        c[max(e1 - s, 0):] = 0
        blocks.append(O.pack(c, bits))
    flags = enc["flags"][e0:e1]
    exact = cur[e0:e1][~flags]
    prefix = np.zeros(b1 - b0 + 1, dtype=np.uint64)
    inc = ~flags
    for i, b in enumerate(range(b0, b1 + 1)):
        if b * epb >= e0:
            prefix[i] = int(inc[: b * epb - e0].sum())
    return D.RankPart(e0, e1 - e0, b0, blocks, exact, prefix, int(inc.sum()))


@pytest.mark.parametrize("world,n,bits,block_bytes", [(2, 30011, 10, 4096), (3, 50000, 8, 4096),
                                                      (4, 8191, 3, 4096), (5, 100, 8, 4096)])
def test_merge_parts_equals_single_encode(world, n, bits, block_bytes):
    base, cur = workloads.cfg5_host(n, seed=world)
    enc = O.encode(base, cur, 1e-3, bits, block_bytes)
    # unaligned shard boundaries on purpose: boundary bytes are shared
    cuts = sorted({0, n, *np.random.default_rng(world).integers(1, n, world - 1).tolist()})
    parts = [emulate_rank_part(enc, cur, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    blocks, exact, prefix, n_inc = D.merge_parts(parts, n, enc["epb"], bits)
    assert blocks == enc["blocks"]
    assert exact.tobytes() == enc["exact"].tobytes()
    assert prefix.tobytes() == enc["prefix"].tobytes()
    assert n_inc == enc["n_inc"]


def test_shard_bounds_cover_and_align():
    for world in (1, 2, 3, 8):
        got = [D.shard_bounds(1000003, world, r, align=8) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == 1000003
        assert all(a[1] == b[0] for a, b in zip(got[:-1], got[1:]))
        assert all(a % 8 == 0 for a, _ in got)


def _worker(rank, world, port, n, bits, q):
    try:
        _worker_body(rank, world, port, n, bits, q)
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, {"exception": repr(exc)}))
        raise


def _worker_body(rank, world, port, n, bits, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.ProcessGroupComm()
        base, cur = workloads.cfg5_host(n, seed=11)
        lo, hi = D.shard_bounds(n, world, rank)
        r, v = O.ratios_of(base[lo:hi], cur[lo:hi])
        mm = O.minmax_of(r, v)
        inf = np.float64(np.inf)
        stats = torch.tensor([np.float64(mm[0] if mm else inf).view(np.int64),
                              np.float64(mm[1] if mm else -inf).view(np.int64), int(v.sum()), 0],
                             dtype=torch.int64)
        stats2 = stats.clone()
        comm.allreduce_stats(stats)
        comm.allreduce_stats_device(stats2)
        rg, vg = O.ratios_of(base, cur)
        gmin, gmax = O.minmax_of(rg, vg)
        ok = {}
        for nm, st in (("stats", stats), ("stats_device", stats2)):
            f = st[:2].numpy().view(np.float64)
            ok[nm] = (f[0] == gmin and f[1] == gmax and int(st[2]) == int(vg.sum()))
        # dense histogram counts
        w = 2e-3
        q_local = O.bin_ordinals(r[v], gmin, w).astype(np.int64)
        nb = int(np.floor((gmax - gmin) / w)) + 1
        counts = torch.from_numpy(np.bincount(q_local, minlength=nb + 1).astype(np.int64))
        comm.allreduce_counts(counts)
        keys, cnts = O.histogram(rg[vg], gmin, w)
        dense = np.zeros(nb + 1, dtype=np.int64)
        dense[keys.astype(np.int64)] = cnts
        ok["counts"] = bool((counts.numpy() == dense).all())
        # sparse runs
        lk, lc = O.histogram(r[v], gmin, w)
        kt = torch.from_numpy(lk.view(np.int64).copy())
        ct = torch.from_numpy(lc.copy())
        ks, cs = comm.gather_runs(kt, ct, torch.tensor([lk.size], dtype=torch.int64))
        mk, inv = np.unique(ks.numpy().view(np.float64), return_inverse=True)
        mc = np.zeros(mk.size, dtype=np.int64)
        np.add.at(mc, inv, cs.numpy())
        ok["sparse"] = mk.size == keys.size and bool((mk == keys).all() and (mc == cnts).all())
        # incompressible-count scan (host and device forms)
        enc = O.encode(base, cur, 1e-3, bits, 4096)
        part = emulate_rank_part(enc, cur, lo, hi)
        off, tot = comm.exscan(part.n_inc)
        n_inc_t = torch.tensor([part.n_inc], dtype=torch.int64)
        off_t = torch.zeros(1, dtype=torch.int64)
        pre = torch.from_numpy(part.prefix.view(np.int64).copy())
        pre_g = torch.zeros_like(pre)
        comm.exscan_device(n_inc_t, off_t, pre, pre_g)
        ok["exscan"] = tot == enc["n_inc"] and int(off_t) == off and bool((pre_g - pre == off).all())
        parts = [None] * world
        dist.all_gather_object(parts, part)
        if rank == 0:
            blocks, exact, prefix, n_inc = D.merge_parts(parts, n, enc["epb"], bits)
            ok["merge"] = (blocks == enc["blocks"] and exact.tobytes() == enc["exact"].tobytes()
                           and prefix.tobytes() == enc["prefix"].tobytes() and n_inc == enc["n_inc"])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_exchanges_and_assembly(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 40_009, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok in results.items():
        assert all(ok.values()), (rank, ok)
    assert "merge" in results[0]
