"""Multi-GPU data parallelism: one process per GPU, contiguous element shards.

The reference emulates the paper's MPI design with a thread pool
(pkg/src/nmk/pipeline.py:84-109, 190-276): local compute, then associative
reductions (min/max, histogram merge), global decisions taken once, and a
prefix scan of incompressible counts that places every shard's output.  Here
each rank owns the element range [elem0, elem0 + n_local) of the global
stream in its own HBM, and exactly three small exchanges go over
torch.distributed (NCCL over NVLink on the GPU box, gloo in the CPU tests):

  1. min / max / valid-count of the ratios   (pipeline.py:209-210; MPI_Allreduce)
  2. the histogram: dense u64 all-reduce SUM, or an all-gather of
     (ordinal, count) runs + merge for wide spans (binning.py:119-132)
  3. an all-gather of the per-rank incompressible counts -> exclusive scan
     (pipeline.py:257-261; MPI_Scan)

Bin selection runs redundantly and deterministically on every rank (no
broadcast).  Shard boundaries need no alignment: a rank packs its own
elements' bits at their global positions; a packed byte shared by two ranks
is completed by OR-ing both halves at assembly (pipeline.py:262-276's
neighbour exchange becomes a byte merge).  The result is byte-identical to a
single-GPU run over the concatenated field.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_bounds(n_total: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous shard of rank ``rank`` (sizes differ by at most ``align``)."""
    units = -(-n_total // align)
    lo_u = units * rank // world
    hi_u = units * (rank + 1) // world
    return min(lo_u * align, n_total), min(hi_u * align, n_total)


class ProcessGroupComm:
    """The three exchanges over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    # -- 1. ratio statistics -------------------------------------------------
    def allreduce_stats(self, stats) -> None:
        """stats: int64[4] = [bits(gmin), bits(gmax), nvalid, 0] (nmk_stats).
        One all-gather of the 32-byte records, reduced identically on every rank."""
        import torch
        gathered = torch.empty(self.world * 4, dtype=torch.int64, device=stats.device)
        self.dist.all_gather_into_tensor(gathered, stats[:4].contiguous(), group=self.group)
        g = gathered.cpu().numpy().reshape(self.world, 4)
        f = g[:, :2].copy().view(np.float64)
        nv = int(g[:, 2].sum())
        out = np.array([np.float64(f[:, 0].min()).view(np.int64), np.float64(f[:, 1].max()).view(np.int64),
                        nv, 0], dtype=np.int64)
        stats[:4].copy_(torch.from_numpy(out).to(stats.device))

    def allreduce_stats_device(self, stats) -> None:
        """Same reduction without a host copy: one all-gather of the 32-byte
        records, then MIN over gmin, MAX over gmax and SUM over the valid
        counts on the device (one collective instead of three)."""
        import torch
        g = self._stats_buf(stats)
        self.dist.all_gather_into_tensor(g, stats[:4].contiguous(), group=self.group)
        g2 = g.view(self.world, 4)
        f = g2[:, :2].contiguous().view(torch.float64)
        torch.amin(f[:, 0], dim=0, keepdim=True, out=stats[0:1].view(torch.float64))
        torch.amax(f[:, 1], dim=0, keepdim=True, out=stats[1:2].view(torch.float64))
        torch.sum(g2[:, 2], dim=0, keepdim=True, out=stats[2:3])

    def _stats_buf(self, stats):
        import torch
        buf = getattr(self, "_sbuf", None)
        if buf is None or buf.device != stats.device:
            buf = torch.empty(self.world * 4, dtype=torch.int64, device=stats.device)
            self._sbuf = buf
        return buf

    def exscan_device(self, n_inc, offset_out, prefix=None, prefix_global=None) -> None:
        """Exclusive scan of the per-rank incompressible counts on the device:
        offset_out[0] = sum over lower ranks; prefix_global = prefix + offset."""
        import torch
        allv = getattr(self, "_nbuf", None)
        if allv is None or allv.device != n_inc.device:
            allv = self._nbuf = torch.empty(self.world, dtype=torch.int64, device=n_inc.device)
        self.dist.all_gather_into_tensor(allv, n_inc.reshape(1), group=self.group)
        torch.sum(allv[: self.rank], dim=0, keepdim=True, out=offset_out) if self.rank else offset_out.zero_()
        if prefix is not None and prefix_global is not None:
            torch.add(prefix, offset_out, out=prefix_global)

    def agree_dense(self, dense: bool) -> bool:
        # every rank derives the same span from the same global (gmin, gmax)
        return dense

    # -- 2. histogram ------------------------------------------------------------
    def allreduce_counts(self, counts) -> None:
        self.dist.all_reduce(counts, op=self.dist.ReduceOp.SUM, group=self.group)

    def gather_runs(self, keys, counts, nruns):
        """All-gather every rank's sparse runs; returns concatenated (keys,
        counts) tensors on this rank's device (unmerged)."""
        import torch
        m = torch.tensor([int(nruns.reshape(-1)[0].item())], dtype=torch.int64, device=keys.device)
        sizes_t = torch.empty(self.world, dtype=torch.int64, device=keys.device)
        self.dist.all_gather_into_tensor(sizes_t, m, group=self.group)
        sizes = [int(s) for s in sizes_t.cpu().tolist()]
        mx = max(max(sizes), 1)
        pk = torch.zeros(mx, dtype=torch.int64, device=keys.device)
        pc = torch.zeros(mx, dtype=torch.int64, device=keys.device)
        pk[: sizes[self.rank]] = keys[: sizes[self.rank]]
        pc[: sizes[self.rank]] = counts[: sizes[self.rank]]
        ak = torch.empty(self.world * mx, dtype=torch.int64, device=keys.device)
        ac = torch.empty(self.world * mx, dtype=torch.int64, device=keys.device)
        self.dist.all_gather_into_tensor(ak, pk, group=self.group)
        self.dist.all_gather_into_tensor(ac, pc, group=self.group)
        ks = torch.cat([ak[r * mx: r * mx + sizes[r]] for r in range(self.world)])
        cs = torch.cat([ac[r * mx: r * mx + sizes[r]] for r in range(self.world)])
        return ks, cs

    def merge_sparse(self, keys, counts, nruns, ws):
        """Gathered runs merged on the device (nmk_hist_merge: sort by key and
        sum equal keys) -> (keys, counts, nruns) as nmk_select expects."""
        ks, cs = self.gather_runs(keys, counts, nruns)
        return merge_gathered_runs(ks, cs, ws)

    # -- 3. incompressible-count scan --------------------------------------------
    def exscan(self, value: int) -> tuple[int, int]:
        """(exclusive prefix of ``value`` over ranks, global total)."""
        import torch
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        v = torch.tensor([int(value)], dtype=torch.int64, device=dev)
        allv = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.dist.all_gather_into_tensor(allv, v, group=self.group)
        a = allv.cpu().tolist()
        return int(sum(a[: self.rank])), int(sum(a))


def merge_gathered_runs(ks, cs, ws):
    """Every rank's sparse (key, count) runs, concatenated -> one sorted
    histogram on the device (binning.merge_histograms, binning.py:119-132):
    nmk_hist_merge sorts by key and sums the counts of equal keys.  Returns
    (keys, counts, nruns) as nmk_select's sparse form expects."""
    import torch
    from . import _native as N
    from .engine import _stream
    ks, cs = ks.contiguous(), cs.contiguous()
    out_n = torch.zeros(1, dtype=torch.int64, device=ks.device)
    lib = N.lib()
    nb = lib.nmk_hist_merge_ws_bytes(ks.numel())
    buf = ws.get("hist_merge_ws", nb)
    N.check(lib.nmk_hist_merge(ks.data_ptr(), cs.data_ptr(), ks.numel(), out_n.data_ptr(), buf.data_ptr(), nb,
                               _stream()))
    if ks.numel() == 0:
        ks = torch.zeros(1, dtype=torch.int64, device=ks.device)
        cs = torch.zeros(1, dtype=torch.int64, device=ks.device)
    return ks, cs, out_n


@dataclass
class RankPart:
    """One rank's share of a compressed variable, on the host."""

    elem0: int
    n_local: int
    b0: int
    blocks: list          # per local block: bytes of the full block length
    exact: np.ndarray     # this rank's incompressible values, element order
    prefix: np.ndarray    # u64 per local block (local count before block start)
    n_inc: int


def encode_shard(base, cur, elem0: int, n_total: int, tolerance: float, bits=None,
                 block_bytes: int = 1 << 20, comm=None, ws=None, stream=None, timing=False):
    """Encode this rank's range and place it globally.

    Returns ``(DeviceEncoding, inc_offset, n_inc_total)``; ``enc.prefix`` is
    rebased in place to global prefix values for the blocks whose start this
    rank owns."""
    from . import engine
    enc = engine.encode(base, cur, tolerance, bits, block_bytes, elem0=elem0, n_total=n_total,
                        comm=comm, ws=ws, stream=stream, timing=timing)
    if comm is None:
        return enc, 0, enc.n_inc
    off, total = comm.exscan(enc.n_inc)
    if off:
        enc.prefix.add_(off)
    return enc, off, total


def rank_part_from_encoding(enc) -> RankPart:
    """Host copy of a rank's DeviceEncoding (prefix holds LOCAL counts here:
    call before rebasing, or subtract the rank offset)."""
    nlb = enc.prefix.numel()
    packed = enc.packed[: nlb * enc.stride].cpu().numpy()
    lens = enc.block_lengths()
    blocks = [packed[i * enc.stride: i * enc.stride + int(lens[i])].tobytes() for i in range(nlb)]
    return RankPart(enc.elem0, enc.n_local, enc.b0, blocks, enc.exact.cpu().numpy(),
                    enc.prefix.cpu().numpy().view(np.uint64).copy(), enc.n_inc)


def merge_parts(parts: list[RankPart], n_total: int, epb: int, bits: int):
    """Global (blocks, exact, prefix) from rank parts in rank order.

    Each byte of block b is the OR of the bytes of every rank covering it
    (a rank's bytes carry only its own elements' bits); prefix[b] comes from
    the rank owning the block's first element, offset by the exclusive scan
    of incompressible counts."""
    nblocks = -(-n_total // epb)
    lens = [(min((b + 1) * epb, n_total) - b * epb) * bits + 7 >> 3 for b in range(nblocks)]
    out = [np.zeros(lens[b], dtype=np.uint8) for b in range(nblocks)]
    prefix = np.zeros(nblocks, dtype=np.uint64)
    offsets = np.cumsum([0] + [p.n_inc for p in parts])
    for r, p in enumerate(parts):
        if p.n_local == 0:
            continue
        lo, hi = p.elem0, p.elem0 + p.n_local
        for i, blk in enumerate(p.blocks):
            b = p.b0 + i
            bs = b * epb
            e_lo = max(lo, bs) - bs
            e_hi = min(hi, min(bs + epb, n_total)) - bs
            if e_hi <= e_lo:
                continue
            y0, y1 = (e_lo * bits) >> 3, (e_hi * bits + 7) >> 3
            src = np.frombuffer(blk, dtype=np.uint8)
            out[b][y0:y1] |= src[y0:y1]
            if lo <= bs < hi:
                prefix[b] = np.uint64(int(offsets[r]) + int(p.prefix[i]))
    exact = np.concatenate([p.exact for p in parts]) if parts else np.zeros(0)
    return [o.tobytes() for o in out], exact, prefix, int(offsets[-1])
