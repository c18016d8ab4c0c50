"""Multi-GPU data path emulated on one GPU: the element range of every rank
is encoded by the real per-range kernels (elem0 / n_total geometry, zero
bits outside the range), the exchanges return the global values, and the
parts are assembled with distributed.merge_parts.  The result must equal the
single-range encode byte for byte, and every rank must decode its own range.
(Ranks run one after another: no kernel waits on another rank's kernel.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import _native as N, distributed as D, engine, workloads  # noqa: E402


class EmulatedComm:
    """Exchanges of ProcessGroupComm answered from a full-range pass."""

    def __init__(self, full_stats, full_counts=None, full_sparse=None):
        self.full_stats, self.full_counts, self.full_sparse = full_stats, full_counts, full_sparse

    def allreduce_stats(self, stats):
        stats.copy_(self.full_stats)

    def agree_dense(self, dense):
        return dense

    def allreduce_counts(self, counts):
        counts.copy_(self.full_counts[: counts.numel()])

    def merge_sparse(self, keys, counts, nruns, ws):
        return self.full_sparse


def _full_exchanges(base, cur, E):
    lib = N.lib()
    st = torch.cuda.current_stream().cuda_stream
    n = base.numel()
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    mm = torch.zeros(lib.nmk_minmax_ws_bytes(n), dtype=torch.uint8, device="cuda")
    dt = engine.torch_dtype_code(base)
    N.check(lib.nmk_minmax(base.data_ptr(), cur.data_ptr(), n, dt, stats.data_ptr(), None, mm.data_ptr(), mm.numel(),
                           st))
    sv = engine._read_struct(stats, N.NmkStats)
    width = 2.0 * E
    span = (sv.gmax - sv.gmin) / width
    if np.isfinite(span) and span < engine.DENSE_MAX_BINS:
        nb = int(np.floor(span)) + 1
        counts = torch.zeros(nb + 1, dtype=torch.int64, device="cuda")
        N.check(lib.nmk_hist_dense(base.data_ptr(), cur.data_ptr(), n, dt, stats.data_ptr(), width, nb,
                                   counts.data_ptr(), st))
        return EmulatedComm(stats, full_counts=counts)
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    cnts = torch.empty(n, dtype=torch.int64, device="cuda")
    nruns = torch.zeros(1, dtype=torch.int64, device="cuda")
    wsb = torch.empty(lib.nmk_hist_sparse_ws_bytes(n), dtype=torch.uint8, device="cuda")
    N.check(lib.nmk_hist_sparse(base.data_ptr(), cur.data_ptr(), n, dt, stats.data_ptr(), width, keys.data_ptr(),
                                cnts.data_ptr(), nruns.data_ptr(), wsb.data_ptr(), wsb.numel(), st))
    return EmulatedComm(stats, full_sparse=(keys, cnts, nruns))


def _blocks(enc):
    nlb = enc.prefix.numel()
    packed = enc.packed[: nlb * enc.stride].cpu().numpy()
    lens = enc.block_lengths()
    return [packed[i * enc.stride: i * enc.stride + int(lens[i])].tobytes() for i in range(nlb)]


@pytest.mark.parametrize("case,world", [("cfg1", 2), ("cfg1", 5), ("cfg5_b10", 3), ("outliers", 4),
                                        ("f32_b12", 3)])
def test_sharded_encode_equals_single(case, world):
    if case == "cfg1":
        b, c = workloads.cfg1_host(1 << 19, seed=6); E, bits, bb = 1e-3, 8, 1 << 14
    elif case == "cfg5_b10":
        b, c = workloads.cfg5_host(300_007, seed=7); E, bits, bb = 1e-3, 10, 1 << 13
    elif case == "outliers":
        b, c = workloads.outlier_pair(100_003, seed=8); E, bits, bb = 1e-3, 2, 4096
    else:
        b, c = workloads.uniform_pair(200_001, seed=9, dtype=np.float32, spread=0.3); E, bits, bb = 1e-3, 12, 1 << 13
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    n = base.numel()
    single = engine.encode(base, cur, E, bits, bb)
    ref_blocks, ref_exact = _blocks(single), single.exact.cpu().numpy().copy()
    ref_prefix = single.prefix.cpu().numpy().view(np.uint64).copy()
    ref_out = engine.decode_encoding(single, base).out.cpu().numpy()
    comm = _full_exchanges(base, cur, E)
    rng = np.random.default_rng(world)
    cuts = sorted({0, n, *rng.integers(1, n, world - 1).tolist()})   # unaligned on purpose
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        ws = engine.Workspace()
        bs, cs = base[lo:hi].clone(), cur[lo:hi].clone()
        enc = engine.encode(bs, cs, E, bits, bb, elem0=lo, n_total=n, comm=comm, ws=ws)
        assert enc.bits == single.bits and enc.k == single.k
        parts.append(D.rank_part_from_encoding(enc))
        # each rank decodes its own range from its own stream
        out = engine.decode_encoding(enc, bs, ws=ws)
        assert not out.bad_index and not out.exhausted
        assert out.out.cpu().numpy().tobytes() == ref_out[lo:hi].tobytes()
    blocks, exact, prefix, n_inc = D.merge_parts(parts, n, single.epb, single.bits)
    assert n_inc == single.n_inc
    assert blocks == ref_blocks
    assert exact.tobytes() == ref_exact.tobytes()
    assert prefix.tobytes() == ref_prefix.tobytes()


# ---------------------------------------------------------------------------
# sparse histogram merge across ranks (binning.merge_histograms, A4)
# ---------------------------------------------------------------------------

def _sparse_hist(base, cur, stats, E):
    lib = N.lib()
    n = base.numel()
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    cnts = torch.empty(n, dtype=torch.int64, device="cuda")
    nruns = torch.zeros(1, dtype=torch.int64, device="cuda")
    wsb = torch.empty(lib.nmk_hist_sparse_ws_bytes(n), dtype=torch.uint8, device="cuda")
    N.check(lib.nmk_hist_sparse(base.data_ptr(), cur.data_ptr(), n, engine.torch_dtype_code(base), stats.data_ptr(),
                                2.0 * E, keys.data_ptr(), cnts.data_ptr(), nruns.data_ptr(), wsb.data_ptr(),
                                wsb.numel(), torch.cuda.current_stream().cuda_stream))
    m = int(nruns.item())
    return keys[:m].clone(), cnts[:m].clone()


class GatheringComm(EmulatedComm):
    """merge_sparse runs the production merge (distributed.merge_gathered_runs
    -> nmk_hist_merge) over every rank's own sparse runs, as
    ProcessGroupComm.merge_sparse does after its all-gather."""

    def __init__(self, full_stats, rank_runs):
        super().__init__(full_stats)
        self.rank_runs = rank_runs

    def merge_sparse(self, keys, counts, nruns, ws):
        ks = torch.cat([k for k, _ in self.rank_runs])
        cs = torch.cat([c for _, c in self.rank_runs])
        return D.merge_gathered_runs(ks, cs, ws)


@pytest.mark.parametrize("world", [2, 3, 7])
def test_sparse_merge_across_ranks(world):
    """Planted outliers (a 5e8-bin span, sparse path): every rank histograms
    its own range, the runs are merged on the device, and the result equals
    the single-range sparse histogram and the single-range encode."""
    E, bits, bb = 1e-3, 8, 4096
    b, c = workloads.outlier_pair(200_003, seed=world)
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    n = base.numel()
    comm0 = _full_exchanges(base, cur, E)
    assert comm0.full_sparse is not None
    full_k, full_c, full_n = comm0.full_sparse
    m = int(full_n.item())
    rng = np.random.default_rng(world)
    cuts = sorted({0, n, *rng.integers(1, n, world - 1).tolist()})
    runs = [_sparse_hist(base[lo:hi].clone(), cur[lo:hi].clone(), comm0.full_stats, E)
            for lo, hi in zip(cuts[:-1], cuts[1:])]
    assert sum(int(k.numel()) for k, _ in runs) > m        # some bins are split across ranks
    mk, mc, mn = D.merge_gathered_runs(torch.cat([k for k, _ in runs]), torch.cat([c for _, c in runs]),
                                       engine.Workspace())
    assert int(mn.item()) == m
    assert torch.equal(mk[:m], full_k[:m]) and torch.equal(mc[:m], full_c[:m])
    # the merged histogram drives each rank's encode: same bytes as one range
    single = engine.encode(base, cur, E, bits, bb)
    assert single.hist_form == "sparse"
    comm = GatheringComm(comm0.full_stats, runs)
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        enc = engine.encode(base[lo:hi].clone(), cur[lo:hi].clone(), E, bits, bb, elem0=lo, n_total=n, comm=comm,
                            ws=engine.Workspace())
        assert enc.hist_form == "sparse" and enc.k == single.k
        parts.append(D.rank_part_from_encoding(enc))
    blocks, exact, prefix, n_inc = D.merge_parts(parts, n, single.epb, single.bits)
    assert n_inc == single.n_inc
    assert blocks == _blocks(single)
    assert exact.tobytes() == single.exact.cpu().numpy().tobytes()
    assert prefix.tobytes() == single.prefix.cpu().numpy().view(np.uint64).tobytes()


# ---------------------------------------------------------------------------
# the sync-free pipeline (bench.py's multi-GPU path) on shards with elem0 > 0
# ---------------------------------------------------------------------------

class DeviceEmulatedComm:
    """DevicePipeline's device-side exchanges for one rank, answered from the
    full range without a host round trip: stats and histogram copied from a
    full-range pass, the incompressible offset = sum over the lower ranks."""

    def __init__(self, world, full_stats, full_counts, offset):
        self.world, self.full_stats, self.full_counts, self.offset = world, full_stats, full_counts, offset

    def allreduce_stats_device(self, stats):
        stats[:3].copy_(self.full_stats[:3])

    def allreduce_counts(self, counts):
        m = min(counts.numel(), self.full_counts.numel())
        counts.zero_()
        counts[:m].copy_(self.full_counts[:m])

    def exscan_device(self, n_inc, offset_out, prefix=None, prefix_global=None):
        offset_out.fill_(self.offset)
        if prefix is not None and prefix_global is not None:
            torch.add(prefix, offset_out, out=prefix_global)


@pytest.mark.parametrize("case,world", [("cfg2", 2), ("cfg1", 3), ("cfg5_b10", 4), ("f32_b12", 3)])
def test_device_pipeline_shards(case, world):
    if case == "cfg2":
        b, c = workloads.cfg2_host(128, seed=3); E, bits, bb = 1e-3, 8, 1 << 16
    elif case == "cfg1":
        b, c = workloads.cfg1_host(1 << 20, seed=11); E, bits, bb = 1e-3, 8, 1 << 15
    elif case == "cfg5_b10":
        b, c = workloads.cfg5_host(700_001, seed=12); E, bits, bb = 1e-3, 10, 1 << 14
    else:
        b, c = workloads.uniform_pair(500_003, seed=13, dtype=np.float32, spread=0.3); E, bits, bb = 1e-3, 12, 1 << 14
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    n = base.numel()
    full = engine.DevicePipeline(n, base.dtype, E, bits, bb)
    ref_out = torch.empty_like(base)
    full.step(base, cur, ref_out)
    fchk = full.check()
    assert fchk["status"] == 0
    single = full.encoding()
    rng = np.random.default_rng(world + 100)
    cuts = sorted({0, n, *rng.integers(1, n, world - 1).tolist()})
    parts, offset = [], 0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        comm = DeviceEmulatedComm(world, full.stats, full.counts, offset)
        pipe = engine.DevicePipeline(hi - lo, base.dtype, E, bits, bb, elem0=lo, n_total=n, comm=comm)
        bs, cs = base[lo:hi].clone(), cur[lo:hi].clone()
        out = torch.empty_like(bs)
        pipe.step(bs, cs, out)
        chk = pipe.check()
        assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
        assert chk["k"] == fchk["k"] and chk["n_sentinel"] == chk["n_inc"]
        assert torch.equal(out.view(torch.uint8), ref_out[lo:hi].view(torch.uint8))
        enc = pipe.encoding()
        parts.append(D.rank_part_from_encoding(enc))
        # global prefix of the blocks whose first element this rank owns
        gp = pipe.prefix_global.cpu().numpy()
        sp = single.prefix.cpu().numpy()
        for i in range(pipe.nlb):
            blk = pipe.b0 + i
            if lo <= blk * pipe.epb < hi:
                assert gp[i] == sp[blk], (lo, blk)
        offset += chk["n_inc"]
    blocks, exact, prefix, n_inc = D.merge_parts(parts, n, single.epb, single.bits)
    assert n_inc == single.n_inc
    assert blocks == _blocks(single)
    assert exact.tobytes() == single.exact.cpu().numpy().tobytes()
    assert prefix.tobytes() == single.prefix.cpu().numpy().view(np.uint64).tobytes()
