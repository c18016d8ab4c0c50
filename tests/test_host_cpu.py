"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/nmk_b200.h declares, config validation, block geometry,
container round trip.  No kernel is launched (no GPU here)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

from paper_1703_02438_b200 import _native as N
from paper_1703_02438_b200 import codec, container, pipeline, workloads


def _header_functions():
    src = open(os.path.join(ROOT, "include", "nmk_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(nmk_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = N.load()
    names = _header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(N.SIGNATURES), "ctypes signatures out of sync with the header"
    assert lib.nmk_version() == 1


def test_struct_sizes_match_header():
    import ctypes
    assert ctypes.sizeof(N.NmkStats) == 32
    assert ctypes.sizeof(N.NmkModel) == 4 * 4 + 8 + 17 * 8
    assert ctypes.sizeof(N.NmkDecodeErr) == 16
    assert ctypes.sizeof(N.NmkSegmentInfo) == 16


def test_workspace_queries_need_no_device():
    lib = N.load()
    assert lib.nmk_minmax_ws_bytes(1 << 20) > 0
    assert lib.nmk_encode_ws_bytes(1 << 20, 0, 1 << 20, N.NMK_F64) >= 8 * (1 << 20)
    assert lib.nmk_hist_sparse_ws_bytes(1000) > 3 * 8 * 1000


def test_argument_errors_are_reported_without_device():
    lib = N.load()
    rc = lib.nmk_encode(None, None, 10, 0, 10, N.NMK_F64, None, None, 1, 8, 1e-3, 1e-3, 16, None, 16,
                        None, None, None, None, None, 0, None)
    assert rc == N.NMK_ERR_ARG
    assert b"bad argument" in lib.nmk_last_error()


@pytest.mark.parametrize("kwargs", [{"workers": 0}, {"block_bytes": 100}, {"strategy": "nope"},
                                    {"bits": 1}, {"bits": 31}, {"deflate_level": 11}, {"tolerance": 0.0}])
def test_config_rejects(kwargs):
    with pytest.raises(ValueError):
        pipeline.PipelineConfig(**kwargs)


def test_block_geometry_kats():
    layout = codec.BlockLayout(block_bytes=1 << 20, bits=13, n=3_758_400)
    assert layout.elements_per_block == 645_277 and layout.nblocks == 6
    layout = codec.BlockLayout(block_bytes=4096, bits=8, n=4096 * 4)
    assert list(layout.covering_blocks(4095, 2)) == [0, 1]
    assert list(layout.covering_blocks(100, 0)) == []


def test_deflate_stage_round_trip():
    data = bytes(range(256)) * 4
    for level in (0, 1, 6, 9):
        assert codec.decompress_block(codec.compress_block(data, level)) == data
    with pytest.raises(codec.CodecError):
        codec.decompress_block(b"\x00\x01\x02not deflate")


def test_container_round_trip(tmp_path):
    v = container.CompressedVariable(
        name="x", dtype_code=1, n=10, bits=4, tolerance=1e-3, elements_per_block=8, nblocks=2,
        n_incompressible=1, centers=np.array([0.0, 0.5]), index_offsets=np.array([0, 3], dtype=np.uint64),
        incompressible_prefix=np.array([0, 1], dtype=np.uint64), index_table=b"abcdef",
        incompressible_table=np.array([7.0]))
    p = tmp_path / "v.nmk"
    container.write_file(p, [v])
    (w,) = container.read_file(p)
    assert container.to_bytes([w]) == container.to_bytes([v])


def test_scan_file_reads_metadata_and_byte_ranges(tmp_path):
    """container.scan_file / VariableHandle (container.py:273-347): bodies stay
    on disk, byte ranges read back exactly, bounds and truncation raise."""
    vs = []
    for i, (nb, n_inc) in enumerate(((2, 1), (3, 4))):
        vs.append(container.CompressedVariable(
            name=f"v{i}", dtype_code=i % 2, n=8 * nb, bits=4, tolerance=1e-3, elements_per_block=8, nblocks=nb,
            n_incompressible=n_inc, centers=np.array([0.0, 0.5]), index_offsets=np.arange(nb, dtype=np.uint64) * 3,
            incompressible_prefix=np.array([0] + [1] * (nb - 1), dtype=np.uint64),
            index_table=bytes(range(3 * nb + 2)), incompressible_table=np.arange(n_inc, dtype=np.float64) + 7))
    p = tmp_path / "two.nmk"
    size = container.write_file(p, vs)
    hs = container.scan_file(p)
    assert [h.variable.name for h in hs] == ["v0", "v1"]
    assert sum(h.record_size() for h in hs) == size - 10
    for h, v in zip(hs, vs):
        assert len(h.variable.index_table) == 0 and h.index_table_len == len(v.index_table)
        assert h.read_index_range(1, 4) == v.index_table[1:4]
        got = h.read_incompressible_range(1, v.n_incompressible - 1)
        assert got.tobytes() == v.incompressible_table.astype(v.numpy_dtype)[1:].tobytes()
        assert container.to_bytes([h.load()]) == container.to_bytes([v])
        with pytest.raises(container.InvariantError):
            h.read_index_range(0, h.index_table_len + 1)
        with pytest.raises(container.InvariantError):
            h.read_incompressible_range(0, v.n_incompressible + 1)
    data = p.read_bytes()
    (tmp_path / "cut.nmk").write_bytes(data[:-3])
    with pytest.raises(container.TruncatedFileError):
        container.scan_file(tmp_path / "cut.nmk")
    (tmp_path / "magic.nmk").write_bytes(b"XXXX" + data[4:])
    with pytest.raises(container.BadMagicError):
        container.scan_file(tmp_path / "magic.nmk")


def test_workloads_are_seeded():
    a = workloads.cfg1_host(1000, seed=3)
    b = workloads.cfg1_host(1000, seed=3)
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    base, cur = workloads.cfg2_host(16, seed=1)
    assert base.size == 16 ** 3


def test_product_path_does_not_import_oracle():
    import subprocess
    import sys
    code = ("import sys; import paper_1703_02438_b200 as p; "
            "assert 'nmk_oracle' not in sys.modules; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.stdout.strip() == "ok", out.stderr
    pkg = os.path.join(ROOT, "paper_1703_02438_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, fn)).read().replace("no CPU fallback", ""), fn


def _swar_model(raw: bytes, bits: int) -> int:
    """Python model of k_decode.cu lane_sentinels_swar: the lane's bytes as a
    big-endian 128-bit string, 8 codes as fields from the top; a field of ~X
    is zero iff the code is the sentinel; ((Z & LO) + LO) | Z) & MSB marks the
    nonzero fields of a 64-bit word of whole fields."""
    m64 = (1 << 64) - 1
    x = int.from_bytes(raw.ljust(16, b"\0"), "big")
    hi, lo = x >> 64, x & m64
    fa = 64 // bits
    sh = fa * bits
    wb = ((hi << sh) | (lo >> (64 - sh))) & m64

    def fields(nf, msb):
        m = 0
        for e in range(nf):
            low = 64 - (e + 1) * bits
            m |= (1 << (low + bits - 1)) if msb else (((1 << (bits - 1)) - 1) << low)
        return m

    def zero_fields(w, nf):
        z = ~w & m64
        lom, msb = fields(nf, False), fields(nf, True)
        t = ((((z & lom) + lom) & m64) | z) & msb
        return nf - bin(t).count("1")

    return zero_fields(hi, fa) + zero_fields(wb, 8 - fa)


@pytest.mark.parametrize("bits", [10, 12, 14])
def test_swar_sentinel_count_model(bits):
    """The SWAR sentinel count equals a plain count of all-ones codes for
    random lanes, all-sentinel lanes and lanes cut short by the block end."""
    rng = np.random.default_rng(bits)
    sentinel = (1 << bits) - 1
    for trial in range(3000):
        codes = rng.integers(0, 1 << bits, 8)
        codes[rng.uniform(size=8) < (0.5 if trial % 3 else 1.0)] = sentinel
        acc = 0
        for c in codes:
            acc = (acc << bits) | int(c)
        raw = acc.to_bytes(bits, "big")
        keep = bits if trial % 5 else int(rng.integers(0, bits + 1))   # bytes past nbytes read as 0
        raw = raw[:keep] + b"\0" * (bits - keep)
        got = _swar_model(raw, bits)
        full = int.from_bytes(raw, "big")
        want = sum(((full >> (8 * bits - (e + 1) * bits)) & sentinel) == sentinel for e in range(8))
        assert got == want


def test_ref_dropin_plugin_binds_every_entry_point():
    """The parity-level-4 plugin finds every reference entry point it rebinds
    (CPU, in a subprocess: binding only, no kernel launches)."""
    import subprocess
    import sys
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "nmk", "pipeline.py")):
        pytest.skip("oracle/_ref not vendored")
    code = ("import ref_dropin, nmk, paper_1703_02438_b200 as o; p = ref_dropin.install(); "
            "assert nmk.pipeline.compress_pair is o.pipeline.compress_pair; "
            "assert nmk.binning.top_k_bins is o.binning.top_k_bins; "
            "assert nmk.codec.partial_decode is o.codec.partial_decode; "
            "print(sum(len(v) for v in p.values()))")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), ROOT]))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "19"


def test_deflate_segment_size_rule():
    """The GPU deflate stage takes the largest segment that still leaves one
    warp's worth of work for >= 2048 warps (codec.deflate_segment_bytes)."""
    from paper_1703_02438_b200 import codec
    assert codec.deflate_segment_bytes(128 << 20) == 65520
    assert codec.deflate_segment_bytes(64 << 20 | 1) == 32768
    assert codec.deflate_segment_bytes(39 << 20) == 16384
    assert codec.deflate_segment_bytes(1) == 16384
    for total in (1, 1 << 20, 1 << 27, 1 << 33):
        seg = codec.deflate_segment_bytes(total)
        assert seg % 16 == 0 and 64 <= seg <= 65535
