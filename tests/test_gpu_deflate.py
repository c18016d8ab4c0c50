"""The optional GPU lossless stage (k_deflate.cu): every stream
it emits is a valid raw DEFLATE stream that zlib inflates back to the packed
bytes exactly; .nmk files written with it decompress through the unchanged
host inflate path to the same values as the default (zlib) stage."""

import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import codec, container, engine, pipeline, workloads  # noqa: E402
from paper_1703_02438_b200.core import TemporalPair  # noqa: E402


def _inflate(data: bytes) -> bytes:
    d = zlib.decompressobj(-zlib.MAX_WBITS)
    out = d.decompress(data) + d.flush()
    assert d.eof and not d.unused_data
    return out


def _blocks_on_device(blocks, stride):
    buf = np.zeros(len(blocks) * stride, dtype=np.uint8)
    for i, b in enumerate(blocks):
        buf[i * stride: i * stride + len(b)] = np.frombuffer(b, dtype=np.uint8)
    return torch.from_numpy(buf).cuda()


def test_index_stream_shapes_compress(tmp_path):
    """B = 10 (period-5 byte pattern) and B = 12 noisy streams: exact round
    trip, and the ratio stays within reach of zlib's (fewer match candidates
    than zlib's hash chains: 7.4 vs 8.4 on cfg3, 1.19 vs 1.20 on cfg5)."""
    for (b, c), E, bits, lo in ((workloads.cfg5_host(1 << 19, seed=5), 1e-4, 12, 0.97),
                                (tuple(workloads.cfg3_host(shape=(4, 240, 480), steps=2, seed=3)[:2]), 5e-3, 10, 0.75)):
        enc = engine.encode(torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda(), E, bits, 1 << 16)
        lens = enc.block_lengths()
        gpu = codec.gpu_deflate_blocks(enc.packed, enc.stride, lens)
        packed = enc.packed.cpu().numpy()
        tot_gpu = tot_zlib = 0
        for i, (g, ln) in enumerate(zip(gpu, lens)):
            raw = packed[i * enc.stride: i * enc.stride + int(ln)].tobytes()
            assert _inflate(g) == raw
            tot_gpu += len(g)
            tot_zlib += len(codec.compress_block(raw))
        assert tot_zlib > lo * tot_gpu, (bits, tot_gpu, tot_zlib)


def _patterns(rng, n):
    yield rng.integers(0, 256, n, dtype=np.uint8).tobytes()                      # incompressible
    yield bytes(n)                                                                # one long run
    yield (np.arange(n) % 7).astype(np.uint8).tobytes()                          # short period
    x = np.full(n, 127, dtype=np.uint8)                                           # index-stream-like
    pos = rng.choice(n, n // 50, replace=False)
    x[pos] = rng.integers(0, 255, pos.size)
    yield x.tobytes()
    yield np.repeat(rng.integers(0, 256, n // 300 + 1, dtype=np.uint8), 300)[:n].tobytes()


@pytest.mark.parametrize("seg", [64, 1024, 8192, 65520])
@pytest.mark.parametrize("n,last", [(1, 1), (100_000, 100_000), (70_000, 12_345), (4096, 17)])
def test_streams_inflate_exactly(seg, n, last):
    rng = np.random.default_rng(seg + n)
    for data in _patterns(rng, n):
        nb = 3 if last != n else 1
        blocks = [data] * (nb - 1) + [data[:last]]
        stride = (n + 15) // 16 * 16
        out = codec.gpu_deflate_blocks(_blocks_on_device(blocks, stride), stride, [len(b) for b in blocks], seg)
        assert len(out) == nb
        for o, b in zip(out, blocks):
            assert _inflate(o) == b


def test_compression_of_real_index_streams():
    """cfg2 packed stream: inflates exactly and compresses about as well as
    zlib level 6 (the cost-aware parse: ratio 6.21 vs 6.20 on the 512^3 stream,
    10.6 vs 11.9 on this 256^3 one, whose longer repeats favour zlib's chains)."""
    base, cur = workloads.cfg2_device(256, seed=0)
    enc = engine.encode(base, cur, 1e-3, 8)
    lens = enc.block_lengths()
    gpu = codec.gpu_deflate_blocks(enc.packed, enc.stride, lens)
    packed = enc.packed.cpu().numpy()
    tot_gpu = tot_zlib = 0
    for b, (g, ln) in enumerate(zip(gpu, lens)):
        raw = packed[b * enc.stride: b * enc.stride + int(ln)].tobytes()
        assert _inflate(g) == raw
        tot_gpu += len(g)
        tot_zlib += len(codec.compress_block(raw))
    assert tot_gpu < 1.2 * tot_zlib, (tot_gpu, tot_zlib)
    assert tot_gpu < 0.25 * int(sum(lens))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pipeline_gpu_deflate_round_trip(tmp_path, dtype):
    b, c = workloads.cfg5_host(200_003, seed=71)
    b, c = b.astype(dtype), c.astype(dtype)
    host_cfg = pipeline.PipelineConfig(tolerance=1e-3, bits=10, block_bytes=1 << 14)
    gpu_cfg = pipeline.PipelineConfig(tolerance=1e-3, bits=10, block_bytes=1 << 14, deflate="gpu")
    v_host, _ = pipeline.compress_pair(TemporalPair(b, c), host_cfg, name="h")
    v_gpu, t = pipeline.compress_pair(TemporalPair(b, c), gpu_cfg, name="g")
    assert t.zlib >= 0.0
    # same model and exact values; same index stream after inflate
    assert v_gpu.centers.tobytes() == v_host.centers.tobytes()
    assert v_gpu.incompressible_table.tobytes() == v_host.incompressible_table.tobytes()
    assert (codec.decode_all_indices(v_gpu) == codec.decode_all_indices(v_host)).all()
    path = tmp_path / "g.nmk"
    container.write_file(path, [v_gpu])
    (w,) = container.read_file(path)
    assert pipeline.decompress(w, b).tobytes() == pipeline.decompress(v_host, b).tobytes()
    h = container.scan_file(path)[0]
    s, n = 20_000, 50_000
    assert codec.partial_decode_file(h, s, n, b[s:s + n]).tobytes() == pipeline.decompress(v_host, b)[s:s + n].tobytes()


def test_config_rejects_unknown_engine():
    with pytest.raises(ValueError):
        pipeline.PipelineConfig(deflate="cpu")


def test_deflate_adversarial_patterns():
    """Warp-per-segment deflate on inputs that stress its parse: every period
    2..40, runs that cross step and segment edges, far repeats (up to the
    32 KiB window and beyond the segment), tiny and ragged segments."""
    rng = np.random.default_rng(77)
    cases = []
    for period in list(range(2, 41)) + [63, 64, 65, 257, 258, 259, 4095, 4096, 4097]:
        unit = rng.integers(0, 256, period, dtype=np.uint8)
        x = np.tile(unit, 40_000 // period + 1)[:40_000].copy()
        x[rng.choice(x.size, 200, replace=False)] ^= 0x5a          # sparse deviations
        cases.append(x.tobytes())
    blockrep = rng.integers(0, 256, 3000, dtype=np.uint8)
    cases.append(np.concatenate([blockrep, rng.integers(0, 256, 29_000, dtype=np.uint8), blockrep,
                                 rng.integers(0, 4, 20_000, dtype=np.uint8), blockrep]).tobytes())
    cases.append(bytes([255]) * 70_001)
    cases.append(bytes(range(256)) * 300)
    for data in cases:
        for seg in (64, 4096, 16384, 65520):
            n = len(data)
            stride = (n + 15) // 16 * 16
            out = codec.gpu_deflate_blocks(_blocks_on_device([data], stride), stride, [n], seg)
            assert _inflate(out[0]) == data, (n, seg)
    for n in (1, 2, 3, 4, 5, 31, 32, 33, 63, 64, 65, 257, 258, 259, 260):   # shorter than a match, a step, a probe
        data = bytes((7 * i) % 3 for i in range(n))
        stride = (n + 15) // 16 * 16
        for seg in (64, 128):
            out = codec.gpu_deflate_blocks(_blocks_on_device([data] * 2, stride), stride, [n, n], seg)
            assert [_inflate(o) for o in out] == [data, data], (n, seg)
