"""GPU inflate (k_inflate.cu) against the host's zlib: the decode half of the
lossless index-table stage (codec.decompress_block, pkg/src/nmk/codec.py:119-128).
Byte-equality with zlib's output on zlib's own streams at every level (stored,
fixed and dynamic blocks, long and overlapping matches), on the GPU deflate
stage's streams, and zlib's accept/reject decision on corrupt inputs."""

import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import codec, engine, workloads  # noqa: E402


def _raw(data: bytes, level: int = 6, strategy: int = zlib.Z_DEFAULT_STRATEGY) -> bytes:
    c = zlib.compressobj(level, zlib.DEFLATED, -zlib.MAX_WBITS, 9, strategy)
    return c.compress(data) + c.flush()


def _payloads():
    rng = np.random.default_rng(0)
    yield b""
    yield b"a"
    yield b"abc" * 1000
    yield bytes(rng.integers(0, 256, 70_000, dtype=np.uint8))              # incompressible: stored blocks
    yield bytes(rng.integers(0, 4, 200_000, dtype=np.uint8))               # small alphabet
    yield bytes(np.repeat(rng.integers(0, 256, 3000, dtype=np.uint8), rng.integers(1, 300, 3000)))  # runs
    codes = np.where(rng.uniform(size=1 << 20) < 0.9, 127, rng.integers(0, 255, 1 << 20)).astype(np.uint8)
    yield codes.tobytes()                                                    # a cfg2-like packed index block


@pytest.mark.parametrize("level", [0, 1, 6, 9])
def test_inflate_equals_zlib(level):
    for data in _payloads():
        comp = _raw(data, level)
        assert codec.gpu_decompress_block(comp) == data


@pytest.mark.parametrize("strategy", [zlib.Z_FIXED, zlib.Z_HUFFMAN_ONLY, zlib.Z_RLE, zlib.Z_FILTERED])
def test_inflate_zlib_strategies(strategy):
    for data in _payloads():
        assert codec.gpu_decompress_block(_raw(data, 6, strategy)) == data


def test_inflate_many_streams_strided():
    rng = np.random.default_rng(1)
    blobs, datas = [], []
    for i in range(37):
        d = bytes(rng.integers(0, 1 + i % 7, int(rng.integers(1, 40_000)), dtype=np.uint8))
        datas.append(d)
        blobs.append(_raw(d, i % 10))
    stride = 40_064
    out, produced = codec.gpu_inflate_blocks(blobs, stride)
    host = out.cpu().numpy()
    for i, d in enumerate(datas):
        assert int(produced[i]) == len(d)
        assert host[i * stride: i * stride + len(d)].tobytes() == d


def test_inflate_gpu_deflate_streams():
    """The GPU deflate stage's streams (k_deflate.cu) inflate on the GPU."""
    base, cur = workloads.cfg2_device(64, seed=3)
    enc = engine.encode(base, cur, 1e-3, 8, 1 << 14)
    lens = enc.block_lengths()
    blobs = codec.gpu_deflate_blocks(enc.packed, enc.stride, lens)
    out, produced = codec.gpu_inflate_blocks(blobs, enc.stride)
    assert np.array_equal(produced, lens)
    for i, ln in enumerate(lens):
        a = out[i * enc.stride: i * enc.stride + int(ln)]
        b = enc.packed[i * enc.stride: i * enc.stride + int(ln)]
        assert torch.equal(a, b), i
        assert zlib.decompress(blobs[i], -15) == b.cpu().numpy().tobytes()


def test_inflate_rejects_what_zlib_rejects():
    good = _raw(b"hello world" * 500)
    bad_inputs = [
        b"\x00\x01\x02this is not deflate",   # reference test_codec.py:84-85
        good + b"extra",                      # trailing bytes (test_codec.py:89-90)
        good[: len(good) // 2],               # truncated
        b"\x07",                              # block type 3
        b"\x00\x05\x00\x00\x00",              # stored LEN/NLEN mismatch
    ]
    for data in bad_inputs:
        with pytest.raises(zlib.error):
            d = zlib.decompressobj(-15)
            d.decompress(data)
            d.flush()
            if not d.eof or d.unused_data:
                raise zlib.error("truncated or trailing")
        with pytest.raises(codec.CodecError):
            codec.gpu_decompress_block(data)
