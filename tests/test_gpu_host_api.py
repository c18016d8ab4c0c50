"""Host-buffer entry points (what the e2e benchmark times): encode_host /
decode_host and the overlapped StreamCompressor must give the oracle's bytes
and reconstruction for every step of a stream."""

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import pipeline, workloads  # noqa: E402


def _blocks(h):
    return [bytes(h.block(b)) for b in range(h.b0, h.b0 + len(h.prefix))]


@pytest.mark.parametrize("case", ["cfg1", "cfg5_f32"])
def test_encode_decode_host_match_oracle(case):
    if case == "cfg1":
        b, c = workloads.cfg1_host(1 << 18, seed=11); E, bits, bb = 1e-3, 8, 1 << 14
    else:
        b, c = workloads.uniform_pair(150_001, seed=12, dtype=np.float32, spread=0.2); E, bits, bb = 1e-3, 10, 1 << 13
    cfg = pipeline.PipelineConfig(tolerance=E, bits=bits, block_bytes=bb)
    h = pipeline.encode_host(b, c, cfg)
    o = O.encode(b, c, E, bits, bb)
    assert h.n_inc == o["n_inc"] and h.k == len(o["centers"])
    assert _blocks(h) == o["blocks"]
    assert h.exact.tobytes() == o["exact"].tobytes()
    assert h.prefix.tobytes() == o["prefix"].astype(np.uint64).tobytes()
    assert h.centers.tobytes() == o["centers"].astype(h.centers.dtype).tobytes()
    out = pipeline.decode_host(h, b)
    assert out.tobytes() == O.decode(o, b).tobytes()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_stream_compressor_matches_oracle(dtype, depth):
    n, steps, E, bits, bb = 200_003, 5, 1e-3, 8, 1 << 14
    series = workloads.drift_series(n, steps + 1, seed=13, dtype=dtype)
    cfg = pipeline.PipelineConfig(tolerance=E, bits=bits, block_bytes=bb)
    sc = pipeline.StreamCompressor(n, dtype, cfg, depth=depth)
    host = [torch.from_numpy(np.ascontiguousarray(s)).pin_memory() for s in series]
    tickets, got = [], []
    for i in range(steps):
        tickets.append(sc.submit(host[i], host[i + 1]))
        if len(tickets) == depth:      # consume before the slot is reused
            t = tickets.pop(0)
            h, rec = sc.result(t)
            got.append((t, _blocks(h), h.exact.copy(), h.prefix.copy(), rec.copy()))
    for t in tickets:
        h, rec = sc.result(t)
        got.append((t, _blocks(h), h.exact.copy(), h.prefix.copy(), rec.copy()))
    assert [g[0] for g in got] == list(range(steps))
    for t, blocks, exact, prefix, rec in got:
        b, c = series[t], series[t + 1]
        o = O.encode(b, c, E, bits, bb)
        assert blocks == o["blocks"]
        assert exact.tobytes() == o["exact"].tobytes()
        assert prefix.tobytes() == o["prefix"].astype(np.uint64).tobytes()
        assert rec.tobytes() == O.decode(o, b).tobytes()


def test_stream_compressor_requires_bits():
    with pytest.raises(ValueError):
        pipeline.StreamCompressor(1000, np.float64, pipeline.PipelineConfig())


def test_stream_compressor_falls_back_for_wide_spans():
    """A 5e8-bin span cannot use the dense device histogram: the step reruns
    through the sort-based general path and still equals the oracle."""
    b, c = workloads.outlier_pair(60_000, seed=81)
    cfg = pipeline.PipelineConfig(tolerance=1e-3, bits=4, block_bytes=1 << 12)
    sc = pipeline.StreamCompressor(b.size, np.float64, cfg, depth=2)
    hb, hc = torch.from_numpy(b).pin_memory(), torch.from_numpy(c).pin_memory()
    h, rec = sc.result(sc.submit(hb, hc))
    o = O.encode(b, c, 1e-3, 4, 1 << 12)
    assert _blocks(h) == o["blocks"] and h.exact.tobytes() == o["exact"].tobytes()
    assert rec.tobytes() == O.decode(o, b).tobytes()


@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.uint8])
def test_staging_round_trip_sizes(dtype):
    """staging.h2d / d2h (threaded fills of two pinned chunks overlapped with
    their DMA): empty, tiny, chunk-boundary and multi-chunk arrays, contiguous
    or not, arrive and return bit for bit."""
    from paper_1703_02438_b200 import staging
    rng = np.random.default_rng(5)
    item = np.dtype(dtype).itemsize
    per_chunk = staging.CHUNK_BYTES // item
    for n in (0, 1, 1000, per_chunk - 1, per_chunk, per_chunk + 1, 2 * per_chunk + 3):
        a = rng.integers(0, 255, n * item, dtype=np.uint8).view(dtype)
        t = staging.h2d(a)
        assert t.numel() == n and tuple(t.shape) == (n,)
        assert t.cpu().numpy().tobytes() == a.tobytes()
        back = staging.d2h(t)
        assert back.dtype == np.dtype(dtype) and back.tobytes() == a.tobytes()
    strided = rng.normal(size=(1000, 6))[:, ::2].astype(np.float64)   # non-contiguous input is copied first
    t = staging.h2d(strided)
    assert t.cpu().numpy().tobytes() == np.ascontiguousarray(strided).tobytes()
