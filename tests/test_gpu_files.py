"""On-disk partial decompression (codec.partial_decode_file over
container.scan_file handles, codec.py:261-278 / container.py:273-347): equal
to the slice of a full decompress and to the oracle, reading only the
covering blocks and the exact values they reference."""

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import codec, container, pipeline, workloads  # noqa: E402
from paper_1703_02438_b200.core import TemporalPair  # noqa: E402


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_partial_decode_file_matches_full_and_oracle(tmp_path, dtype):
    b, c = workloads.cfg5_host(300_007, seed=61)
    b, c = b.astype(dtype), c.astype(dtype)
    cfg = pipeline.PipelineConfig(tolerance=1e-3, bits=10, block_bytes=1 << 14)
    var, _ = pipeline.compress_pair(TemporalPair(b, c), cfg, name="t")
    other, _ = pipeline.compress_pair(TemporalPair(c, b), cfg, name="u")
    path = tmp_path / "pair.nmk"
    container.write_file(path, [other, var])
    handles = {h.variable.name: h for h in container.scan_file(path)}
    h = handles["t"]
    full = pipeline.decompress(var, b)
    o = O.encode(b, c, 1e-3, 10, 1 << 14)
    ref = O.decode(o, b)
    assert full.tobytes() == ref.tobytes()
    epb = var.elements_per_block
    reads = {"index": 0, "exact": 0}
    real_idx, real_inc = h.read_index_range, h.read_incompressible_range

    def count_idx(lo, hi):
        reads["index"] += hi - lo
        return real_idx(lo, hi)

    def count_inc(start, count):
        reads["exact"] += count
        return real_inc(start, count)

    h.read_index_range, h.read_incompressible_range = count_idx, count_inc
    for start, count in [(0, 1), (0, epb), (epb - 3, 7), (5 * epb + 11, 3 * epb), (var.n - 1, 1),
                         (var.n - 2 * epb - 5, 2 * epb + 5), (123, 0)]:
        reads["index"] = reads["exact"] = 0
        got = codec.partial_decode_file(h, start, count, b[start:start + count])
        assert got.tobytes() == full[start:start + count].tobytes()
        assert got.tobytes() == codec.partial_decode(var, start, count, b[start:start + count]).tobytes()
        if count:
            first, last = start // epb, (start + count - 1) // epb
            offs = var.index_offsets.astype(np.int64)
            hi = int(offs[last + 1]) if last + 1 < var.nblocks else len(var.index_table)
            assert reads["index"] == hi - int(offs[first])
            pre = var.incompressible_prefix.astype(np.int64)
            inc_hi = int(pre[last + 1]) if last + 1 < var.nblocks else var.n_incompressible
            assert reads["exact"] == inc_hi - int(pre[first])
    with pytest.raises(ValueError):
        codec.partial_decode_file(h, var.n - 1, 2, b[-1:])
