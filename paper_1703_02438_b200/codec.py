"""Block codec surface (mirror of nmk.codec, pkg/src/nmk/codec.py).

* Block geometry (`BlockLayout`) is plain integer arithmetic, as in the
  reference (codec.py:28-59).
* Bit packing / unpacking and range decoding run on the GPU (K4/K5 and the
  standalone nmk_pack / nmk_unpack kernels).
* The lossless per-block DEFLATE stage: `compress_block` / `decompress_block`
  are the reference's host-zlib functions (the same raw RFC 1951 stream at
  the same level, codec.py:108-128), looked up through this module's
  attributes so fault injection by monkeypatching still works; compress_pair
  deflates with them by default (byte-identical .nmk files).  The decode
  path inflates on the GPU instead (k_inflate.cu, any raw DEFLATE stream:
  zlib's or the optional GPU deflate's), so a decode ships only compressed
  bytes to the device and never runs host zlib.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass

import numpy as np

from . import _native as N

DEFAULT_BLOCK_BYTES = 1 << 20
DEFAULT_DEFLATE_LEVEL = 6
MIN_BLOCK_BYTES = 4096


class CodecError(Exception):
    """Packing or lossless-backend failure (codec.py:24-25)."""


@dataclass(frozen=True)
class BlockLayout:
    """Partition of an n-element index stream into byte-capacity blocks."""

    block_bytes: int
    bits: int
    n: int

    def __post_init__(self) -> None:
        if self.elements_per_block < 1:
            raise ValueError("block capacity below one element")

    @property
    def elements_per_block(self) -> int:
        return (self.block_bytes * 8) // self.bits

    @property
    def nblocks(self) -> int:
        return -(-self.n // self.elements_per_block)

    def block_range(self, ordinal: int) -> tuple[int, int]:
        epb = self.elements_per_block
        start = ordinal * epb
        return start, min(start + epb, self.n)

    def covering_blocks(self, start: int, count: int) -> range:
        if count <= 0:
            return range(0)
        epb = self.elements_per_block
        return range(start // epb, (start + count - 1) // epb + 1)


def packed_size(element_count: int, bits: int) -> int:
    return (element_count * bits + 7) // 8


# ---------------------------------------------------------------------------
# GPU bit packing (codec.py:83-105)
# ---------------------------------------------------------------------------

def pack_block(indices, bits: int) -> bytes:
    """MSB-first B-bit packing, zero-padded to a byte, on the GPU."""
    import torch
    idx = np.asarray(indices)
    if idx.size == 0:
        return b""
    if idx.min() < 0 or int(idx.max()) >= (1 << bits):
        raise CodecError(f"index out of range for {bits}-bit packing")
    N.require_cuda()
    n = idx.size
    codes = torch.from_numpy(idx.astype(np.uint32).view(np.int32)).cuda()
    out = torch.empty(packed_size(n, bits), dtype=torch.uint8, device=codes.device)
    N.check(N.lib().nmk_pack(codes.data_ptr(), n, bits, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return out.cpu().numpy().tobytes()


def unpack_block(data: bytes, bits: int, element_count: int) -> np.ndarray:
    """Exact inverse of :func:`pack_block` on the GPU; pad bits ignored."""
    import torch
    expected = packed_size(element_count, bits)
    if len(data) < expected:
        raise CodecError(f"short buffer: {len(data)} bytes, need {expected}")
    if element_count == 0:
        return np.zeros(0, dtype=np.int32)
    N.require_cuda()
    raw = torch.from_numpy(np.frombuffer(data, dtype=np.uint8, count=expected).copy()).cuda()
    codes = torch.empty(element_count, dtype=torch.int32, device=raw.device)
    N.check(N.lib().nmk_unpack(raw.data_ptr(), element_count, bits, codes.data_ptr(),
                               torch.cuda.current_stream().cuda_stream))
    return codes.cpu().numpy()


# ---------------------------------------------------------------------------
# Lossless stage (outside the accelerated path; host zlib, codec.py:108-128)
# ---------------------------------------------------------------------------

def compress_block(packed: bytes, level: int = DEFAULT_DEFLATE_LEVEL) -> bytes:
    """Deflate one packed block as a raw RFC 1951 stream (no zlib wrapper)."""
    if not 0 <= level <= 9:
        raise CodecError(f"deflate level {level} outside 0..9")
    try:
        c = zlib.compressobj(level, zlib.DEFLATED, -zlib.MAX_WBITS)
        return c.compress(packed) + c.flush()
    except zlib.error as exc:  # pragma: no cover
        raise CodecError(f"deflate failed: {exc}") from exc


def deflate_segment_bytes(total_bytes: int) -> int:
    """Segment size of the GPU deflate stage: the largest of 16 KiB / 32 KiB /
    65 520 bytes that still leaves >= 2048 segments (one warp each: enough to
    fill a B200).  Larger segments carry fewer Huffman headers (cfg2: ratio
    6.21 -> 6.33, and 13 ms less to inflate) but each is one warp's serial work."""
    for seg in (65520, 32768):
        if total_bytes // seg >= 2048:
            return seg
    return 16384


def gpu_deflate_blocks(packed_dev, stride: int, lengths, seg_bytes: int | None = None) -> list[bytes]:
    """Raw DEFLATE of every packed block on the GPU (k_deflate.cu): block b
    is ``packed_dev[b*stride : b*stride + lengths[b]]`` (all blocks but the
    last have equal length).  Inflates (zlib or any inflater) to the packed
    bytes; not byte-equal to zlib's stream (opt-in: PipelineConfig.deflate).
    ``seg_bytes`` (a multiple of 16 in [64, 65535]) defaults to
    :func:`deflate_segment_bytes` of the total size."""
    import torch
    from . import engine
    lengths = [int(x) for x in lengths]
    nb = len(lengths)
    if nb == 0:
        return []
    if any(x != lengths[0] for x in lengths[:-1]) or lengths[-1] > lengths[0] or lengths[-1] < 1:
        raise CodecError("gpu deflate: blocks must share one length (the last may be shorter)")
    if seg_bytes is None:
        seg_bytes = deflate_segment_bytes(sum(lengths))
    lib = N.lib()
    dev = packed_dev.device
    ws_bytes = lib.nmk_deflate_ws_bytes(nb, lengths[0], seg_bytes)
    bound = lib.nmk_deflate_bound(nb, lengths[0], seg_bytes)
    if not ws_bytes or not bound:
        raise CodecError(f"gpu deflate: unsupported segment size {seg_bytes}")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    out = torch.empty(bound, dtype=torch.uint8, device=dev)
    off = torch.empty(nb + 1, dtype=torch.int64, device=dev)
    N.check(lib.nmk_deflate(packed_dev.data_ptr(), stride, nb, lengths[0], lengths[-1], seg_bytes, out.data_ptr(),
                            off.data_ptr(), ws.data_ptr(), ws_bytes, torch.cuda.current_stream().cuda_stream))
    o = off.cpu().numpy()
    data = out[: int(o[-1])].cpu().numpy().tobytes()
    return [data[int(o[b]): int(o[b + 1])] for b in range(nb)]


_INFLATE_ERRORS = {
    1: "inflate failed: invalid block type",
    2: "inflate failed: invalid stored block lengths",
    3: "inflate failed: invalid dynamic block header",
    4: "inflate failed: invalid code",
    5: "inflate failed: invalid distance",
    6: "corrupt block: truncated or trailing bytes",
    7: "corrupt block: truncated or trailing bytes",
    8: "inflate failed: block inflates past its packed size",
}


def gpu_inflate_blocks(blobs, out_stride: int, device=None, slots=None, nslots: int | None = None,
                       defer: bool = False):
    """Inflate raw DEFLATE streams on the GPU (k_inflate.cu), the decode half
    of the lossless stage (codec.py:119-128): stream i lands at
    ``out[j*out_stride : j*out_stride + produced[i]]`` of the returned device
    buffer, j = slots[i] (default i) of ``nslots`` slots -- the strided
    packed-block layout K5 reads.  Returns ``(out, produced)``; a stream that
    zlib would reject raises CodecError (truncated or trailing bytes with the
    reference's message).  ``defer=True`` returns a function that waits for
    the kernel and yields that pair, so the caller can do host work (e.g. the
    upload of the base snapshot) while the streams inflate."""
    import torch
    N.require_cuda()
    blobs = [bytes(b) for b in blobs]
    nb = len(blobs)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    total_slots = nslots if nslots is not None else nb
    out = torch.zeros(max(total_slots * out_stride, 1), dtype=torch.uint8, device=dev)
    if nb == 0:
        res = (out, np.zeros(0, dtype=np.int64))
        return (lambda: res) if defer else res
    d_slot = None
    if slots is not None:
        d_slot = torch.from_numpy(np.asarray(slots, dtype=np.int64) * out_stride).to(dev)
    off = np.zeros(nb + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(b) for b in blobs])
    comp = np.frombuffer(b"".join(blobs) + bytes(16), dtype=np.uint8)   # k_inflate reads 8-byte words: pad
    d_comp = torch.from_numpy(comp.copy()).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    status = torch.empty(nb, dtype=torch.int32, device=dev)
    produced = torch.empty(nb, dtype=torch.int64, device=dev)
    N.check(N.lib().nmk_inflate(d_comp.data_ptr(), d_off.data_ptr(), nb, out.data_ptr(), out_stride,
                                d_slot.data_ptr() if d_slot is not None else None, status.data_ptr(),
                                produced.data_ptr(), torch.cuda.current_stream().cuda_stream))
    def finish():
        st = status.cpu().numpy()
        bad = np.flatnonzero(st)
        if bad.size:
            raise CodecError(_INFLATE_ERRORS.get(int(st[bad[0]]), "inflate failed"))
        _ = d_comp, d_off, d_slot   # inputs stay alive until the kernel is done
        return out, produced.cpu().numpy()

    return finish if defer else finish()


def gpu_decompress_block(data: bytes, capacity: int | None = None) -> bytes:
    """:func:`decompress_block` on the GPU (one stream).  ``capacity`` bounds
    the inflated size (default: 1032x the input, DEFLATE's maximum ratio)."""
    cap = capacity if capacity is not None else max(1032 * len(data) + 64, 64)
    cap = (cap + 15) // 16 * 16
    out, produced = gpu_inflate_blocks([data], cap)
    return out[: int(produced[0])].cpu().numpy().tobytes()


def decompress_block(data: bytes) -> bytes:
    """Inflate one raw deflate stream produced by :func:`compress_block`."""
    try:
        d = zlib.decompressobj(-zlib.MAX_WBITS)
        out = d.decompress(data) + d.flush()
    except zlib.error as exc:
        raise CodecError(f"inflate failed: {exc}") from exc
    if not d.eof or d.unused_data:
        raise CodecError("corrupt block: truncated or trailing bytes")
    return out


# ---------------------------------------------------------------------------
# Range decode on the GPU (codec.py:181-258)
# ---------------------------------------------------------------------------

def _block_bytes_of(variable, ordinal: int) -> bytes:
    offsets = variable.index_offsets
    lo = int(offsets[ordinal])
    hi = int(offsets[ordinal + 1]) if ordinal + 1 < len(offsets) else len(variable.index_table)
    return variable.index_table[lo:hi]


def _inflate_covering(compressed, first, bits, epb, n, defer: bool = False):
    """The covering blocks' DEFLATE streams inflated on the GPU straight into
    the strided packed layout K5 reads (k_inflate.cu): only compressed bytes
    cross PCIe.  A block that inflates to fewer bytes than its element count
    needs fails as unpack_block would (codec.py:97-99).  ``defer=True``: the
    kernel is launched and a function returning the buffer (after the checks)
    comes back."""
    from . import engine
    stride = engine.block_stride(epb, bits)
    pending = gpu_inflate_blocks(compressed, stride, defer=True)

    def finish():
        d_packed, produced = pending()
        for i in range(len(compressed)):
            s, e = (first + i) * epb, min((first + i + 1) * epb, n)
            need_b = packed_size(e - s, bits)
            if int(produced[i]) < need_b:
                raise CodecError(f"short buffer: {int(produced[i])} bytes, need {need_b}")
        return d_packed

    return finish if defer else finish()


def _gpu_decode_blocks(blocks, bits, epb, n, prefix, centers64, exact, exact_offset, start, count, base,
                       d_base=None):
    """Decode [start, start+count) of the covering block ordinals first..last
    on the GPU.  ``blocks``: the blocks' packed bytes (a list of host byte
    strings) or a device buffer already in the strided layout
    (_inflate_covering).

    ``prefix`` = incompressible_prefix (global), ``exact`` = the exact values
    from global index ``exact_offset`` on.  Returns
    (out, need, have, bad_index, max_bad_index) with need/have the sentinel
    count inside the range and the exact values available for it."""
    import torch
    from . import engine
    N.require_cuda()
    first = start // epb
    stride = engine.block_stride(epb, bits)
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(blocks, (list, tuple)):
        nb = len(blocks)
        host = np.zeros(nb * stride, dtype=np.uint8)
        for i, blk in enumerate(blocks):
            s, e = (first + i) * epb, min((first + i + 1) * epb, n)
            need_b = packed_size(e - s, bits)
            if len(blk) < need_b:
                raise CodecError(f"short buffer: {len(blk)} bytes, need {need_b}")
            host[i * stride: i * stride + need_b] = np.frombuffer(blk, dtype=np.uint8, count=need_b)
        d_packed = torch.from_numpy(host).to(dev)
    else:
        d_packed = blocks
        nb = (start + count - 1) // epb - first + 1
    pre = np.asarray(prefix, dtype=np.uint64)[first:first + nb].astype(np.int64)
    base_inc = int(pre[0])
    d_prefix_rel = torch.from_numpy(pre - base_inc).to(dev)
    d_centers = torch.tensor(np.asarray(centers64, dtype=np.float64), device=dev)   # copies (read-only ok)
    from . import staging
    ex = np.asarray(exact)[max(base_inc - exact_offset, 0):]   # covering blocks only
    if base_inc < exact_offset:
        raise ValueError("exact values start after the covering block")
    d_exact = staging.h2d(ex, dev) if ex.size else torch.empty(0, dtype=_tdt(base.dtype), device=dev)
    if d_base is None:
        d_base = staging.h2d(np.asarray(base), dev)
    res = engine.decode(d_packed, stride, first, bits, epb, n, d_prefix_rel, d_centers, d_exact, d_base,
                        [(start, count, 0)])
    need = int(res.n_sentinel[0])
    avail = ex.shape[0] - int(res.inc_before[0])
    have = max(0, min(need, avail))
    return staging.d2h(res.out), need, have, res.bad_index, res.max_bad_index


def _tdt(np_dtype):
    import torch
    return torch.float64 if np.dtype(np_dtype).itemsize == 8 else torch.float32


_side_streams: dict = {}


def _upload_stream():
    """A per-device side stream for uploads that overlap a kernel on the current stream."""
    import torch
    dev = torch.cuda.current_device()
    if dev not in _side_streams:
        _side_streams[dev] = torch.cuda.Stream()
    return _side_streams[dev]


def _decode_range(variable, start, count, base, block_bytes, inc_slice_all) -> np.ndarray:
    """Shared range decoder (codec.py:204-239): validation, GPU inflate of the
    covering blocks, then one K5 launch (no host zlib on the decode path)."""
    if start < 0 or count < 0 or start + count > variable.n:
        raise ValueError(f"range [{start}, {start + count}) outside 0..{variable.n}")
    base = np.asarray(base)
    if base.shape[0] != count:
        raise ValueError(f"base slice holds {base.shape[0]} elements, need {count}")
    if count == 0:
        return np.zeros(0, dtype=variable.numpy_dtype)
    epb = variable.elements_per_block
    first = start // epb
    last = (start + count - 1) // epb
    from . import staging
    inflating = _inflate_covering([block_bytes(b) for b in range(first, last + 1)], first, variable.bits, epb,
                                  variable.n, defer=True)
    import torch
    cur_stream = torch.cuda.current_stream()
    side = _upload_stream()
    with torch.cuda.stream(side):  # the host fills and the DMA run while the streams inflate
        d_base = staging.h2d(base)
        uploaded = torch.cuda.Event()
        uploaded.record(side)
    d_base.record_stream(cur_stream)
    blocks = inflating()
    cur_stream.wait_event(uploaded)
    inc_lo = int(variable.incompressible_prefix[first])
    exact, exact_offset = inc_slice_all(inc_lo)
    exact = np.asarray(exact)
    if exact.dtype != base.dtype:
        exact = exact.astype(base.dtype)   # core.py:207 (astype to the base dtype)
    centers = variable.centers.astype(np.float64, copy=False)
    out, need, have, bad, maxbad = _gpu_decode_blocks(
        blocks, variable.bits, epb, variable.n, variable.incompressible_prefix, centers, exact,
        exact_offset, start, count, base, d_base=d_base)
    if bad:
        raise ValueError(f"index {maxbad} out of range for {len(centers)} centers")
    if have < need:
        raise ValueError(f"incompressible values exhausted: need {need}, have {have}")
    return out


def partial_decode(variable, start: int, count: int, base_reconstructed) -> np.ndarray:
    """Reconstruct ``[start, start + count)`` touching only the covering
    blocks (codec.py:242-258); bit-identical to a full-decode slice."""
    epb = variable.elements_per_block

    def inc_slice(lo: int):
        # only the exact values of the covering blocks travel to the device
        last = (start + count - 1) // epb if count else start // epb
        hi = int(variable.incompressible_prefix[last + 1]) if last + 1 < variable.nblocks \
            else variable.n_incompressible
        return variable.incompressible_table[lo:max(hi, lo)], lo

    return _decode_range(variable, start, count, base_reconstructed,
                         lambda b: _block_bytes_of(variable, b), inc_slice)


def partial_decode_many(variable, ranges, bases) -> list:
    """Batched :func:`partial_decode`: ``ranges`` = [(start, count), ...],
    ``bases[i]`` the base slice of range i.  Every covering block is inflated
    once on the GPU (k_inflate.cu) and ALL ranges decode in one K5 launch.
    Results equal ``partial_decode`` range by range (codec.py:242-258),
    including its errors."""
    import torch
    from . import engine
    ranges = [(int(a), int(c)) for a, c in ranges]
    if len(bases) != len(ranges):
        raise ValueError("one base slice per range")
    out = [None] * len(ranges)
    live = []
    for i, (a, c) in enumerate(ranges):
        if a < 0 or c < 0 or a + c > variable.n:
            raise ValueError(f"range [{a}, {a + c}) outside 0..{variable.n}")
        if np.asarray(bases[i]).shape[0] != c:
            raise ValueError(f"base slice holds {np.asarray(bases[i]).shape[0]} elements, need {c}")
        if c == 0:
            out[i] = np.zeros(0, dtype=variable.numpy_dtype)
        else:
            live.append(i)
    if not live:
        return out
    epb, bits, n = variable.elements_per_block, variable.bits, variable.n
    need = sorted({b for i in live for b in range(ranges[i][0] // epb, (ranges[i][0] + ranges[i][1] - 1) // epb + 1)})
    first, last = need[0], need[-1]
    stride = engine.block_stride(epb, bits)
    d_packed, produced = gpu_inflate_blocks([_block_bytes_of(variable, b) for b in need], stride,
                                            slots=[b - first for b in need], nslots=last - first + 1)
    for i, b in enumerate(need):
        s_, e_ = b * epb, min((b + 1) * epb, n)
        nb = packed_size(e_ - s_, bits)
        if int(produced[i]) < nb:
            raise CodecError(f"short buffer: {int(produced[i])} bytes, need {nb}")
    prefix = np.asarray(variable.incompressible_prefix, dtype=np.uint64)
    lo = int(prefix[first])
    hi = int(prefix[last + 1]) if last + 1 < variable.nblocks else int(variable.n_incompressible)
    dt = variable.numpy_dtype
    exact = np.array(variable.incompressible_table[lo:max(hi, lo)], dtype=dt, copy=True)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_prefix = torch.from_numpy(prefix[first:last + 1].astype(np.int64) - lo).to(dev)
    d_centers = torch.tensor(np.asarray(variable.centers, dtype=np.float64), device=dev)
    d_exact = torch.from_numpy(exact).to(dev) if exact.size else torch.empty(0, dtype=_tdt(dt), device=dev)
    offs = np.zeros(len(live) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([ranges[i][1] for i in live])
    base_all = np.concatenate([np.asarray(bases[i], dtype=dt) for i in live])
    d_base = torch.from_numpy(base_all).to(dev)
    segs = [(ranges[i][0], ranges[i][1], int(offs[j])) for j, i in enumerate(live)]
    res = engine.decode(d_packed, stride, first, bits, epb, n, d_prefix, d_centers, d_exact, d_base, segs)
    if res.bad_index:
        raise ValueError(f"index {res.max_bad_index} out of range for {len(variable.centers)} centers")
    avail = exact.shape[0] - res.inc_before
    if (res.n_sentinel > np.maximum(avail, 0)).any():
        j = int(np.flatnonzero(res.n_sentinel > np.maximum(avail, 0))[0])
        raise ValueError(f"incompressible values exhausted: need {int(res.n_sentinel[j])}, have {max(int(avail[j]), 0)}")
    flat = res.out.cpu().numpy()
    for j, i in enumerate(live):
        out[i] = flat[offs[j]:offs[j + 1]].copy()
    return out


def partial_decode_file(handle, start: int, count: int, base_reconstructed) -> np.ndarray:
    """Like ``partial_decode`` straight from an on-disk variable
    (codec.py:261-278): only the covering blocks' DEFLATE bytes and the exact
    values those blocks reference are read from the file."""
    variable = handle.variable
    offsets = variable.index_offsets
    epb = variable.elements_per_block

    def block_bytes(b: int) -> bytes:
        lo = int(offsets[b])
        hi = int(offsets[b + 1]) if b + 1 < len(offsets) else handle.index_table_len
        return handle.read_index_range(lo, hi)

    def inc_slice(lo: int):
        last = (start + count - 1) // epb if count else start // epb
        hi = int(variable.incompressible_prefix[last + 1]) if last + 1 < variable.nblocks \
            else variable.n_incompressible
        return handle.read_incompressible_range(lo, max(hi - lo, 0)), lo

    return _decode_range(variable, start, count, base_reconstructed, block_bytes, inc_slice)


def decode_block_indices(variable, ordinal: int) -> np.ndarray:
    start = ordinal * variable.elements_per_block
    stop = min(start + variable.elements_per_block, variable.n)
    packed = gpu_decompress_block(_block_bytes_of(variable, ordinal),
                                  capacity=packed_size(variable.elements_per_block, variable.bits) + 16)
    return unpack_block(packed, variable.bits, stop - start)


def decode_all_indices(variable) -> np.ndarray:
    """Full index stream (sentinels included), unpacked on the GPU."""
    parts = [decode_block_indices(variable, b) for b in range(variable.nblocks)]
    if not parts:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate(parts)
