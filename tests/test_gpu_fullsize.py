"""BASELINE configs 3, 4 (weak, one GPU's share) and 5 at their full sizes,
checked through size-independent properties (the oracle would take minutes
at these sizes; it pins the same kernels at reduced sizes elsewhere):

* decode(encode(x)) reproduces the incompressible elements bit for bit and
  every other element within E * |base|;
* the exact-value list is the element-order compaction of the sentinels;
* the prefix table is the exclusive scan of sentinels per block;
* the sync-free pipeline and the general path emit the same bytes;
* 1000 partial segments equal the matching slices of the full decode.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import _native as N, engine, workloads  # noqa: E402


def _codes(enc):
    codes = torch.empty(enc.n, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for b in range(enc.nblocks):
        s, e = b * enc.epb, min((b + 1) * enc.epb, enc.n)
        N.check(N.lib().nmk_unpack(enc.packed.data_ptr() + b * enc.stride, e - s, enc.bits,
                                   codes.data_ptr() + 4 * s, st))
    return codes


def _bits(t):
    return t.view(torch.int64) if t.dtype == torch.float64 else t.view(torch.int32)


def _check_properties(enc, base, cur, out, E):
    codes = _codes(enc)
    sent = codes == (1 << enc.bits) - 1
    assert int(sent.sum()) == enc.n_inc
    assert int(codes[~sent].max()) < enc.k if bool((~sent).any()) else True
    assert torch.equal(_bits(out[sent]), _bits(cur[sent]))
    assert torch.equal(_bits(enc.exact), _bits(cur[sent]))
    comp = ~sent
    err = (out[comp].double() - cur[comp].double()).abs()
    assert bool((err <= E * base[comp].double().abs()).all())
    nb = enc.nblocks
    per = torch.zeros(nb, dtype=torch.int64, device="cuda")
    per.index_add_(0, torch.arange(enc.n, device="cuda") // enc.epb, sent.long())
    pre = torch.zeros_like(per)
    pre[1:] = torch.cumsum(per, 0)[:-1]
    assert torch.equal(enc.prefix.view(torch.int64), pre)
    c = enc.centers.cpu().numpy()
    assert c.size == enc.k <= (1 << enc.bits) - 1 and (np.diff(c) > 0).all()


def _same_bytes(a, b):
    """Same model, same valid packed bytes per block (the stride padding after
    a short last block is not part of the stream), same exact list / prefix."""
    assert a.bits == b.bits and a.k == b.k and a.n_inc == b.n_inc and a.stride == b.stride
    for i, ln in enumerate(a.block_lengths()):
        o = i * a.stride
        assert torch.equal(a.packed[o: o + int(ln)], b.packed[o: o + int(ln)]), i
    assert torch.equal(_bits(a.exact), _bits(b.exact))
    assert torch.equal(a.prefix, b.prefix)
    assert torch.equal(a.centers, b.centers)


def test_cfg3_series_full_size():
    """1440 x 720 x 30 fp32, 16 steps, E = 5e-3, B = 10: each transition is
    encoded against the previous reconstruction, on the device."""
    E, bits = 5e-3, 10
    x = workloads.cfg3_device_first(seed=0)
    n = x.numel()
    assert n == 31_104_000
    pipe = engine.DevicePipeline(n, torch.float32, E, bits)
    recon = x.clone()
    out = torch.empty_like(x)
    for t in range(1, 16):
        x = workloads.cfg3_device_step(x, t, seed=0)
        pipe.step(recon, x, out)
        chk = pipe.check()
        assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
        enc = pipe.encoding()
        _check_properties(enc, recon, x, out, E)
        if t in (1, 15):   # the general path agrees byte for byte
            ref = engine.encode(recon, x, E, bits)
            _same_bytes(enc, ref)
            assert torch.equal(_bits(engine.decode_encoding(ref, recon).out), _bits(out))
        recon, out = out, recon


def test_cfg4_weak_share_full_size():
    """One GPU's weak-scaling share: 2^29 fp64 with config 1's distribution."""
    base, cur = workloads.cfg1_device(1 << 29, seed=4)
    pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 8)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
    assert chk["n_sentinel"] == chk["n_inc"]
    _check_properties(pipe.encoding(), base, cur, out, 1e-3)


@pytest.mark.parametrize("bits,E", [(8, 1e-2), (10, 1e-3), (12, 1e-4)])
def test_cfg5_full_size(bits, E):
    """2^28 fp64 bimodal + 20 % outliers: full decode, then 1000 random 2^16
    segments in one launch equal the slices of the full decode."""
    base, cur = workloads.cfg5_device(1 << 28, seed=5)
    enc = engine.encode(base, cur, E, bits)
    res = engine.decode_encoding(enc, base)
    assert not res.bad_index and not res.exhausted
    _check_properties(enc, base, cur, res.out, E)
    pipe = engine.DevicePipeline(base.numel(), base.dtype, E, bits)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    if pipe.check()["status"] == 0:   # dense span: the sync-free path must agree
        _same_bytes(pipe.encoding(), enc)
        assert torch.equal(_bits(out), _bits(res.out))
    rng = np.random.default_rng(bits)
    starts = rng.integers(0, enc.n - (1 << 16), 1000)
    segs = [(int(s), 1 << 16, i << 16) for i, s in enumerate(starts)]
    idx = torch.from_numpy(np.concatenate([np.arange(s, s + (1 << 16)) for s, _, _ in segs])).cuda()
    part = engine.decode(enc.packed, enc.stride, 0, enc.bits, enc.epb, enc.n, enc.prefix, enc.centers, enc.exact,
                         base[idx], segs)
    assert not part.bad_index and not part.exhausted
    assert torch.equal(_bits(part.out), _bits(res.out[idx]))
    sent_total = int(part.n_sentinel.sum())
    codes = _codes(enc)[idx]
    assert sent_total == int((codes == (1 << bits) - 1).sum())
