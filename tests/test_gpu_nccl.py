"""The multi-GPU code path over real NCCL on the one GPU a box has: a world
of one rank drives every exchange (device all-reduces, all-gathers, the
exclusive scan) through NCCL and must reproduce the single-process bytes.
(Larger worlds are covered by the gloo tests and the emulated shards.)"""

import socket

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_1703_02438_b200 import distributed as D, engine, workloads  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def nccl_world1():
    if dist.is_initialized():  # pragma: no cover
        pytest.skip("a process group is already initialised")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield D.ProcessGroupComm()
    dist.destroy_process_group()


def _blocks(enc):
    nlb = enc.prefix.numel()
    packed = enc.packed[: nlb * enc.stride].cpu().numpy()
    lens = enc.block_lengths()
    return [packed[i * enc.stride: i * enc.stride + int(lens[i])].tobytes() for i in range(nlb)]


@pytest.mark.parametrize("case", ["cfg1", "cfg2"])
def test_device_pipeline_over_nccl(nccl_world1, case):
    if case == "cfg1":
        b, c = workloads.cfg1_host(1 << 19, seed=41); E, bits, bb = 1e-3, 8, 1 << 16
    else:
        b, c = workloads.cfg2_host(64, seed=42); E, bits, bb = 1e-3, 8, 1 << 15
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    ref = engine.DevicePipeline(base.numel(), base.dtype, E, bits, bb)
    out_ref = torch.empty_like(base)
    ref.step(base, cur, out_ref)
    pipe = engine.DevicePipeline(base.numel(), base.dtype, E, bits, bb, elem0=0, n_total=base.numel(),
                                 comm=nccl_world1)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and chk["n_inc"] == ref.check()["n_inc"]
    e1, e0 = pipe.encoding(), ref.encoding()
    assert _blocks(e1) == _blocks(e0)
    assert e1.exact.cpu().numpy().tobytes() == e0.exact.cpu().numpy().tobytes()
    assert out.cpu().numpy().tobytes() == out_ref.cpu().numpy().tobytes()
    o = O.encode(b, c, E, bits, bb)
    assert _blocks(e1) == o["blocks"]


def test_general_encode_over_nccl(nccl_world1):
    b, c = workloads.cfg5_host(200_003, seed=43)
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    enc = engine.encode(base, cur, 1e-3, 10, 1 << 14, elem0=0, n_total=base.numel(), comm=nccl_world1)
    part = D.rank_part_from_encoding(enc)
    blocks, exact, prefix, n_inc = D.merge_parts([part], base.numel(), enc.epb, enc.bits)
    o = O.encode(b, c, 1e-3, 10, 1 << 14)
    assert n_inc == o["n_inc"] and blocks == o["blocks"]
    assert exact.tobytes() == o["exact"].tobytes()
    assert prefix.tobytes() == np.asarray(o["prefix"], dtype=np.uint64).tobytes()


def test_device_pipeline_graph_with_nccl_exchanges(nccl_world1):
    """The bench captures the multi-GPU step (kernels + NCCL exchanges) as one
    CUDA graph: replays must equal the eager step."""
    b, c = workloads.cfg1_host(1 << 18, seed=44)
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 8, 1 << 15, elem0=0, n_total=base.numel(),
                                 comm=nccl_world1)
    out_e = torch.empty_like(base)
    pipe.step(base, cur, out_e)
    ref_blocks = _blocks(pipe.encoding())
    out_g = torch.empty_like(base)
    g = pipe.capture(base, cur, out_g)
    out_g.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert pipe.check()["status"] == 0
    assert _blocks(pipe.encoding()) == ref_blocks
    assert out_g.cpu().numpy().tobytes() == out_e.cpu().numpy().tobytes()
