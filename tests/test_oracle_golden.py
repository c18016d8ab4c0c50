"""Pin the CPU oracle (oracle/nmk_oracle.py) against golden vectors produced
by the reference implementation itself (tests/golden/make_golden.py).

CPU-only: no GPU needed.  If these pass, the oracle is a trustworthy checker
for the CUDA path in the ``-m gpu`` tests.
"""

import numpy as np
import pytest

import nmk_oracle as O
from conftest import golden_bits, golden_blocks, golden_names, load_golden

CASES = golden_names()


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    g = load_golden(name)
    enc = O.encode(g["base"], g["cur"], float(g["E"]), golden_bits(g), int(g["block_bytes"]))
    # phase 1 + 2 intermediates
    if int(g["nvalid"]) == 0:
        assert enc["gmin"] is None
    else:
        assert np.float64(enc["gmin"]).tobytes() == g["gmin"].tobytes()
        assert np.float64(enc["gmax"]).tobytes() == g["gmax"].tobytes()
        keys, counts = enc["hist"]
        np.testing.assert_array_equal(keys, g["hist_keys"])
        np.testing.assert_array_equal(counts, g["hist_counts"])
    # model
    assert enc["bits"] == int(g["bits"])
    assert enc["centers"].astype(g["centers"].dtype).tobytes() == g["centers"].tobytes()
    assert enc["epb"] == int(g["epb"]) and enc["nblocks"] == int(g["nblocks"])
    # outputs
    assert enc["n_inc"] == int(g["n_inc"])
    assert enc["prefix"].tobytes() == g["prefix"].tobytes()
    assert enc["exact"].tobytes() == g["exact"].tobytes()
    assert enc["blocks"] == golden_blocks(g)
    # decode
    full = O.decode(enc, g["base"])
    assert full.tobytes() == g["decoded"].tobytes()
    pos = 0
    for s, c in g["ranges"]:
        part = O.decode(enc, g["base"][s:s + c], rng=(int(s), int(c)))
        assert part.tobytes() == g["range_out"][pos:pos + c].tobytes()
        pos += c


@pytest.mark.parametrize("name", ["series_drift_f32", "series_cfg3_b10"])
def test_oracle_series(name):
    g = load_golden(name)
    snaps = [g[f"snap{i}"] for i in range(int(g["nsteps"]))]
    encs = O.encode_series(snaps, float(g["E"]), golden_bits(g), int(g["block_bytes"]))
    recon = snaps[0]
    for i, e in enumerate(encs, start=1):
        assert e["bits"] == int(g[f"bits{i}"])
        assert e["centers"].astype(snaps[0].dtype).tobytes() == g[f"centers{i}"].tobytes()
        assert b"".join(e["blocks"]) == g[f"packed{i}"].tobytes()
        assert e["exact"].tobytes() == g[f"exact{i}"].tobytes()
        recon = O.decode(e, recon)
        assert recon.tobytes() == g[f"recon{i}"].tobytes()


def test_oracle_workers_invariant():
    g = load_golden("cfg1_blocks")
    a = O.encode(g["base"], g["cur"], 1e-3, 8, 4096, workers=1)
    b = O.encode(g["base"], g["cur"], 1e-3, 8, 4096, workers=5)
    assert a["blocks"] == b["blocks"] and a["exact"].tobytes() == b["exact"].tobytes()


def test_pack_kats():
    # MSB-first, zero padded (codec.py:83-92; reference KATs test_codec.py:20-29)
    assert O.pack(np.array([0xA, 0x5]), 4) == b"\xa5"
    assert O.pack(np.array([7, 7, 7]), 3) == b"\xff\x80"
    assert O.pack(np.arange(256), 8) == bytes(range(256))
    assert list(O.unpack(b"\xff\x80", 3, 3)) == [7, 7, 7]
