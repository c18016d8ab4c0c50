"""pytest plugin (test infrastructure): run the REFERENCE's own hot-path
tests against the B200 drop-in -- SURVEY §8(c) parity level 4.

Loaded with ``-p ref_dropin`` for a pytest session over
oracle/_ref/tests/ (the reference's test files, vendored by
oracle/make_ref.py).  Before the test modules are imported it swaps every
hot-path entry point of the reference package ``nmk`` (oracle/_ref/nmk) for
the drop-in's GPU implementation, the way a deployment would install it:

  nmk.core      compute_change_ratios, ratio_arrays, reconstruct
  nmk.binning   build_histogram, histogram_of, merge_histograms, top_k_bins,
                _coverage_by_bits, select_index_length, incompressible_ratio,
                nearest_center, compressible_mask
  nmk.codec     pack_block, unpack_block, partial_decode, partial_decode_file
  nmk.pipeline  compress_pair, decompress, compress_series

(each also rebound in the ``nmk`` package namespace).  The reference's
exception classes replace the drop-in's (so ``pytest.raises(CodecError)``
sees one class), and the drop-in's lossless stage forwards to the
reference's ``codec.compress_block`` / ``decompress_block`` at call time,
so the tests' fault injection by monkeypatching reaches the drop-in.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
for p in (REF, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

PATCHED: dict[str, list[str]] = {}


def install() -> dict:
    import nmk
    import nmk.binning
    import nmk.codec
    import nmk.container
    import nmk.core
    import nmk.pipeline

    from paper_1703_02438_b200 import binning as ob
    from paper_1703_02438_b200 import codec as oc
    from paper_1703_02438_b200 import container as ocont
    from paper_1703_02438_b200 import core as ocore
    from paper_1703_02438_b200 import pipeline as op

    assert os.path.dirname(nmk.__file__) == os.path.join(REF, "nmk"), nmk.__file__

    # one set of exception classes
    oc.CodecError = nmk.codec.CodecError
    op.PipelineError = nmk.pipeline.PipelineError
    for name in dir(nmk.container):
        obj = getattr(nmk.container, name)
        if isinstance(obj, type) and issubclass(obj, Exception) and hasattr(ocont, name):
            setattr(ocont, name, obj)

    # lossless stage stays the reference's (looked up at call time)
    oc.compress_block = lambda data, level=oc.DEFAULT_DEFLATE_LEVEL: nmk.codec.compress_block(data, level)
    oc.decompress_block = lambda data: nmk.codec.decompress_block(data)

    table = {
        nmk.core: {"compute_change_ratios": ocore.compute_change_ratios, "ratio_arrays": ocore.ratio_arrays,
                   "reconstruct": ocore.reconstruct},
        nmk.binning: {"build_histogram": ob.build_histogram, "histogram_of": ob.histogram_of,
                      "merge_histograms": ob.merge_histograms, "top_k_bins": ob.top_k_bins,
                      "_coverage_by_bits": ob._coverage_by_bits, "select_index_length": ob.select_index_length,
                      "incompressible_ratio": ob.incompressible_ratio, "nearest_center": ob.nearest_center,
                      "compressible_mask": ob.compressible_mask},
        nmk.codec: {"pack_block": oc.pack_block, "unpack_block": oc.unpack_block,
                    "partial_decode": oc.partial_decode, "partial_decode_file": oc.partial_decode_file},
        nmk.pipeline: {"compress_pair": op.compress_pair, "decompress": op.decompress,
                       "compress_series": op.compress_series},
    }
    for mod, attrs in table.items():
        for name, fn in attrs.items():
            assert hasattr(mod, name), f"{mod.__name__}.{name} missing in the reference"
            setattr(mod, name, fn)
            if hasattr(nmk, name):
                setattr(nmk, name, fn)
            PATCHED.setdefault(mod.__name__, []).append(name)
    return PATCHED


def pytest_configure(config):
    install()


def pytest_report_header(config):
    n = sum(len(v) for v in PATCHED.values())
    return f"ref_dropin: {n} reference entry points bound to the B200 drop-in ({REF})"
