"""B200-native NUMARCK hot path (arXiv 1703.02438) behind the reference's
Python API (package `nmk`, pkg/src/nmk/__init__.py).

Phases 1-4a of ``compress_pair`` and the decode chain run as hand-written
sm_100a kernels in ``libnmkgpu.so`` (C ABI: include/nmk_b200.h); the host
side keeps the reference's names, arguments and exceptions.  No CPU
fallback: without the library or a CUDA device the entry points raise
``NativeUnavailable``.
"""

from ._native import NativeError, NativeUnavailable
from .binning import (BinModel, Histogram, build_histogram, compressible_mask, merge_histograms, nearest_center,
                      select_index_length, top_k_bins)
from .codec import (BlockLayout, CodecError, decode_all_indices, pack_block, partial_decode, partial_decode_file,
                    partial_decode_many,
                    unpack_block)
from .container import CompressedVariable, ContainerError, VariableHandle, read_file, scan_file, write_file
from .core import (ChangeRatioField, TemporalPair, Tolerance, compute_change_ratios, ratio_arrays,
                   reconstruct)
from .pipeline import (PhaseTimings, PipelineConfig, PipelineError, compress_pair, compress_series,
                       decompress)

__version__ = "0.1.0"

__all__ = [
    "BinModel", "Histogram", "build_histogram", "compressible_mask", "merge_histograms", "nearest_center",
    "select_index_length", "top_k_bins",
    "BlockLayout", "ChangeRatioField", "CodecError", "CompressedVariable", "ContainerError",
    "NativeError", "NativeUnavailable", "PhaseTimings", "PipelineConfig", "PipelineError",
    "TemporalPair", "Tolerance", "compress_pair", "compress_series", "compute_change_ratios",
    "decode_all_indices", "decompress", "pack_block", "partial_decode", "partial_decode_file", "partial_decode_many", "ratio_arrays",
    "read_file", "reconstruct", "scan_file", "unpack_block", "VariableHandle", "write_file",
]
