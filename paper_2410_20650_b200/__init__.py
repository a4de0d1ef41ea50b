"""B200-native NeuZip bf16 weight codec (arxiv 2410.20650).

The hot path -- bit split/reassembly, lossy mantissa rounding with block
normalisation, chunked rANS exponent encode/decode -- runs as hand-written
sm_100a CUDA kernels in ``libnzgpu.so`` behind the C ABI of
``include/nzgpu.h``.  ``codec`` mirrors the reference's C++ API
(``/root/reference/proj/include/neuzip``) in Python; ``include/neuzip/*.hpp``
mirrors it in C++.  Importing this package loads the CUDA library and fails
loudly if it is missing: there is no CPU fallback.
"""
from . import nzgpu
from .codec import (  # noqa: F401
    Blob,
    ChecksumError,
    DecodePlan,
    EntropyReport,
    DeviceBlob,
    Error,
    FormatError,
    Footprint,
    LosslessBlob,
    LossyBlob,
    NonFiniteError,
    TensorMeta,
    analyze_tensor,
    ans_decode,
    ans_encode,
    build_table,
    component_histogram,
    compress_lossless,
    compress_lossy,
    crc32,
    decompress_batch,
    release_host_buffers,
    decompress_lossless,
    decompress_lossy,
    footprint,
    kChunkSymbols,
    kDefaultBlockSize,
    kLosslessPrecision,
    lossy_roundtrip,
    pack_signed_mantissas,
    ratio,
    read_nzt,
    unpack_signed_mantissas,
    write_nzt,
)

LIB_PATH = nzgpu.LIB_PATH
__all__ = [n for n in dir() if not n.startswith("_")]
