"""ctypes binding of the C ABI in include/nzgpu.h (libnzgpu.so).

This is the Python host side of the product: it loads the in-tree
``libnzgpu.so`` and nothing else.  There is no CPU fallback -- if the library
is missing the import fails, and if no GPU is present every data-path call
raises ``NoDeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# NZGPU_LIB may select an in-tree tuning variant (e.g. libnzgpu_ch4.so).
LIB_PATH = os.path.join(HERE, os.path.basename(os.environ.get("NZGPU_LIB", "libnzgpu.so")))

OK, INVALID_ARGUMENT, FORMAT_TRUNCATED, FORMAT_DESYNC, FORMAT_LENGTH = 0, 1, 2, 3, 4
NONFINITE, FORMAT_TABLE, CUDA_ERROR, OUT_OF_MEMORY, NO_DEVICE = 5, 6, 7, 8, 9
CHECKSUM = 10
LOSSLESS = 7
DEFAULT_BLOCK = 512
DEFAULT_CHUNK = 65536
DEFAULT_INTERVAL = 64


# --- exception taxonomy of the reference (errors.hpp:9-32) ----------------
class Error(RuntimeError):
    """neuzip::Error"""


class FormatError(Error):
    """neuzip::FormatError: truncation, desync, length mismatch, bad table."""


class ChecksumError(FormatError):
    """neuzip::ChecksumError"""


class NonFiniteError(Error):
    """neuzip::NonFiniteError"""


class NoDeviceError(Error):
    """No CUDA device: the codec never falls back to the CPU."""


class CudaError(Error):
    pass


def _raise(rc: int, what: str) -> None:
    if rc == OK:
        return
    msg = f"{what}: {lib.nzgpu_status_string(rc).decode()}"
    detail = lib.nzgpu_last_error_message().decode()
    if rc in (CUDA_ERROR, OUT_OF_MEMORY) and detail:
        msg += f" ({detail})"
    if rc == INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc in (FORMAT_TRUNCATED, FORMAT_DESYNC, FORMAT_LENGTH, FORMAT_TABLE):
        err = FormatError(msg)
        err.status = rc
        raise err
    if rc == CHECKSUM:
        err = ChecksumError(msg)
        err.status = rc
        raise err
    if rc == NONFINITE:
        raise NonFiniteError(msg)
    if rc == NO_DEVICE:
        raise NoDeviceError(msg + " " + detail)
    raise CudaError(msg)


class HostTensor(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("precision", C.c_int32),
        ("block_size", C.c_uint32),
        ("freqs", C.c_void_p),
        ("stream", C.c_void_p),
        ("stream_len", C.c_uint64),
        ("mantissas", C.c_void_p),
        ("mantissa_len", C.c_uint64),
        ("scales", C.c_void_p),
        ("scales_len", C.c_uint64),
        ("index", C.c_void_p),
        ("index_len", C.c_uint64),
    ]


class ChunkView(C.Structure):
    """nzgpu_chunk_view: one AnsChunk (ans.hpp:159-164)."""
    _fields_ = [("payload", C.c_void_p), ("len", C.c_uint32), ("nsym", C.c_uint32)]


class HostSections(C.Structure):
    """nzgpu_host_sections: a host tensor with the stream as chunk views."""
    _fields_ = [
        ("n", C.c_uint64),
        ("precision", C.c_int32),
        ("block_size", C.c_uint32),
        ("freqs", C.c_void_p),
        ("chunks", C.POINTER(ChunkView)),
        ("nchunks", C.c_uint64),
        ("mantissas", C.c_void_p),
        ("mantissa_len", C.c_uint64),
        ("scales", C.c_void_p),
        ("scales_len", C.c_uint64),
        ("index", C.c_void_p),
        ("index_len", C.c_uint64),
    ]


class BlobInfo(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("precision", C.c_int32),
        ("block_size", C.c_uint32),
        ("chunk_symbols", C.c_uint32),
        ("interval", C.c_uint32),
        ("num_chunks", C.c_uint64),
        ("stream_len", C.c_uint64),
        ("mantissa_len", C.c_uint64),
        ("scales_len", C.c_uint64),
        ("index_len", C.c_uint64),
        ("payload_bytes", C.c_uint64),
        ("d_stream", C.c_void_p),
        ("d_freqs", C.c_void_p),
        ("d_mantissas", C.c_void_p),
        ("d_scales", C.c_void_p),
        ("flags", C.c_uint32),
        ("max_window", C.c_uint32),
    ]


# Every exported symbol of include/nzgpu.h with its ctypes signature.
_vp, _u64, _u32, _i, _p = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER
SIGNATURES = {
    "nzgpu_status_string": (C.c_char_p, [_i]),
    "nzgpu_version": (_i, []),
    "nzgpu_device_check": (_i, [_p(_i)]),
    "nzgpu_last_error_message": (C.c_char_p, []),
    "nzgpu_set_decode_kernel": (_i, [_i]),
    "nzgpu_compress": (_i, [_vp, _u64, _i, _u32, _u32, _u32, _vp, _p(_vp)]),
    "nzgpu_compress_batch_workspace_size": (_i, [_p(_u64), _i, _i, _u32, _p(_u64)]),
    "nzgpu_compress_batch": (_i, [_p(_vp), _p(_u64), _i, _i, _u32, _u32, _u32, _vp, _u64, _vp, _p(_vp)]),
    "nzgpu_decompress": (_i, [_vp, _vp, _vp]),
    "nzgpu_blob_status": (_i, [_vp, _vp]),
    "nzgpu_blob_info_get": (_i, [_vp, _p(BlobInfo)]),
    "nzgpu_blob_free": (_i, [_vp]),
    "nzgpu_blob_export": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "nzgpu_blob_chunks": (_i, [_vp, _vp, _vp]),
    "nzgpu_blob_export_chunks": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "nzgpu_blob_import": (_i, [_p(HostTensor), _u32, _vp, _p(_vp)]),
    "nzgpu_blob_decompress_host": (_i, [_vp, _vp]),
    "nzgpu_decompress_host_sections": (_i, [_p(HostSections), _vp]),
    "nzgpu_trim_device_pool": (_i, []),
    "nzgpu_shannon_entropy": (_i, [_vp, _u64, _vp]),
    "nzgpu_plan_create": (_i, [_p(_vp), _p(_vp), _i, _p(_vp)]),
    "nzgpu_plan_launch": (_i, [_vp, _vp]),
    "nzgpu_plan_status": (_i, [_vp, _vp]),
    "nzgpu_plan_free": (_i, [_vp]),
    "nzgpu_plan_launch_count": (_i, [_vp]),
    "nzgpu_plan_kernel": (_i, [_vp]),
    "nzgpu_plan_set_max_ctas": (_i, [_vp, _u32]),
    "nzgpu_compress_host": (_i, [_vp, _u64, _i, _u32, _u32, _u32, _p(_vp)]),
    "nzgpu_decompress_host": (_i, [_p(HostTensor), _vp]),
    "nzgpu_decompress_host_batch": (_i, [_p(HostTensor), _i, _p(_vp)]),
    "nzgpu_host_release": (_i, []),
    "nzgpu_split": (_i, [_vp, _u64, _vp, _vp, _vp, _vp]),
    "nzgpu_build_table": (_i, [_vp, _vp, _vp]),
    "nzgpu_build_table_host": (_i, [_vp, _vp]),
    "nzgpu_ans_encode_host": (_i, [_vp, _u64, _vp, _u32, _vp, _u64, _p(_u64)]),
    "nzgpu_ans_decode_host": (_i, [_vp, _u64, _vp, _vp, _u64]),
    "nzgpu_lossy_roundtrip_host": (_i, [_vp, _vp, _u64, _i, _vp]),
    "nzgpu_pack_host": (_i, [_vp, _u64, _i, _vp]),
    "nzgpu_unpack_host": (_i, [_vp, _u64, _i, _u64, _vp]),
    "nzgpu_crc32": (_i, [_vp, _u64, _vp, _p(_u32)]),
    "nzgpu_crc32_host": (_i, [_vp, _u64, _p(_u32)]),
    "nzgpu_crc32_host_sections": (_i, [_p(_vp), _p(_u64), _i, _p(_u32)]),
    "nzgpu_blob_nzt_size": (_i, [_vp, _i, _p(_u64)]),
    "nzgpu_blob_write_nzt": (_i, [_vp, _p(_u64), _i, _vp, _u64, _p(_u64)]),
    "nzgpu_blob_read_nzt": (_i, [_vp, _u64, _u32, _vp, _p(_vp), _p(_u64), _p(_i)]),
    "nzgpu_component_histogram": (_i, [_vp, _u64, _vp, _vp]),
    "nzgpu_component_histogram_host": (_i, [_vp, _u64, _vp]),
    "nzgpu_entropy_from_histogram": (_i, [_vp, _vp]),
    "nzgpu_entropy_report": (_i, [_vp, _u64, _vp, _vp]),
    "nzgpu_entropy_report_host": (_i, [_vp, _u64, _vp]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the codec has no CPU fallback)"
        )
    L = C.CDLL(LIB_PATH)
    variant = "NZGPU_LIB" in os.environ  # dev A/B of an older build may lack newer entry points
    for name, (res, args) in SIGNATURES.items():
        if variant and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def device_count() -> int:
    n = C.c_int(0)
    lib.nzgpu_device_check(C.byref(n))
    return n.value


def check(rc: int, what: str) -> None:
    _raise(rc, what)
