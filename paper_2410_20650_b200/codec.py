"""Python host mirror of the reference's codec API (tensorstore.hpp, ans.hpp),
backed by the B200 kernels through the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/neuzip/:

=====================================  =====================================
reference (C++)                        here
=====================================  =====================================
compress_lossless(span, meta)  :87     compress_lossless(values, meta)
decompress_lossless(blob)      :112    decompress_lossless(blob)
compress_lossy(v, k, B, meta)  :141    compress_lossy(values, k, block_size, meta)
decompress_lossy(blob)         :215    decompress_lossy(blob)
footprint(blob)                :265    footprint(blob).total()
build_table(counts)   ans.hpp:154      build_table(counts)
ans_encode / serialize_stream  :260    ans_encode(symbols, freqs) -> bytes
deserialize_stream / ans_decode :273   ans_decode(stream, freqs, n)
std::invalid_argument                  ValueError
FormatError / NonFiniteError           FormatError / NonFiniteError
=====================================  =====================================

Blobs hold the reference's byte formats (table, serialized exponent stream,
sign/mantissa plane, scales) plus an optional ``index`` -- the GPU side
index, which is not part of the format and not counted by ``footprint``.

``DeviceBlob`` / ``DecodePlan`` are the device-resident API (torch CUDA
tensors in and out, stream-ordered) used for layer-by-layer decoding.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import nzgpu as N

kDefaultBlockSize = N.DEFAULT_BLOCK
kLosslessPrecision = N.LOSSLESS
kChunkSymbols = N.DEFAULT_CHUNK
kTableBytes = 512


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else None


@dataclass
class TensorMeta:
    """tensorstore.hpp:38-56"""
    shape: tuple = ()

    def element_count(self) -> int:
        n = 1
        for d in self.shape:
            n *= int(d)
        return n if self.shape else 0

    def validate(self) -> None:
        if not self.shape:
            raise ValueError("tensor shape is empty")
        if len(self.shape) > 8:
            raise ValueError("tensor rank exceeds 8")
        if any(int(d) == 0 for d in self.shape):
            raise ValueError("tensor dimension is zero")


@dataclass
class LosslessBlob:
    """tensorstore.hpp:64-70 (exp_stream serialized; table = freqs)."""
    meta: TensorMeta
    freqs: np.ndarray
    stream: bytes
    signmant: np.ndarray
    index: Optional[bytes] = field(default=None, repr=False)

    precision = kLosslessPrecision


@dataclass
class LossyBlob:
    """tensorstore.hpp:72-81"""
    meta: TensorMeta
    precision: int
    block_size: int
    scales: np.ndarray
    freqs: np.ndarray
    stream: bytes
    signmant: np.ndarray
    index: Optional[bytes] = field(default=None, repr=False)


Blob = Union[LosslessBlob, LossyBlob]


@dataclass
class Footprint:
    """tensorstore.hpp:242-253"""
    exponent_bytes: int = 0
    mantissa_bytes: int = 0
    scale_bytes: int = 0
    table_bytes: int = 0
    header_bytes: int = 0

    def total(self) -> int:
        return self.exponent_bytes + self.mantissa_bytes + self.scale_bytes + self.table_bytes + self.header_bytes


def nzt_header_bytes(ndim: int) -> int:
    """detail::nzt_header_bytes, tensorstore.hpp:259-261"""
    return 4 + 1 + 1 + 4 + 1 + 8 * ndim + 4 + 8 + 8 + 4


def footprint(blob: Blob) -> Footprint:
    """tensorstore.hpp:265-287 (the side index is not counted)."""
    return Footprint(
        exponent_bytes=len(blob.stream),
        mantissa_bytes=int(blob.signmant.size),
        scale_bytes=int(blob.scales.size) if isinstance(blob, LossyBlob) else 0,
        table_bytes=kTableBytes,
        header_bytes=nzt_header_bytes(len(blob.meta.shape)),
    )


def ratio(blob: Blob) -> float:
    """2n / footprint total (neuzip.cpp:78, acceptance.cpp:106-108)."""
    return 2 * blob.meta.element_count() / footprint(blob).total()


def _as_u16(values) -> np.ndarray:
    if hasattr(values, "detach"):  # torch tensor
        import torch

        t = values.detach()
        if t.dtype == torch.bfloat16:
            t = t.view(torch.int16)
        values = t.cpu().numpy().view(np.uint16)
    a = np.asarray(values)
    if a.dtype != np.uint16:
        a = a.astype(np.uint16)
    return np.ascontiguousarray(a.reshape(-1))


# ------------------------------------------------------------ blob <-> C ABI
class DeviceBlob:
    """A compressed tensor resident in HBM (C ABI ``nzgpu_blob``)."""

    def __init__(self, handle: C.c_void_p, meta: Optional[TensorMeta] = None):
        self._h = handle
        info = N.BlobInfo()
        N.check(N.lib.nzgpu_blob_info_get(handle, C.byref(info)), "blob info")
        self.info = info
        self.meta = meta or TensorMeta((int(info.n),))

    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return int(self.info.n)

    @property
    def precision(self) -> int:
        return int(self.info.precision)

    def free(self) -> None:
        if self._h:
            N.lib.nzgpu_blob_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # -- construction
    @classmethod
    def compress(cls, values, precision: int = kLosslessPrecision, block_size: int = kDefaultBlockSize,
                 chunk_symbols: int = kChunkSymbols, interval: int = 0, stream=None,
                 meta: Optional[TensorMeta] = None) -> "DeviceBlob":
        """values: CUDA tensor of bf16 (or int16/uint16 bit patterns), 16-B aligned."""
        import torch

        if values.dtype == torch.bfloat16:
            values = values.view(torch.int16)
        values = values.contiguous().view(-1)
        h = C.c_void_p()
        rc = N.lib.nzgpu_compress(C.c_void_p(values.data_ptr()), values.numel(), precision, block_size,
                                  chunk_symbols, interval, _stream_ptr(stream), C.byref(h))
        N.check(rc, "compress")
        return cls(h, meta)

    @classmethod
    def compress_batch(cls, values: Sequence, precision: int = kLosslessPrecision,
                       block_size: int = kDefaultBlockSize, chunk_symbols: int = kChunkSymbols,
                       interval: int = 0, stream=None, metas: Optional[Sequence[TensorMeta]] = None,
                       max_batch_elements: int = 1 << 32, workspace=None) -> list:
        """Compress many CUDA tensors with one encode launch per batch
        (nzgpu_compress_batch); result i is byte-identical to
        ``compress(values[i], ...)``.  Batches are cut at
        ``max_batch_elements`` (temporaries are ~3 B per element).
        ``workspace``: an optional uint8 CUDA tensor reused for the
        temporaries when large enough (see ``compress_workspace_bytes``)."""
        import torch

        flat = []
        for v in values:
            if v.dtype == torch.bfloat16:
                v = v.view(torch.int16)
            flat.append(v.contiguous().view(-1))
        out: list = []
        i = 0
        while i < len(flat):
            j, tot = i, 0
            while j < len(flat) and (j == i or tot + flat[j].numel() <= max_batch_elements):
                tot += flat[j].numel()
                j += 1
            part = flat[i:j]
            ptrs = (C.c_void_p * len(part))(*[t.data_ptr() for t in part])
            ns = (C.c_uint64 * len(part))(*[t.numel() for t in part])
            hs = (C.c_void_p * len(part))()
            # temporaries from torch's caching allocator: repeated batches
            # reuse the mapping instead of paying for fresh device memory
            wsb = C.c_uint64()
            N.check(N.lib.nzgpu_compress_batch_workspace_size(ns, len(part), precision, chunk_symbols,
                                                              C.byref(wsb)), "compress_batch")
            if workspace is not None and workspace.numel() >= wsb.value + 256:
                ws = workspace
            else:
                ws = torch.empty(wsb.value + 256, dtype=torch.uint8, device=part[0].device)
            wp = (ws.data_ptr() + 255) & ~255
            rc = N.lib.nzgpu_compress_batch(ptrs, ns, len(part), precision, block_size, chunk_symbols, interval,
                                            C.c_void_p(wp), wsb.value, _stream_ptr(stream), hs)
            N.check(rc, "compress_batch")
            for k in range(len(part)):
                out.append(cls(C.c_void_p(hs[k]), metas[i + k] if metas else None))
            i = j
        return out

    @staticmethod
    def compress_workspace_bytes(sizes: Sequence[int], precision: int = kLosslessPrecision,
                                 chunk_symbols: int = kChunkSymbols) -> int:
        """Workspace bytes of one compress_batch over tensors of these sizes."""
        ns = (C.c_uint64 * len(sizes))(*sizes)
        out = C.c_uint64()
        N.check(N.lib.nzgpu_compress_batch_workspace_size(ns, len(sizes), precision, chunk_symbols, C.byref(out)),
                "compress_workspace_bytes")
        return int(out.value) + 256

    @classmethod
    def from_host(cls, blob: Blob, interval: int = 0) -> "DeviceBlob":
        t, keep = _host_tensor(blob)
        h = C.c_void_p()
        N.check(N.lib.nzgpu_blob_import(C.byref(t), interval, None, C.byref(h)), "import")
        del keep
        return cls(h, blob.meta)

    # -- decode
    def decompress_into(self, out, stream=None) -> None:
        _check_output(out, self.n, "decompress_into")
        rc = N.lib.nzgpu_decompress(self._h, C.c_void_p(out.data_ptr()), _stream_ptr(stream))
        N.check(rc, "decompress")

    def decompress(self, stream=None):
        import torch

        out = torch.empty(self.n, dtype=torch.bfloat16, device="cuda")
        self.decompress_into(out, stream)
        self.status(stream)
        return out

    def status(self, stream=None) -> None:
        N.check(N.lib.nzgpu_blob_status(self._h, _stream_ptr(stream)), "decode")

    # -- export to the reference's host formats
    def to_host(self) -> Blob:
        i = self.info
        freqs = np.zeros(256, np.uint16)
        stream = np.zeros(max(int(i.stream_len), 1), np.uint8)
        mant = np.zeros(max(int(i.mantissa_len), 1), np.uint8)
        scales = np.zeros(max(int(i.scales_len), 1), np.uint8)
        index = np.zeros(max(int(i.index_len), 1), np.uint8)
        N.check(N.lib.nzgpu_blob_export(self._h, _ptr(freqs), _ptr(stream), _ptr(mant), _ptr(scales),
                                        _ptr(index)), "export")
        stream_b = stream[: i.stream_len].tobytes()
        idx = index[: i.index_len].tobytes() if i.index_len else None
        if i.precision == kLosslessPrecision:
            return LosslessBlob(self.meta, freqs, stream_b, mant[: i.mantissa_len], idx)
        return LossyBlob(self.meta, int(i.precision), int(i.block_size), scales[: i.scales_len], freqs, stream_b,
                         mant[: i.mantissa_len], idx)


    # -- NZT container (tensorstore.hpp:289-477)
    def to_nzt(self, shape=None) -> bytes:
        """write_nzt of this blob: sections D2H, CRC-32 on the GPU."""
        shape = tuple(shape if shape is not None else (self.meta.shape if self.meta else (self.n,)))
        size = C.c_uint64()
        N.check(N.lib.nzgpu_blob_nzt_size(self._h, len(shape), C.byref(size)), "nzt size")
        out = np.zeros(size.value, np.uint8)
        dims = (C.c_uint64 * len(shape))(*shape)
        written = C.c_uint64()
        N.check(N.lib.nzgpu_blob_write_nzt(self._h, dims, len(shape), _ptr(out), size.value, C.byref(written)),
                "write_nzt")
        return out[: written.value].tobytes()

    @classmethod
    def from_nzt(cls, data: bytes, interval: int = 0) -> "DeviceBlob":
        """read_nzt into a device blob (CRC checked on the GPU)."""
        buf = np.frombuffer(data, np.uint8)
        h = C.c_void_p()
        dims = (C.c_uint64 * 8)()
        nd = C.c_int()
        N.check(N.lib.nzgpu_blob_read_nzt(_ptr(buf) if buf.size else None, buf.size, interval, None, C.byref(h),
                                          dims, C.byref(nd)), "read_nzt")
        return cls(h, TensorMeta(tuple(int(dims[i]) for i in range(nd.value))))


def crc32(*sections) -> int:
    """crc32.hpp:38-42 over the concatenation of host byte sections,
    computed on the GPU."""
    arrs = [np.ascontiguousarray(np.frombuffer(bytes(s), np.uint8) if isinstance(s, (bytes, bytearray, memoryview))
                                 else np.asarray(s).view(np.uint8).reshape(-1)) for s in sections]
    ptrs = (C.c_void_p * max(len(arrs), 1))(*[_ptr(a) if a.size else None for a in arrs])
    lens = (C.c_uint64 * max(len(arrs), 1))(*[a.size for a in arrs])
    out = C.c_uint32()
    N.check(N.lib.nzgpu_crc32_host_sections(ptrs, lens, len(arrs), C.byref(out)), "crc32")
    return int(out.value)


@dataclass
class EntropyReport:
    """entropy.hpp:57-66"""
    h_sign: float
    h_exp: float
    h_mant: float
    ideal_ratio: float
    exponent_only_ratio: float


def component_histogram(values):
    """ComponentHistogram (entropy.hpp:17-39) on the GPU: (sign[2], exp[256],
    mant[128]) counts.  values: CUDA bf16/int16 tensor."""
    import torch

    if values.dtype == torch.bfloat16:
        values = values.view(torch.int16)
    values = values.contiguous().view(-1)
    counts = np.zeros(386, np.uint64)
    N.check(N.lib.nzgpu_component_histogram(C.c_void_p(values.data_ptr()), values.numel(), _stream_ptr(None),
                                            _ptr(counts)), "component_histogram")
    return counts[:2], counts[2:258], counts[258:]


def analyze_tensor(values) -> EntropyReport:
    """analyze_tensor (entropy.hpp:89-94): host bf16 bit patterns or a CUDA
    tensor; the histogram runs on the GPU."""
    out = np.zeros(5, np.float64)
    if hasattr(values, "is_cuda") and values.is_cuda:
        import torch

        v = values.view(torch.int16).contiguous().view(-1) if values.dtype == torch.bfloat16 else values.contiguous().view(-1)
        if v.numel() == 0:
            raise ValueError("analyze_tensor: empty input")
        N.check(N.lib.nzgpu_entropy_report(C.c_void_p(v.data_ptr()), v.numel(), _stream_ptr(None), _ptr(out)),
                "analyze_tensor")
    else:
        v = _as_u16(values)
        if v.size == 0:
            raise ValueError("analyze_tensor: empty input")
        N.check(N.lib.nzgpu_entropy_report_host(_ptr(v), v.size, _ptr(out)), "analyze_tensor")
    return EntropyReport(*[float(x) for x in out])


def write_nzt(blob: Blob) -> bytes:
    """write_nzt (tensorstore.hpp:352-376) of a host blob; the CRC is computed
    on the GPU.  Byte-identical to the reference's file."""
    import struct

    blob.meta.validate()
    lossless = isinstance(blob, LosslessBlob)
    prec = kLosslessPrecision if lossless else int(blob.precision)
    block = 0 if lossless else int(blob.block_size)
    table = np.ascontiguousarray(blob.freqs, dtype="<u2").tobytes()
    scales = b"" if lossless else np.ascontiguousarray(blob.scales, np.uint8).tobytes()
    stream = bytes(blob.stream)
    sm = np.ascontiguousarray(blob.signmant, np.uint8).tobytes()
    crc = crc32(table, scales, stream, sm)
    head = b"NZT1" + struct.pack("<BBIB", 1, prec, block, len(blob.meta.shape))
    head += b"".join(struct.pack("<Q", d) for d in blob.meta.shape)
    return b"".join([head, table, struct.pack("<I", len(scales)), scales, struct.pack("<Q", len(stream)), stream,
                     struct.pack("<Q", len(sm)), sm, struct.pack("<I", crc)])


def read_nzt(data: bytes) -> Blob:
    """read_nzt (tensorstore.hpp:403-477): framing, CRC (on the GPU;
    ChecksumError), table and stream validation; returns the host blob with
    the GPU checkpoint index attached."""
    db = DeviceBlob.from_nzt(data)
    try:
        return db.to_host()
    finally:
        db.free()


def _check_output(out, n: int, what: str) -> None:
    """The kernels write n bf16 with 16-byte stores through a raw pointer:
    reject anything that would turn into an out-of-bounds device write."""
    if not hasattr(out, "data_ptr") or not hasattr(out, "is_cuda"):
        raise ValueError(f"{what}: expected a CUDA tensor")
    if not out.is_cuda:
        raise ValueError(f"{what}: output must be a CUDA tensor, got {out.device}")
    if out.element_size() != 2:
        raise ValueError(f"{what}: output must have 2-byte elements (bf16/int16), got {out.dtype}")
    if not out.is_contiguous():
        raise ValueError(f"{what}: output must be contiguous")
    if out.numel() < n:
        raise ValueError(f"{what}: output holds {out.numel()} elements, the blob decodes {n}")
    if n and out.data_ptr() % 16:
        raise ValueError(f"{what}: output must be 16-byte aligned")


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _host_tensor(blob: Blob):
    n = blob.meta.element_count()
    freqs = np.ascontiguousarray(blob.freqs, dtype=np.uint16)
    if freqs.size != 256:
        raise FormatError("frequency table must be 512 bytes")
    stream = np.frombuffer(blob.stream, np.uint8) if len(blob.stream) else np.zeros(0, np.uint8)
    mant = np.ascontiguousarray(blob.signmant, dtype=np.uint8)
    t = N.HostTensor()
    t.n = n
    t.precision = blob.precision
    t.freqs = _ptr(freqs)
    t.stream = _ptr(stream)
    t.stream_len = stream.size
    t.mantissas = _ptr(mant)
    t.mantissa_len = mant.size
    keep = [freqs, stream, mant]
    if isinstance(blob, LossyBlob):
        sc = np.ascontiguousarray(blob.scales, dtype=np.uint8)
        t.block_size = blob.block_size
        t.scales = _ptr(sc)
        t.scales_len = sc.size
        keep.append(sc)
    if blob.index:
        idx = np.frombuffer(blob.index, np.uint8)
        t.index = _ptr(idx)
        t.index_len = idx.size
        keep.append(idx)
    return t, keep


FormatError = N.FormatError
NonFiniteError = N.NonFiniteError
ChecksumError = N.ChecksumError
Error = N.Error


# --------------------------------------------------------- reference API ---
def compress_lossless(values, meta: Optional[TensorMeta] = None, chunk_symbols: int = kChunkSymbols,
                      interval: int = 0) -> LosslessBlob:
    """tensorstore.hpp:87-110"""
    v = _as_u16(values)
    meta = meta or TensorMeta((v.size,))
    meta.validate()
    if meta.element_count() != v.size:
        raise ValueError("compress: shape does not match value count")
    h = C.c_void_p()
    N.check(N.lib.nzgpu_compress_host(_ptr(v), v.size, kLosslessPrecision, 0, chunk_symbols, interval,
                                      C.byref(h)), "compress_lossless")
    db = DeviceBlob(h, meta)
    try:
        return db.to_host()
    finally:
        db.free()


def compress_lossy(values, k: int, block_size: int = kDefaultBlockSize, meta: Optional[TensorMeta] = None,
                   chunk_symbols: int = kChunkSymbols, interval: int = 0) -> LossyBlob:
    """tensorstore.hpp:141-213"""
    if k not in (0, 1, 3):
        raise ValueError("compress_lossy: precision must be 0, 1 or 3")
    if block_size == 0:
        raise ValueError("compress_lossy: block size must be >= 1")
    v = _as_u16(values)
    meta = meta or TensorMeta((v.size,))
    meta.validate()
    if meta.element_count() != v.size:
        raise ValueError("compress: shape does not match value count")
    h = C.c_void_p()
    N.check(N.lib.nzgpu_compress_host(_ptr(v), v.size, k, block_size, chunk_symbols, interval, C.byref(h)),
            "compress_lossy")
    db = DeviceBlob(h, meta)
    try:
        return db.to_host()
    finally:
        db.free()


def _decompress(blob: Blob) -> np.ndarray:
    n = blob.meta.element_count()
    out = np.zeros(max(n, 1), np.uint16)
    t, keep = _host_tensor(blob)
    N.check(N.lib.nzgpu_decompress_host(C.byref(t), _ptr(out)), "decompress")
    del keep
    return out[:n]


def decompress_lossless(blob: LosslessBlob) -> np.ndarray:
    """tensorstore.hpp:112-125 -> bf16 bit patterns (uint16)."""
    return _decompress(blob)


def decompress_lossy(blob: LossyBlob) -> np.ndarray:
    """tensorstore.hpp:215-238 -> bf16 bit patterns (uint16)."""
    return _decompress(blob)


def decompress_batch(blobs: Sequence[Blob]) -> list:
    """Pipelined host decode of many blobs (nzgpu_decompress_host_batch)."""
    outs = [np.zeros(max(b.meta.element_count(), 1), np.uint16) for b in blobs]
    ts, keeps = zip(*[_host_tensor(b) for b in blobs]) if blobs else ((), ())
    arr = (N.HostTensor * len(ts))(*ts)
    ptrs = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
    N.check(N.lib.nzgpu_decompress_host_batch(arr, len(ts), ptrs), "decompress_batch")
    return [o[: b.meta.element_count()] for o, b in zip(outs, blobs)]


def release_host_buffers() -> None:
    """Free the calling thread's host-tier device staging (nzgpu_host_release)."""
    N.check(N.lib.nzgpu_host_release(), "host_release")


def build_table(counts) -> np.ndarray:
    """FrequencyTable::from_counts (ans.hpp:52-93), run by the K2 kernel."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    if c.size != 256:
        raise ValueError("frequency table needs 256 counts")
    f = np.zeros(256, np.uint16)
    N.check(N.lib.nzgpu_build_table_host(_ptr(c), _ptr(f)), "build_table")
    return f


def ans_encode(symbols, freqs, chunk_symbols: int = kChunkSymbols) -> bytes:
    """serialize_stream(ans_encode(symbols, table)) (ans.hpp:260-271, :306-316)."""
    x = np.ascontiguousarray(symbols, dtype=np.uint8).reshape(-1)
    f = np.ascontiguousarray(freqs, dtype=np.uint16)
    nch = (x.size + chunk_symbols - 1) // chunk_symbols
    cap = 4 + 12 * nch + 2 * x.size + 16
    out = np.zeros(cap, np.uint8)
    ln = C.c_uint64(0)
    N.check(N.lib.nzgpu_ans_encode_host(_ptr(x), x.size, _ptr(f), chunk_symbols, _ptr(out), cap, C.byref(ln)),
            "ans_encode")
    return out[: ln.value].tobytes()


def ans_decode(stream: bytes, freqs, n: int) -> np.ndarray:
    """ans_decode(deserialize_stream(bytes, table)) (ans.hpp:273-293, :318-347)."""
    s = np.frombuffer(stream, np.uint8) if len(stream) else np.zeros(0, np.uint8)
    f = np.ascontiguousarray(freqs, dtype=np.uint16)
    out = np.zeros(max(n, 1), np.uint8)
    N.check(N.lib.nzgpu_ans_decode_host(_ptr(s) if s.size else None, s.size, _ptr(f), _ptr(out), n), "ans_decode")
    return out[:n]


def pack_signed_mantissas(signs, mants, k: int) -> np.ndarray:
    """bitfloat.hpp:124-143 on the GPU: (k+1)-bit items, MSB-first."""
    if k not in (0, 1, 3, 7):
        raise ValueError("pack: k must be one of {0,1,3,7}")
    s = np.ascontiguousarray(signs, dtype=np.uint8).reshape(-1)
    m = np.ascontiguousarray(mants, dtype=np.uint8).reshape(-1)
    items = ((s.astype(np.uint32) << k) | m).astype(np.uint8) if s.size else np.zeros(0, np.uint8)
    if s.size and ((s > 1).any() or (m >= (1 << k)).any()):
        raise ValueError("pack: item exceeds k+1 bits")
    out = np.zeros(max((s.size * (k + 1) + 7) // 8, 1), np.uint8)
    N.check(N.lib.nzgpu_pack_host(_ptr(items), s.size, k, _ptr(out)), "pack_signed_mantissas")
    return out[: (s.size * (k + 1) + 7) // 8]


def unpack_signed_mantissas(packed, k: int, n: int):
    """bitfloat.hpp:145-164 on the GPU -> (signs, mantissas)."""
    p = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
    items = np.zeros(max(n, 1), np.uint8)
    N.check(N.lib.nzgpu_unpack_host(_ptr(p), p.size, k, n, _ptr(items)), "unpack_signed_mantissas")
    items = items[:n]
    return items >> k, items & ((1 << k) - 1)


def lossy_roundtrip(values, scales, k: int) -> np.ndarray:
    """Element-wise lossy round trip under explicit scale bytes (exhaustive
    parity harness for tensorstore.hpp:179-198 + :229-236)."""
    v = _as_u16(values)
    s = np.ascontiguousarray(scales, dtype=np.uint8).reshape(-1)
    out = np.zeros(max(v.size, 1), np.uint16)
    N.check(N.lib.nzgpu_lossy_roundtrip_host(_ptr(v), _ptr(s), v.size, k, _ptr(out)), "lossy_roundtrip")
    return out[: v.size]


class DecodePlan:
    """One kernel launch decoding many DeviceBlobs (e.g. one transformer
    layer) into their output tensors (nzgpu_plan_*)."""

    def __init__(self, blobs: Sequence[DeviceBlob], outs):
        self.blobs = list(blobs)
        self.outs = list(outs)
        if not self.blobs or len(self.outs) != len(self.blobs):
            raise ValueError(f"DecodePlan: {len(self.blobs)} blobs but {len(self.outs)} outputs")
        dev = None
        for i, (b, o) in enumerate(zip(self.blobs, self.outs)):
            _check_output(o, b.n, f"DecodePlan output {i}")
            if dev is None:
                dev = o.device
            elif o.device != dev:
                raise ValueError(f"DecodePlan output {i} is on {o.device}, the others on {dev}")
        hs = (C.c_void_p * len(blobs))(*[b.handle for b in blobs])
        ps = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        self._h = C.c_void_p()
        N.check(N.lib.nzgpu_plan_create(hs, ps, len(blobs), C.byref(self._h)), "plan_create")

    def launch(self, stream=None) -> None:
        N.check(N.lib.nzgpu_plan_launch(self._h, _stream_ptr(stream)), "plan_launch")

    def status(self, stream=None) -> None:
        N.check(N.lib.nzgpu_plan_status(self._h, _stream_ptr(stream)), "plan decode")

    @property
    def launches(self) -> int:
        return int(N.lib.nzgpu_plan_launch_count(self._h))

    def set_max_ctas(self, max_ctas: int) -> None:
        """Decode on at most `max_ctas` SMs (0 = all), leaving the rest to
        concurrent kernels on other streams."""
        N.check(N.lib.nzgpu_plan_set_max_ctas(self._h, int(max_ctas)), "plan_set_max_ctas")

    @property
    def kernel(self) -> str:
        """Decode kernel the next launch uses."""
        return {0: "decode_persist_kernel", 1: "decode_tiles_kernel"}.get(
            int(N.lib.nzgpu_plan_kernel(self._h)), "none")

    def free(self) -> None:
        if self._h:
            N.lib.nzgpu_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
