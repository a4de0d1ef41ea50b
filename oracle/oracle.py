"""ctypes front end for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product (``paper_2410_20650_b200``) never does.

Two backends with the same function set:

* ``Oracle(lib="port")`` -- ``oracle/liboracle.so``, the plain-C restatement
  (``neuzip_oracle.c``), always buildable from this repo.
* ``Oracle(lib="ref")``  -- ``oracle/_ref/libneuzip_ref.so``, the UNMODIFIED
  reference headers (``/root/reference/proj/include``) behind a C shim,
  built by ``oracle/Makefile`` where the reference is mounted.

Status codes follow ``neuzip_oracle.h`` (0 ok, -1 invalid_argument,
-2 truncated, -3 desync, -4 length mismatch, -5 non-finite, -6 bad table).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libneuzip_ref.so")

OK, INVALID, TRUNCATED, DESYNC, LENGTH, NONFINITE, BAD_TABLE = 0, -1, -2, -3, -4, -5, -6
CHUNK = 65536


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


_u64, _i64, _int, _u32, _dbl, _vp = C.c_uint64, C.c_int64, C.c_int, C.c_uint32, C.c_double, C.c_void_p


class Oracle:
    def __init__(self, lib: str = "port"):
        path = PORT_SO if lib == "port" else REF_SO
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.kind = lib
        self.lib = C.CDLL(path)
        pre = "orc_" if lib == "port" else "ref_"
        L = self.lib

        def fn(name, res, args):
            f = getattr(L, pre + name)
            f.restype = res
            f.argtypes = args
            return f

        self._build_table = fn("build_table", _int, [_vp, _vp])
        self._enc_chunk = fn("ans_encode_chunk", _i64, [_vp, _u64, _vp, _vp])
        self._dec_chunk = fn("ans_decode_chunk", _int, [_vp, _u64, _u64, _vp, _vp])
        self._enc_stream = fn("ans_encode_stream", _i64, [_vp, _u64, _u64, _vp, _vp])
        self._dec_stream = fn("ans_decode_stream", _int, [_vp, _u64, _vp, _vp, _u64])
        self._comp = fn("compress_lossless", _i64, [_vp, _u64, _u64, _vp, _vp, _vp])
        self._decomp = fn("decompress_lossless", _int, [_vp, _u64, _vp, _vp, _u64, _u64, _vp])
        self._comp_lossy = fn("compress_lossy", _i64, [_vp, _u64, _int, _u32, _u64, _vp, _vp, _vp, _vp])
        self._decomp_lossy = fn(
            "decompress_lossy", _int, [_vp, _u64, _vp, _vp, _u64, _vp, _u64, _int, _u32, _u64, _vp]
        )
        self._gauss = fn("gaussian_bf16", None, [_u64, _u64, _dbl, _vp])
        self._derive = fn("rng_derive", _u64, [_u64, _u64])
        self._crc = fn("crc32", _u32, [_vp, _u64])
        if lib == "port":
            self._lossy_rt = fn("lossy_roundtrip", C.c_uint16, [C.c_uint16, C.c_uint8, _int])
            self._lossy_rt_many = fn("lossy_roundtrip_many", None, [_vp, _vp, _u64, _int, _vp])
            self._round = fn("round_mantissa", _int, [_int, _int, _vp, _vp])
            self._pack = fn("pack_signed_mantissas", _int, [_vp, _vp, _u64, _int, _vp])
            self._unpack = fn("unpack_signed_mantissas", _int, [_vp, _u64, _int, _u64, _vp, _vp])
            self._from_float = fn("bf16_from_float", C.c_uint16, [C.c_float])
        else:
            self._prepare = fn("prepare", _vp, [_vp, _u64, _vp, _vp, _u64, _vp, _u64, _int, _u32, _u64])
            self._dec_prepared = fn("decompress_prepared", _int, [_vp, _vp])
            self._free_prepared = fn("free_prepared", None, [_vp])
            self._entropy = fn("entropy_report", None, [_vp, _u64, _vp])
            self._nzt = fn("write_nzt_lossless", _i64, [_vp, _vp, _int, _vp, _u64])
            self._nzt_lossy = fn("write_nzt_lossy", _i64, [_vp, _vp, _int, _int, _u32, _vp, _u64])
            self._read_nzt = fn("read_nzt", _int, [_vp, _u64, _vp, _u64, _vp])

    # -- tables / coder -------------------------------------------------
    def build_table(self, counts) -> np.ndarray:
        counts = np.ascontiguousarray(counts, dtype=np.uint64)
        assert counts.size == 256
        freqs = np.zeros(256, np.uint16)
        rc = self._build_table(_p(counts), _p(freqs))
        if rc:
            raise OracleError(rc, "build_table")
        return freqs

    def encode_chunk(self, syms, freqs) -> bytes:
        syms = np.ascontiguousarray(syms, dtype=np.uint8)
        freqs = np.ascontiguousarray(freqs, dtype=np.uint16)
        out = np.zeros(2 * syms.size + 8, np.uint8)
        n = self._enc_chunk(_p(syms), syms.size, _p(freqs), _p(out))
        if n < 0:
            raise OracleError(n, "ans_encode_chunk")
        return out[:n].tobytes()

    def decode_chunk(self, payload: bytes, nsym: int, freqs) -> np.ndarray:
        buf = np.frombuffer(payload, np.uint8).copy() if payload else np.zeros(1, np.uint8)
        freqs = np.ascontiguousarray(freqs, dtype=np.uint16)
        out = np.zeros(max(nsym, 1), np.uint8)
        rc = self._dec_chunk(_p(buf), len(payload), nsym, _p(freqs), _p(out))
        if rc:
            raise OracleError(rc, "ans_decode_chunk")
        return out[:nsym]

    def encode_stream(self, syms, freqs, chunk: int = CHUNK) -> bytes:
        syms = np.ascontiguousarray(syms, dtype=np.uint8)
        freqs = np.ascontiguousarray(freqs, dtype=np.uint16)
        nch = (syms.size + chunk - 1) // chunk
        out = np.zeros(4 + 12 * nch + 2 * syms.size + 16, np.uint8)
        n = self._enc_stream(_p(syms), syms.size, chunk, _p(freqs), _p(out))
        if n < 0:
            raise OracleError(n, "ans_encode")
        return out[:n].tobytes()

    def decode_stream(self, stream: bytes, freqs, n: int) -> np.ndarray:
        buf = np.frombuffer(stream, np.uint8).copy()
        freqs = np.ascontiguousarray(freqs, dtype=np.uint16)
        out = np.zeros(max(n, 1), np.uint8)
        rc = self._dec_stream(_p(buf), len(stream), _p(freqs), _p(out), n)
        if rc:
            raise OracleError(rc, "ans_decode")
        return out[:n]

    # -- tensor codec ---------------------------------------------------
    def compress_lossless(self, values, chunk: int = CHUNK):
        """-> (freqs u16[256], stream bytes, signmant u8[n])"""
        v = np.ascontiguousarray(values, dtype=np.uint16)
        n = v.size
        freqs = np.zeros(256, np.uint16)
        nch = (n + chunk - 1) // chunk
        stream = np.zeros(4 + 12 * nch + 2 * n + 16, np.uint8)
        sm = np.zeros(max(n, 1), np.uint8)
        ln = self._comp(_p(v), n, chunk, _p(freqs), _p(stream), _p(sm))
        if ln < 0:
            raise OracleError(ln, "compress_lossless")
        return freqs, stream[:ln].tobytes(), sm[:n]

    def decompress_lossless(self, freqs, stream: bytes, signmant, n: int) -> np.ndarray:
        buf = np.frombuffer(stream, np.uint8).copy()
        freqs = np.ascontiguousarray(freqs, dtype=np.uint16)
        sm = np.ascontiguousarray(signmant, dtype=np.uint8)
        out = np.zeros(max(n, 1), np.uint16)
        rc = self._decomp(_p(buf), len(stream), _p(freqs), _p(sm), sm.size, n, _p(out))
        if rc:
            raise OracleError(rc, "decompress_lossless")
        return out[:n]

    def compress_lossy(self, values, k: int, block: int = 512, chunk: int = CHUNK):
        """-> (freqs, scales u8[ceil(n/B)], stream bytes, packed u8)"""
        v = np.ascontiguousarray(values, dtype=np.uint16)
        n = v.size
        freqs = np.zeros(256, np.uint16)
        nb = (n + block - 1) // block if block else 1
        scales = np.zeros(max(nb, 1), np.uint8)
        nch = (n + chunk - 1) // chunk
        stream = np.zeros(4 + 12 * nch + 2 * n + 16, np.uint8)
        packed = np.zeros(max((n * (k + 1) + 7) // 8, 1), np.uint8)
        ln = self._comp_lossy(_p(v), n, k, block, chunk, _p(freqs), _p(scales), _p(stream), _p(packed))
        if ln < 0:
            raise OracleError(ln, "compress_lossy")
        return freqs, scales[:nb], stream[:ln].tobytes(), packed[: (n * (k + 1) + 7) // 8]

    def decompress_lossy(self, freqs, scales, stream: bytes, packed, k: int, block: int, n: int):
        buf = np.frombuffer(stream, np.uint8).copy()
        freqs = np.ascontiguousarray(freqs, dtype=np.uint16)
        sc = np.ascontiguousarray(scales, dtype=np.uint8)
        pk = np.ascontiguousarray(packed, dtype=np.uint8)
        out = np.zeros(max(n, 1), np.uint16)
        rc = self._decomp_lossy(_p(buf), len(stream), _p(freqs), _p(pk), pk.size, _p(sc), sc.size, k, block, n, _p(out))
        if rc:
            raise OracleError(rc, "decompress_lossy")
        return out[:n]

    # -- inputs / misc --------------------------------------------------
    def gaussian_bf16(self, seed: int, n: int, sigma: float = 0.02) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint16)
        self._gauss(seed, n, sigma, _p(out))
        return out[:n]

    def gaussian_bf16_parallel(self, seed: int, n: int, sigma: float = 0.02, threads: int = 0) -> np.ndarray:
        """gaussian_bf16 filled by host threads over disjoint counter ranges
        (the C restatement; ctypes releases the GIL).  Identical output."""
        import concurrent.futures as cf

        port = self if self.kind == "port" else Oracle("port")
        f = port.lib.orc_gaussian_bf16_range
        f.restype = None
        f.argtypes = [_u64, _u64, _u64, _dbl, _vp]
        out = np.zeros(max(n, 1), np.uint16)
        threads = threads or min(64, os.cpu_count() or 1)
        step = max(1 << 20, -(-n // threads))
        base = out.ctypes.data
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda a: f(seed, a, min(step, n - a), sigma, base + 2 * a), range(0, n, step)))
        return out[:n]

    def derive(self, seed: int, tag: int) -> int:
        return int(self._derive(seed, tag))

    def crc32(self, data: bytes) -> int:
        buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        return int(self._crc(_p(buf), len(data)))

    # port-only helpers
    def lossy_roundtrip(self, bits: int, scale: int, k: int) -> int:
        return int(self._lossy_rt(bits, scale, k))

    def lossy_roundtrip_many(self, bits, scales, k: int) -> np.ndarray:
        b = np.ascontiguousarray(bits, dtype=np.uint16)
        s = np.ascontiguousarray(scales, dtype=np.uint8)
        out = np.zeros(max(b.size, 1), np.uint16)
        self._lossy_rt_many(_p(b), _p(s), b.size, k, _p(out))
        return out[: b.size]

    def round_mantissa(self, m: int, k: int):
        a, b = C.c_int(), C.c_int()
        rc = self._round(m, k, C.byref(a), C.byref(b))
        if rc:
            raise OracleError(rc, "round_mantissa")
        return a.value, bool(b.value)

    def pack(self, signs, mants, k: int) -> np.ndarray:
        s = np.ascontiguousarray(signs, dtype=np.uint8)
        m = np.ascontiguousarray(mants, dtype=np.uint8)
        out = np.zeros(max((s.size * (k + 1) + 7) // 8, 1), np.uint8)
        rc = self._pack(_p(s), _p(m), s.size, k, _p(out))
        if rc:
            raise OracleError(rc, "pack")
        return out[: (s.size * (k + 1) + 7) // 8]

    def unpack(self, packed, k: int, n: int):
        pk = np.ascontiguousarray(packed, dtype=np.uint8)
        s = np.zeros(max(n, 1), np.uint8)
        m = np.zeros(max(n, 1), np.uint8)
        rc = self._unpack(_p(pk) if pk.size else None, pk.size, k, n, _p(s), _p(m))
        if rc:
            raise OracleError(rc, "unpack")
        return s[:n], m[:n]

    def from_float(self, f: float) -> int:
        return int(self._from_float(f))

    # ref-only helpers
    def prepared(self, freqs, stream: bytes, mant, n: int, k: int = 7, scales=None, block: int = 0):
        """A reference Blob built once; .decode(out) times decompress_* alone."""
        lib = self
        buf = np.frombuffer(stream, np.uint8).copy()
        f = np.ascontiguousarray(freqs, dtype=np.uint16)
        m = np.ascontiguousarray(mant, dtype=np.uint8)
        sc = np.ascontiguousarray(scales if scales is not None else np.zeros(1, np.uint8), dtype=np.uint8)
        h = self._prepare(_p(buf), buf.size, _p(f), _p(m), m.size, _p(sc), sc.size if scales is not None else 0,
                          k, block, n)
        if not h:
            raise OracleError(INVALID, "prepare")

        class Prepared:
            def __init__(self):
                self.h, self.n = h, n
                self.out = np.zeros(max(n, 1), np.uint16)

            def decode(self):
                rc = lib._dec_prepared(self.h, _p(self.out))
                if rc:
                    raise OracleError(rc, "decompress")
                return self.out[: self.n]

            def __del__(self):
                lib._free_prepared(self.h)

        return Prepared()

    def entropy_report(self, values):
        v = np.ascontiguousarray(values, dtype=np.uint16)
        out = np.zeros(5, np.float64)
        self._entropy(_p(v), v.size, _p(out))
        return out

    def write_nzt_lossy(self, values, shape, k: int, block: int = 512) -> bytes:
        v = np.ascontiguousarray(values, dtype=np.uint16)
        dims = np.asarray(shape, dtype=np.uint64)
        out = np.zeros(v.size * 4 + 4096, np.uint8)
        n = self._nzt_lossy(_p(v), _p(dims), dims.size, k, block, _p(out), out.size)
        if n < 0:
            raise OracleError(n, "write_nzt")
        return out[:n].tobytes()

    def read_nzt(self, data: bytes, max_n: int):
        """The reference's read_nzt + decompress: (status, values); status 0 or
        the exception class code (-2 truncated, -3 desync, -4 length/format,
        -6 table, -7 checksum)."""
        buf = np.frombuffer(data, np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
        out = np.zeros(max(max_n, 1), np.uint16)
        n = np.zeros(1, np.uint64)
        rc = self._read_nzt(_p(buf), len(data), _p(out), out.size, _p(n))
        return rc, out[: int(n[0])]

    def write_nzt_lossless(self, values, shape) -> bytes:
        v = np.ascontiguousarray(values, dtype=np.uint16)
        dims = np.asarray(shape, dtype=np.uint64)
        out = np.zeros(v.size * 4 + 4096, np.uint8)
        n = self._nzt(_p(v), _p(dims), dims.size, _p(out), out.size)
        if n < 0:
            raise OracleError(n, "write_nzt")
        return out[:n].tobytes()


def footprint_total(stream_len: int, mantissa_bytes: int, scale_bytes: int = 0, ndim: int = 1) -> int:
    """footprint(blob).total(), tensorstore.hpp:242-283 (header :259-261)."""
    header = 4 + 1 + 1 + 4 + 1 + 8 * ndim + 4 + 8 + 8 + 4
    return stream_len + mantissa_bytes + scale_bytes + 512 + header


def exponent_counts(values) -> np.ndarray:
    v = np.asarray(values, dtype=np.uint16)
    return np.bincount(((v >> 7) & 0xFF).astype(np.int64), minlength=256).astype(np.uint64)
