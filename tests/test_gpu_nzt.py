"""GPU: CRC-32 (crc32.hpp) and the NZT container (tensorstore.hpp:289-477),
SURVEY §8(f) rank 1.  The CRC is computed by the CUDA kernels; files must be
byte-identical to the reference's (golden SHA-256s from make_golden.py) and
reading must raise the reference's exception class for every corruption."""
import hashlib
import os

import numpy as np
import pytest

from tests import golden_cases as G
from tests import inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(b):
    return hashlib.sha256(bytes(b)).hexdigest()


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


LENGTHS = [0, 1, 2, 3, 15, 16, 17, 511, 512, 513, 16383, 16384, 16385, 16384 * 33 + 5, 100000, (1 << 20) + 7]


@pytest.mark.parametrize("n", LENGTHS)
def test_gpu_crc32_matches_oracle(nz, port, n):
    data = inputs.uniform_bytes(n, 1234 + n).tobytes()
    assert nz.crc32(data) == port.crc32(data)


def test_gpu_crc32_known_answers(nz):
    assert nz.crc32(b"") == 0
    assert nz.crc32(b"123456789") == 0xCBF43926  # the CRC-32/IEEE check value
    assert nz.crc32(bytes(16384 * 5)) == __import__("zlib").crc32(bytes(16384 * 5))


def test_gpu_crc32_sections_are_concatenation(nz, port):
    parts = [inputs.uniform_bytes(m, 77 + m).tobytes() for m in (512, 0, 3, 70001, 16384, 1)]
    assert nz.crc32(*parts) == port.crc32(b"".join(parts))


def test_gpu_crc32_device_pointer_unaligned(nz, port):
    import ctypes as C

    import torch

    data = inputs.uniform_bytes(1 << 18, 5)
    t = torch.from_numpy(data).cuda()
    for off in (0, 1, 7, 15, 16, 33):
        out = C.c_uint32()
        rc = nz.nzgpu.lib.nzgpu_crc32(C.c_void_p(t.data_ptr() + off), data.size - off - 3, None, C.byref(out))
        nz.nzgpu.check(rc, "crc32")
        assert out.value == port.crc32(data[off:data.size - 3].tobytes()), off


def test_gpu_crc32_large(nz, port):
    data = inputs.uniform_bytes(64 << 20, 99).tobytes()
    assert nz.crc32(data) == port.crc32(data)


@pytest.mark.parametrize("case", G.nzt_cases(), ids=lambda c: c[0])
def test_gpu_write_nzt_matches_reference(nz, port, golden, case):
    name, gen, shape, k, block = case
    rec = golden["nzt"][name]
    v = gen(port)
    meta = nz.TensorMeta(tuple(shape))
    blob = nz.compress_lossless(v, meta) if k == 7 else nz.compress_lossy(v, k, block, meta)
    data = nz.write_nzt(blob)  # host blob, CRC on the GPU
    assert len(data) == rec["len"] and sha(data) == rec["sha"]
    db = nz.DeviceBlob.compress(__import__("torch").from_numpy(v.view(np.int16)).cuda(), precision=k,
                                block_size=block or 512, meta=meta)
    assert db.to_nzt() == data  # device blob: sections D2H + CRC on the GPU
    # read back: same sections, same decoded values as the reference's read_nzt
    back = nz.read_nzt(data)
    assert tuple(back.meta.shape) == tuple(shape)
    assert back.stream == blob.stream and (np.asarray(back.signmant) == np.asarray(blob.signmant)).all()
    if k == 7:
        assert (nz.decompress_lossless(back) == v).all()
    else:
        want = port.decompress_lossy(blob.freqs, blob.scales, blob.stream, blob.signmant, k, block, v.size)
        assert (nz.decompress_lossy(back) == want).all()


def test_gpu_const16_golden_file(nz):
    with open(os.path.join(HERE, "golden", "const16_k7.nzt"), "rb") as fh:
        data = fh.read()
    blob = nz.read_nzt(data)
    assert (nz.decompress_lossless(blob) == 0x3F80).all() and blob.meta.element_count() == 16
    assert nz.write_nzt(blob) == data


def _corruptions(data: bytes):
    """(label, bytes) variants of a valid file: every header field, every
    section, truncation at every boundary."""
    out = [("bad_magic", b"NZT2" + data[4:]), ("version", data[:4] + b"\x02" + data[5:]),
           ("precision", data[:5] + b"\x05" + data[6:]), ("empty", b""), ("magic_only", data[:4])]
    for cut in (5, 11, 19, 100, 530, len(data) // 2, len(data) - 5, len(data) - 1):
        out.append((f"truncated_{cut}", data[:cut]))
    rng = np.random.default_rng(3)
    for pos in sorted(set(rng.integers(12, len(data), 24).tolist()) | {len(data) - 1, len(data) - 4}):
        b = bytearray(data)
        b[pos] ^= 0x5A
        out.append((f"flip_{pos}", bytes(b)))
    out.append(("trailing", data + b"\x00"))
    return out


@pytest.mark.parametrize("k", [7, 3])
def test_gpu_read_nzt_error_classes_match_reference(nz, port, ref, k):
    """For every corruption the GPU reader and the unmodified reference agree:
    both succeed with the same values, or both raise (ChecksumError vs
    FormatError class)."""
    v = port.gaussian_bf16(31, 5000, 0.02)
    data = ref.write_nzt_lossless(v, [50, 100]) if k == 7 else ref.write_nzt_lossy(v, [50, 100], 3, 64)
    for label, bad in _corruptions(data):
        rrc, rvals = ref.read_nzt(bad, v.size)
        try:
            got = nz.read_nzt(bad)
            vals = nz.decompress_lossless(got) if k == 7 else nz.decompress_lossy(got)
            grc = 0
        except nz.ChecksumError:
            grc = -7
        except nz.FormatError:
            grc = -4
        if rrc == -7:
            assert grc == -7, label
        elif rrc == 0:
            assert grc == 0 and (vals == rvals).all(), label
        else:
            assert grc == -4, (label, rrc)
