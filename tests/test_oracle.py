"""CPU tests of the checker itself: the C restatement (oracle/liboracle.so)
must reproduce the reference's frozen outputs (tests/golden/, made from the
unmodified reference) and, where oracle/_ref is built, the reference itself
on fresh seeded inputs.  Known-answer cases are the reference's own unit
tests (proj/tests/test_bitfloat.cpp, test_ans.cpp, test_tensorstore.cpp)."""
import hashlib
import os

import numpy as np
import pytest

from oracle.oracle import DESYNC, LENGTH, NONFINITE, TRUNCATED, INVALID, BAD_TABLE, OracleError, footprint_total
from tests import golden_cases as G
from tests import inputs

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


# ---------------------------------------------------------------- golden --
@pytest.mark.parametrize("case", G.lossless_cases(), ids=lambda c: c[0])
def test_port_lossless_matches_golden(port, golden, case):
    name, gen, chunk, _ = case
    rec = golden["lossless"][name]
    v = gen(port)
    assert sha(v) == rec["input_sha"]
    freqs, stream, sm = port.compress_lossless(v, chunk)
    assert freqs.tobytes().hex() == rec["freqs"]
    assert len(stream) == rec["stream_len"] and sha(stream) == rec["stream_sha"]
    assert sha(sm) == rec["signmant_sha"]
    if "stream_hex" in rec:
        assert stream.hex() == rec["stream_hex"]
    assert footprint_total(len(stream), v.size) == rec["footprint"]
    assert (port.decompress_lossless(freqs, stream, sm, v.size) == v).all()


@pytest.mark.parametrize("case", G.coder_cases(), ids=lambda c: c[0])
def test_port_coder_matches_golden(port, golden, case):
    name, gen, _ = case
    rec = golden["coder"][name]
    x = gen()
    assert sha(x) == rec["input_sha"]
    freqs = port.build_table(inputs.counts_of(x))
    assert freqs.tobytes().hex() == rec["freqs"]
    stream = port.encode_stream(x, freqs)
    assert len(stream) == rec["stream_len"] and sha(stream) == rec["stream_sha"]
    assert (port.decode_stream(stream, freqs, x.size) == x).all()


@pytest.mark.parametrize("case", G.lossy_cases(), ids=lambda c: c[0])
def test_port_lossy_matches_golden(port, golden, case):
    name, gen, k, block, _ = case
    rec = golden["lossy"][name]
    v = gen(port)
    assert sha(v) == rec["input_sha"]
    freqs, scales, stream, packed = port.compress_lossy(v, k, block)
    assert freqs.tobytes().hex() == rec["freqs"]
    assert sha(scales) == rec["scales_sha"]
    assert len(stream) == rec["stream_len"] and sha(stream) == rec["stream_sha"]
    assert sha(packed) == rec["packed_sha"]
    back = port.decompress_lossy(freqs, scales, stream, packed, k, block, v.size)
    assert sha(back) == rec["decoded_sha"]
    if "scales" in rec:
        assert scales.tolist() == rec["scales"] and back.tolist() == rec["decoded"]


def test_port_tables_match_golden(port, golden):
    for name, counts in G.table_cases():
        assert port.build_table(counts).tobytes().hex() == golden["tables"][name], name


def test_gaussian_entropy_fixture_matches_reference_checked_in_file():
    # proj/tests/golden/gaussian_entropy.csv:1-5 (values copied as numbers, not the file)
    want = {"sign": 1.0, "exponent": 2.54503, "mantissa": 6.97126, "ideal_ratio": 1.52145,
            "exponent_only_ratio": 1.5173}
    with open(os.path.join(HERE, "golden", "gaussian_entropy.csv")) as fh:
        got = {k: float(v) for k, v in (line.strip().split(",") for line in fh if line.strip())}
    assert got == want


def test_const16_nzt_fixture(port):
    # SURVEY probe P3: 587 bytes, CRC ec9e894f, stream 01000000 10000000 04000000 00008000
    data = open(os.path.join(HERE, "golden", "const16_k7.nzt"), "rb").read()
    assert len(data) == 587
    assert data[:4] == b"NZT1"
    assert data[-4:] == bytes.fromhex("ec9e894f")
    # CRC-32 over table | scales | stream | signmant (tensorstore.hpp:352-357)
    table = data[4 + 1 + 1 + 4 + 1 + 8:][:512]
    stream = bytes.fromhex("01000000100000000400000000008000")
    crc = port.crc32(table + stream + bytes([0x00] * 16))
    assert crc.to_bytes(4, "little") == data[-4:]
    assert bytes.fromhex("01000000100000000400000000008000") in data


def test_c1_headline_ratio_fixture(golden):
    rec = golden["c1_4096sq_seed42"]
    assert rec["stream_len"] == 5347963
    assert round(rec["ratio"], 6) == 1.516534
    assert [round(rec[f"lossy_k{k}"]["ratio"], 4) for k in (0, 1, 3)] == [4.3961, 3.4468, 2.4086]


# ------------------------------------------------------- port vs reference --
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_equals_reference_random(port, ref, seed):
    rng = inputs.words(seed, 8)
    n = int(rng[0] % np.uint64(300000)) + 1
    sigma = [0.02, 0.3, 1e-3][seed - 1]
    v = port.gaussian_bf16(int(rng[1]), n, sigma)
    assert (v == ref.gaussian_bf16(int(rng[1]), n, sigma)).all()
    a, b = port.compress_lossless(v), ref.compress_lossless(v)
    assert (a[0] == b[0]).all() and a[1] == b[1] and (a[2] == b[2]).all()
    for k in (0, 1, 3):
        block = int(rng[2 + k] % np.uint64(700)) + 1
        a, b = port.compress_lossy(v, k, block), ref.compress_lossy(v, k, block)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all() and a[2] == b[2] and (a[3] == b[3]).all()
        assert (port.decompress_lossy(*a, k, block, n) == ref.decompress_lossy(*a, k, block, n)).all()


def test_port_equals_reference_tables_random(port, ref):
    w = inputs.words(77, 256 * 400)
    for t in range(400):
        r = w[t * 256:(t + 1) * 256]
        mode = t % 4
        if mode == 0:
            c = r % np.uint64(1000)
        elif mode == 1:
            c = np.where(r % np.uint64(3) == 0, r % np.uint64(1 << 30), np.uint64(0))
        elif mode == 2:
            c = np.where(r % np.uint64(7) == 0, np.uint64(1), r % np.uint64(50))
        else:
            c = (r >> np.uint64(40)) * (r % np.uint64(2))
        c = c.astype(np.uint64)
        if c.sum() == 0:
            c[t % 256] = 1
        assert (port.build_table(c) == ref.build_table(c)).all()


# ------------------------------------------------------------ bitfloat KATs --
def test_from_float_rne(port):  # test_bitfloat.cpp:175-184
    assert port.from_float(1.00390625) == 0x3F80
    assert port.from_float(1.0 + 3.0 / 512.0) == 0x3F81
    assert port.from_float(0.0) == 0 and port.from_float(-0.0) == 0x8000
    nan = port.from_float(float("nan"))
    assert (nan & 0x7F80) == 0x7F80 and (nan & 0x7F)
    assert port.from_float(-5.0) == 0xC0A0  # test_bitfloat.cpp:24-37


def test_round_mantissa_vs_real_valued_rne(port):  # test_bitfloat.cpp:52-88
    for k in (0, 1, 3):
        for m in range(128):
            scaled = m / 2 ** (7 - k)
            fl = np.floor(scaled)
            frac = scaled - fl
            r = fl + (1 if frac > 0.5 or (frac == 0.5 and fl % 2 != 0) else 0)
            want = (0, True) if r >= 2 ** k else (int(r) << (7 - k), False)
            assert port.round_mantissa(m, k) == want
            once = port.round_mantissa(m, k)[0]
            assert port.round_mantissa(once, k) == (once, False)
    assert port.round_mantissa(0b1010110, 3) == (0b1010000, False)
    assert port.round_mantissa(127, 3) == (0, True)
    with pytest.raises(OracleError):
        port.round_mantissa(0, 2)


def test_pack_examples_and_bijection(port):  # test_bitfloat.cpp:103-173
    assert port.pack([1, 0, 1, 0, 1, 0, 1, 0], [0] * 8, 0).tolist() == [0xAA]
    assert port.pack([0, 1], [0b101, 0b001], 3).tolist() == [0x59]
    w = inputs.words(11, 4 * 300)
    for k in (0, 1, 3, 7):
        for n in (1, 3, 17, 100, 257):
            s = (w[:n] & np.uint64(1)).astype(np.uint8)
            m = ((w[n:2 * n] >> np.uint64(3)) & np.uint64((1 << k) - 1)).astype(np.uint8)
            packed = port.pack(s, m, k)
            bits = []
            for i in range(n):
                bits.append(int(s[i]))
                bits += [(int(m[i]) >> b) & 1 for b in range(k - 1, -1, -1)]
            naive = np.zeros((len(bits) + 7) // 8, np.uint8)
            for i, bit in enumerate(bits):
                if bit:
                    naive[i // 8] |= 0x80 >> (i % 8)
            assert (packed == naive).all()
            s2, m2 = port.unpack(packed, k, n)
            assert (s2 == s).all() and (m2 == m).all()
    with pytest.raises(OracleError):
        port.pack([0], [2], 1)
    with pytest.raises(OracleError):
        port.unpack(np.zeros(0, np.uint8), 3, 5)


# ----------------------------------------------------------- coder KATs ----
def test_table_kats(port):  # test_ans.cpp:48-154
    c = np.zeros(256, np.uint64); c[42] = 4096
    assert port.build_table(c)[42] == 4096
    assert (port.build_table(np.full(256, 1000, np.uint64)) == 16).all()
    c = np.zeros(256, np.uint64); c[0] = 3; c[1] = 1
    assert port.build_table(c)[:2].tolist() == [3072, 1024]
    c = np.zeros(256, np.uint64); c[0] = 4095; c[1] = 1
    assert port.build_table(c).tobytes()[:4] == bytes([0xFF, 0x0F, 0x01, 0x00])
    with pytest.raises(OracleError) as e:
        port.build_table(np.zeros(256, np.uint64))
    assert e.value.code == INVALID


def test_coder_error_paths(port):  # test_ans.cpp:231-257
    c = np.zeros(256, np.uint64); c[1] = 10
    t = port.build_table(c)
    with pytest.raises(OracleError) as e:
        port.encode_stream(np.array([1, 2, 1], np.uint8), t)
    assert e.value.code == INVALID
    x = inputs.zipf_bytes(1000, 9)
    t = port.build_table(inputs.counts_of(x))
    p = port.encode_chunk(x, t)
    with pytest.raises(OracleError) as e:
        port.decode_chunk(p[:-5], x.size, t)
    assert e.value.code in (TRUNCATED, DESYNC)
    with pytest.raises(OracleError) as e:
        port.decode_chunk(p[:2], x.size, t)
    assert e.value.code == TRUNCATED
    x = inputs.uniform_bytes(5000, 10)
    t = port.build_table(inputs.counts_of(x))
    p = bytearray(port.encode_chunk(x, t))
    p[-1] ^= 1
    with pytest.raises(OracleError) as e:
        port.decode_chunk(bytes(p), x.size, t)
    assert e.value.code in (TRUNCATED, DESYNC)


def test_stream_framing_errors(port):  # test_ans.cpp:259-274
    x = inputs.zipf_bytes(150000, 12)
    t = port.build_table(inputs.counts_of(x))
    s = port.encode_stream(x, t)
    with pytest.raises(OracleError) as e:
        port.decode_stream(s + b"\0", t, x.size)
    assert e.value.code == LENGTH
    with pytest.raises(OracleError) as e:
        port.decode_stream(s[:-3], t, x.size)
    assert e.value.code == TRUNCATED
    bad = np.zeros(256, np.uint16); bad[0] = 1
    with pytest.raises(OracleError) as e:
        port.decode_stream(s, bad, x.size)
    assert e.value.code == BAD_TABLE


def test_empty_stream(port):  # test_ans.cpp:164-170
    t = port.build_table(np.ones(256, np.uint64))
    s = port.encode_stream(np.zeros(0, np.uint8), t)
    assert s == b"\0\0\0\0"
    assert port.decode_stream(s, t, 0).size == 0


def test_chunks_decode_independently(port):  # test_ans.cpp:220-229
    x = inputs.zipf_bytes(200000, 8)
    t = port.build_table(inputs.counts_of(x))
    p = port.encode_chunk(x[65536:2 * 65536], t)
    assert (port.decode_chunk(p, 65536, t) == x[65536:2 * 65536]).all()


# ---------------------------------------------------------- lossy KATs -----
def test_lossy_known_answers(port):  # test_tensorstore.cpp:104-131, :187-203
    v = inputs.f32_to_bf16(np.array([1.0, 0.5], np.float32))
    for k in (0, 1, 3):
        f, sc, st, pk = port.compress_lossy(v, k, 512)
        assert sc.tolist() == [0]
        assert (port.decompress_lossy(f, sc, st, pk, k, 512, 2) == v).all()
    v = inputs.f32_to_bf16(np.array([-1.75, 0.3], np.float32))
    f, sc, st, pk = port.compress_lossy(v, 0, 512)
    assert sc.tolist() == [96]
    back = port.decompress_lossy(f, sc, st, pk, 0, 512, 2)
    assert back[0] == v[0]
    assert [port.lossy_roundtrip(int(x), 96, 0) for x in v] == back.tolist()
    with pytest.raises(OracleError) as e:
        port.compress_lossy(np.array([0x3F80, 0x7FC1], np.uint16), 3, 512)
    assert e.value.code == NONFINITE
    with pytest.raises(OracleError) as e:
        port.compress_lossy(np.array([0x3F80], np.uint16), 2, 512)
    assert e.value.code == INVALID
    with pytest.raises(OracleError) as e:
        port.compress_lossy(np.array([0x3F80], np.uint16), 3, 0)
    assert e.value.code == INVALID


def test_lossy_fp32_arithmetic_is_exact_vs_double(port):
    """SURVEY probe P5 restated: for every finite bf16 x every scale byte,
    float32 correctly-rounded divide/multiply give the same bf16 as the
    reference's double path (tensorstore.hpp:181, :235).  This is what lets
    the CUDA kernels use __fdiv_rn / __fmul_rn instead of FP64."""
    pats = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    pats = pats[(pats & 0x7F80) != 0x7F80]
    x32 = inputs.bf16_to_f32(pats)
    x64 = x32.astype(np.float64)
    np.seterr(over="ignore")
    for s in range(256):
        c = 1.0 + s / 128.0
        d32 = inputs.f32_to_bf16(x32 / np.float32(c))
        d64 = inputs.f32_to_bf16((x64 / c).astype(np.float32))
        assert (d32 == d64).all(), s
        m32 = inputs.f32_to_bf16(x32 * np.float32(c))
        m64 = inputs.f32_to_bf16((x64 * c).astype(np.float32))
        assert (m32 == m64).all(), s


def test_encoder_exact_division_identity():
    """The CUDA encoder divides by f with q = (x m) >> (31 + l), l = ceil(log2 f),
    m = ceil(2^(31+l)/f) (Granlund-Montgomery for x < 2^31), and forms
    (q << 12) + r + cum as x + q (4096 - f) + cum.  Check it against exact
    division over the encoder domain x in [f<<11, f<<19) at edge bands and a
    dense stride for every f in 1..4096."""
    for f in range(1, 4097):
        l = (f - 1).bit_length()
        m = ((1 << (31 + l)) + f - 1) // f
        assert m < (1 << 32)
        lo, hi = f << 11, min(f << 19, 1 << 31)
        x = np.concatenate([np.arange(lo, min(lo + 4096, hi), dtype=np.uint64),
                            np.arange(max(hi - 4096, lo), hi, dtype=np.uint64),
                            np.arange(lo, hi, max(1, (hi - lo) // 2048), dtype=np.uint64)])
        q = (x * np.uint64(m)) >> np.uint64(31 + l)
        assert (q == x // np.uint64(f)).all(), f
        cum = np.uint64(4096 - f)
        assert ((x + q * np.uint64(4096 - f) + cum) == ((x // np.uint64(f)) << np.uint64(12)) + x % np.uint64(f) + cum).all()




