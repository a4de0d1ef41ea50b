"""GPU parity: the CUDA path (through the C ABI) against the reference's
frozen outputs (tests/golden/golden.json, made from the unmodified
reference) and against the C oracle on the same seeded inputs.  Bit-exact
everywhere: streams, tables, sign/mantissa planes, scales, decoded bf16."""
import hashlib

import numpy as np
import pytest

from tests import golden_cases as G
from tests import inputs

pytestmark = pytest.mark.gpu


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


# ----------------------------------------------------------- lossless ------
@pytest.mark.parametrize("case", G.lossless_cases(), ids=lambda c: c[0])
def test_gpu_lossless_matches_reference(nz, port, golden, case):
    name, gen, chunk, _ = case
    rec = golden["lossless"][name]
    v = gen(port)
    blob = nz.compress_lossless(v, chunk_symbols=chunk)
    assert blob.freqs.tobytes().hex() == rec["freqs"]
    assert len(blob.stream) == rec["stream_len"] and sha(blob.stream) == rec["stream_sha"]
    assert sha(blob.signmant) == rec["signmant_sha"]
    assert nz.footprint(blob).total() == rec["footprint"]
    back = nz.decompress_lossless(blob)
    assert (back == v).all()


@pytest.mark.parametrize("case", [c for c in G.lossless_cases() if c[2] == 65536], ids=lambda c: c[0])
def test_gpu_decodes_reference_produced_streams(nz, port, case):
    """Streams from the CPU path carry no side index: the GPU rebuilds it
    (sequential validation, ans.hpp:229-256) and then runs the tiled decoder."""
    name, gen, chunk, _ = case
    v = gen(port)
    freqs, stream, sm = port.compress_lossless(v, chunk)
    blob = nz.LosslessBlob(nz.TensorMeta((v.size,)), freqs, stream, sm)
    assert (nz.decompress_lossless(blob) == v).all()


@pytest.mark.parametrize("interval", [64, 128])
def test_gpu_checkpoint_intervals(nz, port, interval):
    v = port.gaussian_bf16(123, 3 * 65536 + 777, 0.02)
    blob = nz.compress_lossless(v, interval=interval)
    f, s, sm = port.compress_lossless(v)
    assert blob.stream == s and (blob.signmant == sm).all()
    assert (nz.decompress_lossless(blob) == v).all()
    # compact side index: 56-byte header + 6 bytes per sub-range + 4 per unit
    nsub = -(-v.size // interval)
    assert len(blob.index) == 56 + 6 * nsub + 4 * (-(-nsub // 32))
    assert (len(blob.index) - 56) / v.size < (0.0959 if interval == 64 else 0.0480)


@pytest.mark.parametrize("interval", [64, 128])
@pytest.mark.parametrize("k", [7, 3])
def test_gpu_sliced_host_decode_intervals(nz, port, interval, k):
    """The sliced host pipeline (pageable output, >= 4 Mi elements) at both
    checkpoint strides, lossless and lossy: slices are whole chunks, warp
    units (32 K symbols) and lossy blocks."""
    v = port.gaussian_bf16(321 + interval, 5_000_003, 0.02)
    if k == 7:
        blob = nz.compress_lossless(v, interval=interval)
        assert (nz.decompress_lossless(blob) == v).all()
    else:
        blob = nz.compress_lossy(v, k, 512, interval=interval)
        f, sc, st, pk = port.compress_lossy(v, k, 512)
        assert (nz.decompress_lossy(blob) == port.decompress_lossy(f, sc, st, pk, k, 512, v.size)).all()


def test_gpu_interval_256_rejected(nz, port):
    """The decoder's checkpoint strides are 64 and 128 symbols (a unit of
    32 sub-ranges then spans <= 31 * (1.5 K + 2) bytes: 16-bit offsets)."""
    v = port.gaussian_bf16(123, 70001, 0.02)
    with pytest.raises(ValueError):
        nz.compress_lossless(v, interval=256)


@pytest.mark.parametrize("what", ["state", "offset", "base"])
def test_gpu_corrupt_index_is_a_format_error(nz, port, what):
    """A damaged side index (not part of the reference format) must surface
    as the reference's FormatError -- every sub-range has to land exactly on
    the next one's state and position -- never as a wrong decode."""
    v = port.gaussian_bf16(77, 1 << 20, 0.02)
    blob = nz.compress_lossless(v)
    ix = bytearray(blob.index)
    nsub = (1 << 20) // 64
    units = nsub // 32
    j = 12345  # a sub-range in the middle of a chunk (chunk 12, not its first)
    if what == "state":
        off = 56 + 4 * j
        ix[off] ^= 0x40
    elif what == "offset":
        off = 56 + 4 * nsub + 4 * units + 2 * j
        ix[off] = (ix[off] + 3) & 0xFF
    else:
        off = 56 + 4 * nsub + 4 * (j // 32)
        ix[off] ^= 0x08
    bad = nz.LosslessBlob(blob.meta, blob.freqs, blob.stream, blob.signmant, index=bytes(ix))
    with pytest.raises(nz.FormatError):
        nz.decompress_batch([bad])


@pytest.mark.parametrize("dist", ["gaussian", "uniform", "laplace"])
def test_gpu_chunk_sweep_streams_match_oracle(nz, port, dist):
    """C5: chunk sizes 64 Ki .. 4 Mi symbols on the three weight
    distributions of the sweep -- the GPU stream must be the oracle's byte for
    byte (so the ratio is the reference's), and decode back exactly."""
    import math

    n = 1 << 22
    if dist == "gaussian":
        v = port.gaussian_bf16(5, n, 0.02)
    elif dist == "uniform":
        v = inputs.bf16_uniform(n, 7, math.sqrt(3.0) * 0.02)
    else:
        v = inputs.bf16_laplace(n, 11, 0.02 / math.sqrt(2.0))
    for S in (1 << 16, 1 << 18, 1 << 20, 1 << 22):
        blob = nz.compress_lossless(v, chunk_symbols=S)
        f, s, sm = port.compress_lossless(v, S)
        assert blob.stream == s and (blob.freqs == f).all(), S
        assert (nz.decompress_lossless(blob) == v).all(), S


def test_gpu_c1_headline_tensor(nz, port, golden):
    rec = golden["c1_4096sq_seed42"]
    v = port.gaussian_bf16(42, 4096 * 4096)
    blob = nz.compress_lossless(v, nz.TensorMeta((4096, 4096)))
    assert len(blob.stream) == rec["stream_len"] and sha(blob.stream) == rec["stream_sha"]
    assert nz.footprint(blob).total() == rec["footprint"]
    assert round(nz.ratio(blob), 6) == round(rec["ratio"], 6)
    assert (nz.decompress_lossless(blob) == v).all()
    for k in (0, 1, 3):
        lb = nz.compress_lossy(v, k, 512)
        r = rec[f"lossy_k{k}"]
        assert sha(lb.stream) == r["stream_sha"] and sha(lb.signmant) == r["packed_sha"]
        assert sha(lb.scales) == r["scales_sha"]


# ----------------------------------------------------------- coder ---------
@pytest.mark.parametrize("case", G.coder_cases(), ids=lambda c: c[0])
def test_gpu_coder_matches_reference(nz, golden, case):
    name, gen, _ = case
    rec = golden["coder"][name]
    x = gen()
    freqs = nz.build_table(inputs.counts_of(x))
    assert freqs.tobytes().hex() == rec["freqs"]
    stream = nz.ans_encode(x, freqs)
    assert len(stream) == rec["stream_len"] and sha(stream) == rec["stream_sha"]
    assert (nz.ans_decode(stream, freqs, x.size) == x).all()


def test_gpu_tables_match_reference(nz, golden):
    for name, counts in G.table_cases():
        assert nz.build_table(counts).tobytes().hex() == golden["tables"][name], name


# ----------------------------------------------------------- lossy ---------
@pytest.mark.parametrize("case", G.lossy_cases(), ids=lambda c: c[0])
def test_gpu_lossy_matches_reference(nz, port, golden, case):
    name, gen, k, block, _ = case
    rec = golden["lossy"][name]
    v = gen(port)
    blob = nz.compress_lossy(v, k, block)
    assert blob.freqs.tobytes().hex() == rec["freqs"]
    assert sha(blob.scales) == rec["scales_sha"]
    assert len(blob.stream) == rec["stream_len"] and sha(blob.stream) == rec["stream_sha"]
    assert sha(blob.signmant) == rec["packed_sha"]
    assert nz.footprint(blob).total() == rec["footprint"]
    back = nz.decompress_lossy(blob)
    assert sha(back) == rec["decoded_sha"]


@pytest.mark.parametrize("block", [256, 512, 1024, 2048, 4096, 1 << 16])
@pytest.mark.parametrize("k", [0, 1, 3])
def test_gpu_lossy_pow2_blocks_match_oracle(nz, port, k, block):
    """Power-of-two B >= 256: the decoder loads a unit's scale bytes once
    (8/4/2/1 bytes per 2048-element unit) -- every B class, partial last
    units and tensors shorter than one block, against the oracle."""
    for i, n in enumerate([5 * 2048 + 7, 3 * 65536 + 1000, 300]):
        v = port.gaussian_bf16(port.derive(77, 10 * k + i), n, 0.02 if i else 0.7)
        blob = nz.compress_lossy(v, k, block)
        f, sc, st, pk = port.compress_lossy(v, k, block)
        assert blob.stream == st and (blob.scales == sc).all() and (blob.signmant == pk).all()
        want = port.decompress_lossy(f, sc, st, pk, k, block, n)
        assert (nz.decompress_lossy(blob) == want).all()


@pytest.mark.parametrize("block", [256, 512, 1024, 2048])
@pytest.mark.parametrize("k", [0, 1, 3])
def test_gpu_lossy_fused_blocks_random_patterns(nz, port, k, block):
    """The fused normalise/histogram/pack kernel (full blocks of B = 256 ..
    2048) on arbitrary finite bit patterns: subnormals, exponent-254 carries,
    both signs, maxima anywhere in the block, plus a ragged last block that
    takes the three-kernel path."""
    rng = np.random.default_rng(1000 * k + block)
    n = 4 * 2048 + 300
    v = rng.integers(0, 1 << 16, n, dtype=np.uint32).astype(np.uint16)
    v[(v & 0x7F80) == 0x7F80] ^= 0x0080  # exponent 255 -> 254
    v[:block] = (v[:block] & 0x807F) | 0x7F00  # a block of exponent-254 values
    blob = nz.compress_lossy(v, k, block)
    f, sc, st, pk = port.compress_lossy(v, k, block)
    assert (blob.scales == sc).all() and (blob.signmant == pk).all()
    assert (blob.freqs == f).all() and blob.stream == st
    assert (nz.decompress_lossy(blob) == port.decompress_lossy(f, sc, st, pk, k, block, n)).all()


@pytest.mark.parametrize("block", [256, 2048])
def test_gpu_lossy_fused_rejects_nonfinite(nz, port, block):
    """A NaN or Inf inside a full block fails the whole call
    (tensorstore.hpp:153-157), as it does in a ragged block."""
    v = port.gaussian_bf16(5, 3 * block, 0.02)
    for bad in (0x7FC1, 0xFF80, 0x7F80):
        w = v.copy()
        w[block + 77] = bad
        with pytest.raises(nz.NonFiniteError):
            nz.compress_lossy(w, 3, block)


@pytest.mark.parametrize("k", [0, 1, 3])
def test_gpu_lossy_elementwise_exhaustive(nz, port, k):
    """Every finite bf16 pattern x every scale byte (65,280 x 256 pairs)
    against the oracle's double-precision restatement."""
    pats = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    pats = pats[(pats & 0x7F80) != 0x7F80]
    vals = np.tile(pats, 256)
    scales = np.repeat(np.arange(256, dtype=np.uint8), pats.size)
    got = nz.lossy_roundtrip(vals, scales, k)
    want = port.lossy_roundtrip_many(vals, scales, k)
    assert (got == want).all(), int((got != want).sum())


@pytest.mark.parametrize("k", [0, 1, 3])
@pytest.mark.parametrize("variant", ["fast", "wide_scales", "exp255"])
@pytest.mark.parametrize("kernel", [0, 1])
def test_gpu_lossy_decode_merge_exhaustive(nz, port, k, variant, kernel):
    """Every (scale byte, exponent, packed item) triple through the decode
    kernels' merge (block b holds every (exponent, item) pair under scale b).
    'fast' takes the bf16x2 multiply; a scale byte >= 128 or a table that can
    decode exponent 255 (Inf/NaN payloads) must take the float path and still
    match the oracle bit for bit."""
    import torch

    ne = 256 if variant == "exp255" else 255
    ns = 256 if variant == "wide_scales" else 128
    w = 1 << (k + 1)
    e = np.tile(np.arange(ne, dtype=np.uint8), w)
    it = np.repeat(np.arange(w, dtype=np.uint8), ne)
    B = e.size
    exps, items = np.tile(e, ns), np.tile(it, ns)
    scales = np.arange(ns, dtype=np.uint8)
    n = exps.size
    freqs = port.build_table(np.bincount(exps, minlength=256).astype(np.uint64))
    stream = port.encode_stream(exps, freqs)
    packed = port.pack(items >> k, items & ((1 << k) - 1), k)
    want = port.decompress_lossy(freqs, scales, stream, packed, k, B, n)
    blob = nz.LossyBlob(nz.TensorMeta((n,)), k, B, scales, freqs, stream, packed)
    nz.nzgpu.lib.nzgpu_set_decode_kernel(kernel)
    try:
        got = nz.DeviceBlob.from_host(blob).decompress().view(torch.int16).cpu().numpy().view(np.uint16)
        host = nz.decompress_lossy(blob)
    finally:
        nz.nzgpu.lib.nzgpu_set_decode_kernel(0)
    assert (got == want).all(), int((got != want).sum())
    assert (host == want).all(), int((host != want).sum())


def test_gpu_lossy_decodes_reference_produced_blobs(nz, port):
    v = port.gaussian_bf16(31, 200003, 0.02)
    for k, B in ((0, 512), (1, 7), (3, 64)):
        f, sc, st, pk = port.compress_lossy(v, k, B)
        blob = nz.LossyBlob(nz.TensorMeta((v.size,)), k, B, sc, f, st, pk)
        assert (nz.decompress_lossy(blob) == port.decompress_lossy(f, sc, st, pk, k, B, v.size)).all()


def test_gpu_pack_unpack_matches_oracle(nz, port):  # test_bitfloat.cpp:103-173
    assert nz.pack_signed_mantissas([1, 0, 1, 0, 1, 0, 1, 0], [0] * 8, 0).tolist() == [0xAA]
    assert nz.pack_signed_mantissas([0, 1], [0b101, 0b001], 3).tolist() == [0x59]
    w = inputs.words(19, 2 * 100003)
    for k in (0, 1, 3, 7):
        for n in (1, 3, 17, 100, 257, 100003):
            s = (w[:n] & np.uint64(1)).astype(np.uint8)
            m = ((w[n:2 * n] >> np.uint64(5)) & np.uint64((1 << k) - 1)).astype(np.uint8)
            packed = nz.pack_signed_mantissas(s, m, k)
            assert (packed == port.pack(s, m, k)).all()
            s2, m2 = nz.unpack_signed_mantissas(packed, k, n)
            assert (s2 == s).all() and (m2 == m).all()
    with pytest.raises(ValueError):
        nz.pack_signed_mantissas([0], [2], 1)
    with pytest.raises(ValueError):
        nz.unpack_signed_mantissas(np.zeros(0, np.uint8), 3, 5)


# ----------------------------------------------------------- errors --------
def test_gpu_error_contract(nz, port):
    # test_tensorstore.cpp:313-322: meta/stream mismatch and corrupt byte
    v = port.gaussian_bf16(31, 1000, 0.02)
    blob = nz.compress_lossless(v)
    bad_meta = nz.LosslessBlob(nz.TensorMeta((999,)), blob.freqs, blob.stream, blob.signmant[:999])
    with pytest.raises(nz.FormatError):
        nz.decompress_lossless(bad_meta)
    s = bytearray(blob.stream)
    s[-1] ^= 0x10  # final-state byte of the (only) chunk
    with pytest.raises(nz.FormatError):
        nz.decompress_lossless(nz.LosslessBlob(blob.meta, blob.freqs, bytes(s), blob.signmant, blob.index))
    with pytest.raises(nz.FormatError):
        nz.decompress_lossless(nz.LosslessBlob(blob.meta, blob.freqs, bytes(s), blob.signmant))
    # test_ans.cpp:239-249: truncated payload (framing now lies) and tiny payload
    with pytest.raises(nz.FormatError):
        nz.decompress_lossless(nz.LosslessBlob(blob.meta, blob.freqs, blob.stream[:-5], blob.signmant))
    # test_ans.cpp:259-274: trailing bytes
    with pytest.raises(nz.FormatError):
        nz.decompress_lossless(nz.LosslessBlob(blob.meta, blob.freqs, blob.stream + b"\0", blob.signmant))
    # ans.hpp:99-101: table must sum to 4096
    bad = blob.freqs.copy()
    bad[0] += 1
    with pytest.raises(nz.FormatError):
        nz.decompress_lossless(nz.LosslessBlob(blob.meta, bad, blob.stream, blob.signmant))
    # tensorstore.hpp:153-157 / :143-148
    with pytest.raises(nz.NonFiniteError):
        nz.compress_lossy(np.array([0x3F80, 0x7FC1], np.uint16), 3, 512)
    with pytest.raises(nz.NonFiniteError):
        nz.compress_lossy(np.array([0xFF80], np.uint16), 0, 512)
    with pytest.raises(ValueError):
        nz.compress_lossy(np.array([0x3F80], np.uint16), 2, 512)
    with pytest.raises(ValueError):
        nz.compress_lossy(np.array([0x3F80], np.uint16), 3, 0)
    with pytest.raises(ValueError):
        nz.compress_lossless(np.zeros(0, np.uint16))
    # ans.hpp:210-212: symbol with zero frequency
    c = np.zeros(256, np.uint64)
    c[1] = 10
    with pytest.raises(ValueError):
        nz.ans_encode(np.array([1, 2, 1], np.uint8), nz.build_table(c))
    with pytest.raises(ValueError):
        nz.build_table(np.zeros(256, np.uint64))


def test_gpu_corruption_sweep_is_always_detected_or_exact(nz, port):
    """Flip bytes across the payload (stride 37, like the NZT checksum test
    test_tensorstore.cpp:279-299 but without a CRC): every decode either
    raises FormatError or -- if the corruption is invisible to the reference
    too -- returns exactly what the reference decoder returns."""
    v = port.gaussian_bf16(29, 70000, 0.02)
    blob = nz.compress_lossless(v)
    for pos in range(4, len(blob.stream), 37):
        s = bytearray(blob.stream)
        s[pos] ^= 0x40
        try:
            ref = port.decompress_lossless(blob.freqs, bytes(s), blob.signmant, v.size)
        except Exception:
            ref = None
        try:
            got = nz.decompress_lossless(nz.LosslessBlob(blob.meta, blob.freqs, bytes(s), blob.signmant, blob.index))
        except nz.FormatError:
            got = None
        if got is not None:
            assert ref is not None and (got == ref).all(), pos


# ----------------------------------------------------------- device API ----
def test_gpu_device_blob_and_plan(nz, port):
    import torch

    tensors = [port.gaussian_bf16(port.derive(42, i), n, 0.02) for i, n in enumerate([4096, 70000, 1 << 20, 65536 * 3])]
    tensors.append(np.full(4096, 0x3F80, np.uint16))  # RMSNorm weight: single-symbol table
    dev = [torch.from_numpy(t.view(np.int16)).cuda() for t in tensors]
    blobs = [nz.DeviceBlob.compress(d) for d in dev]
    for b, t in zip(blobs, tensors):
        f, s, sm = port.compress_lossless(t)
        h = b.to_host()
        assert h.stream == s and (h.signmant == sm).all() and (h.freqs == f).all()
        out = b.decompress()
        assert (out.view(torch.int16).cpu().numpy().view(np.uint16) == t).all()
    outs = [torch.empty(t.size, dtype=torch.bfloat16, device="cuda") for t in tensors]
    plan = nz.DecodePlan(blobs, outs)
    assert plan.launches == 1
    plan.launch()
    plan.status()
    for o, t in zip(outs, tensors):
        assert (o.view(torch.int16).cpu().numpy().view(np.uint16) == t).all()


def test_gpu_batch_host_decode(nz, port):
    vs = [port.gaussian_bf16(i, 50000 + 1000 * i, 0.02) for i in range(5)]
    blobs = [nz.compress_lossless(v) for v in vs]
    outs = nz.decompress_batch(blobs)
    for o, v in zip(outs, vs):
        assert (o == v).all()
    # more tensors than staging slots, mixed sizes, then release and reuse
    vs = [port.gaussian_bf16(100 + i, n, 0.02) for i, n in enumerate([70000, 3 * 65536 + 5, 1000, 1 << 20] * 5)]
    blobs = [nz.compress_lossless(v) for v in vs]
    for _ in range(2):
        outs = nz.decompress_batch(blobs)
        assert all((o == v).all() for o, v in zip(outs, vs))
        nz.release_host_buffers()


def test_gpu_host_tier_from_concurrent_threads(nz, port):
    """The host tier from several threads at once: per-thread staging (pinned
    ring, device slots), the shared host worker pool and the device pool.
    Large tensors take the sliced pipeline (pageable outputs), compress the
    staged H2D; every result must be exact."""
    import concurrent.futures as cf

    vs = [port.gaussian_bf16(500 + i, n, 0.02) for i, n in enumerate([5_000_000, 9_000_001, 70001, 4_194_304])]
    blobs = [nz.compress_lossless(v) for v in vs]

    def work(i):
        for _ in range(3):
            b = nz.compress_lossless(vs[i])
            assert b.stream == blobs[i].stream and (b.signmant == blobs[i].signmant).all()
            assert (nz.decompress_lossless(blobs[i]) == vs[i]).all()
        return i

    with cf.ThreadPoolExecutor(4) as ex:
        assert sorted(ex.map(work, range(4))) == [0, 1, 2, 3]


def test_gpu_index_window_hint_is_only_a_hint(nz, port):
    """The exported index carries the unit window size (header offset 48).
    A zeroed or implausible hint falls back to a scan and still decodes; an
    understated hint is reported as a FormatError, never a bad decode."""
    import struct

    v = port.gaussian_bf16(5, 1 << 20, 0.02)
    blob = nz.compress_lossless(v)
    ix = bytearray(blob.index)
    (hint,) = struct.unpack_from("<I", ix, 48)
    assert 0 < hint <= 64 * 64 + 64
    for bad in (0, 0xFFFFFFFF):
        struct.pack_into("<I", ix, 48, bad)
        b2 = nz.LosslessBlob(blob.meta, blob.freqs, blob.stream, blob.signmant, index=bytes(ix))
        assert (nz.decompress_batch([b2])[0] == v).all()
    struct.pack_into("<I", ix, 48, 16)
    b3 = nz.LosslessBlob(blob.meta, blob.freqs, blob.stream, blob.signmant, index=bytes(ix))
    with pytest.raises(nz.FormatError):
        nz.decompress_batch([b3])
