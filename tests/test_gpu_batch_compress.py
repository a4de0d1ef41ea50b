"""GPU: batched compress (nzgpu_compress_batch) -- one encode launch over
the chunks of many tensors.  Every blob must be byte-identical to the
single-tensor path and to the oracle (compress_lossless / compress_lossy,
tensorstore.hpp:87-213), including the side index, for mixed sizes,
single-symbol tables, lossy precisions and batch splits; errors leave no
blobs behind."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


def _tensors(port):
    ns = [1, 15, 4096, 65535, 65536, 65537, 70001, 1 << 20, 3 * 65536 + 777]
    ts = [port.gaussian_bf16(port.derive(7, i), n, 0.02 if i % 2 else 0.3) for i, n in enumerate(ns)]
    ts.append(np.full(4096, 0x3F80, np.uint16))  # RMSNorm weight: single-symbol table
    ts.append(np.arange(65536, dtype=np.uint32).astype(np.uint16))  # every pattern incl. NaN/Inf
    return ts


def _dev(ts):
    import torch

    return [torch.from_numpy(t.view(np.int16)).cuda() for t in ts]


@pytest.mark.parametrize("split", [1 << 40, 100000])
def test_gpu_compress_batch_lossless_matches_single_and_oracle(nz, port, split):
    import torch

    ts = _tensors(port)
    dev = _dev(ts)
    batch = nz.DeviceBlob.compress_batch(dev, max_batch_elements=split)
    assert len(batch) == len(ts)
    for b, d, t in zip(batch, dev, ts):
        one = nz.DeviceBlob.compress(d)
        hb, h1 = b.to_host(), one.to_host()
        assert hb.stream == h1.stream and hb.index == h1.index
        assert (hb.freqs == h1.freqs).all() and (hb.signmant == h1.signmant).all()
        f, s, sm = port.compress_lossless(t)
        assert hb.stream == s and (hb.freqs == f).all() and (hb.signmant == sm).all()
        out = b.decompress()
        assert (out.view(torch.int16).cpu().numpy().view(np.uint16) == t).all()


@pytest.mark.parametrize("k", [0, 1, 3])
def test_gpu_compress_batch_lossy_matches_oracle(nz, port, k):
    import torch

    ts = [t for t in _tensors(port)[:-1]]  # lossy rejects NaN/Inf
    dev = _dev(ts)
    batch = nz.DeviceBlob.compress_batch(dev, precision=k, block_size=512)
    for b, t in zip(batch, ts):
        f, sc, s, pk = port.compress_lossy(t, k, 512)
        h = b.to_host()
        assert h.stream == s and (h.freqs == f).all() and (h.scales == sc).all() and (h.signmant == pk).all()
        want = port.decompress_lossy(f, sc, s, pk, k, 512, t.size)
        assert (b.decompress().view(torch.int16).cpu().numpy().view(np.uint16) == want).all()


def test_gpu_compress_batch_plan_decode(nz, port):
    """A batch-compressed layer decodes through one grouped plan launch."""
    import torch

    ts = [port.gaussian_bf16(port.derive(11, i), n, 0.02) for i, n in enumerate([1 << 20, 1 << 18, 1 << 18, 1 << 20])]
    ts.append(np.full(4096, 0x3F80, np.uint16))
    batch = nz.DeviceBlob.compress_batch(_dev(ts))
    outs = [torch.empty(t.size, dtype=torch.bfloat16, device="cuda") for t in ts]
    plan = nz.DecodePlan(batch, outs)
    plan.launch()
    plan.status()
    for o, t in zip(outs, ts):
        assert (o.view(torch.int16).cpu().numpy().view(np.uint16) == t).all()


def test_gpu_compress_batch_errors(nz, port):
    import torch

    good = port.gaussian_bf16(1, 70000, 0.02)
    bad = good.copy()
    bad[12345] = 0x7FC0  # NaN: compress_lossy throws NonFiniteError (tensorstore.hpp:153-157)
    with pytest.raises(nz.NonFiniteError):
        nz.DeviceBlob.compress_batch(_dev([good, bad, good]), precision=3)
    with pytest.raises(ValueError):
        nz.DeviceBlob.compress_batch(_dev([good, np.zeros(0, np.uint16)]))
    # the library stays usable after a failed batch
    b = nz.DeviceBlob.compress_batch(_dev([good]))[0]
    assert (b.decompress().view(torch.int16).cpu().numpy().view(np.uint16) == good).all()


@pytest.mark.parametrize("chunk,interval", [(65536, 128), (3 * 4096, 128), (131072, 0), (1 << 14, 64), (2560, 64),
                                            (100000, 0)])
def test_gpu_compress_batch_chunk_and_interval(nz, port, chunk, interval):
    """Non-default chunk sizes S and checkpoint strides K, including an S no
    stride divides (100000: reference framing, sequential decode, no index)
    and S/K = 40 (2560/64: 32-sub-range warp units straddle chunks, so the
    index's position scan restarts mid-unit)."""
    import torch

    ts = [port.gaussian_bf16(port.derive(21, i), n, 0.02) for i, n in enumerate([5, 70001, 3 * 131072 + 9, 1 << 20])]
    batch = nz.DeviceBlob.compress_batch(_dev(ts), chunk_symbols=chunk, interval=interval)
    for b, d, t in zip(batch, _dev(ts), ts):
        f, s, sm = port.compress_lossless(t, chunk)
        h = b.to_host()
        assert h.stream == s and (h.freqs == f).all() and (h.signmant == sm).all()
        one = nz.DeviceBlob.compress(d, chunk_symbols=chunk, interval=interval).to_host()
        assert one.stream == h.stream and one.index == h.index
        assert (b.decompress().view(torch.int16).cpu().numpy().view(np.uint16) == t).all()


def test_gpu_compress_batch_wide_launch_matches_oracle(nz, port):
    """Enough chunks (>= 600 encoder CTAs) for the byte-queue encoder
    variant; spot-check chunks of every tensor against the oracle's coder."""
    import torch

    # 24 tensors x 820 chunks = 19,680 chunks = 615 CTAs of 32 chains
    g = torch.Generator(device="cuda")
    ts = []
    for i in range(24):
        g.manual_seed(i)
        ts.append((torch.randn(820 * 65536, device="cuda", generator=g) * (0.02 if i % 3 else 0.5)).to(torch.bfloat16))
    batch = nz.DeviceBlob.compress_batch(ts)
    for i in (0, 7, 23):
        v = ts[i].view(torch.int16).cpu().numpy().view(np.uint16)
        f, s, sm = port.compress_lossless(v)
        h = batch[i].to_host()
        assert h.stream == s and (h.freqs == f).all()
        assert torch.equal(batch[i].decompress().view(torch.int16), ts[i].view(torch.int16))


def test_gpu_pool_reuse_and_trim(nz, port):
    """Blob sections come from the library's stream-ordered pool: freed blob
    memory is reused by the next compress (same results), and
    nzgpu_trim_device_pool hands unused pool memory back to the driver."""
    import torch

    t = port.gaussian_bf16(31, 3 * 65536 + 5, 0.02)
    d = torch.from_numpy(t.view(np.int16)).cuda()
    first = nz.DeviceBlob.compress(d).to_host()
    for _ in range(5):
        b = nz.DeviceBlob.compress(d)
        h = b.to_host()
        assert h.stream == first.stream and h.index == first.index
        b.free()
    assert nz.nzgpu.lib.nzgpu_trim_device_pool() == 0
    b = nz.DeviceBlob.compress(d)
    assert (b.decompress().view(torch.int16).cpu().numpy().view(np.uint16) == t).all()


def test_gpu_export_chunks_matches_serialized_export(nz, port):
    """nzgpu_blob_export_chunks (the drop-in's AnsChunk export) hands out the
    same bytes as nzgpu_blob_export: every chunk payload equals its slice of
    the serialized stream (ans.hpp:306-316), and the planes and side index
    are identical -- for tensors below and above the 4 MiB staging cutoff
    and across 32 MiB staging slices (the chunk scatter crosses slices)."""
    import ctypes as C

    N = nz.nzgpu
    for n, k in ((70001, 7), (1 << 22, 3), (40_000_000, 7)):
        v = port.gaussian_bf16(port.derive(71, n), n, 0.02)
        blob = nz.compress_lossless(v) if k == 7 else nz.compress_lossy(v, k, 512)
        db = nz.DeviceBlob.from_host(blob)
        try:
            i = db.info
            want = db.to_host()
            nc = int(i.num_chunks)
            lens = np.zeros(nc, np.uint32)
            nsyms = np.zeros(nc, np.uint32)
            assert N.lib.nzgpu_blob_chunks(db.handle, lens.ctypes.data, nsyms.ctypes.data) == 0
            bufs = [np.zeros(max(int(x), 1), np.uint8) for x in lens]
            ptrs = (C.c_void_p * nc)(*[b.ctypes.data for b in bufs])
            freqs = np.zeros(256, np.uint16)
            mant = np.zeros(max(int(i.mantissa_len), 1), np.uint8)
            scales = np.zeros(max(int(i.scales_len), 1), np.uint8)
            index = np.zeros(max(int(i.index_len), 1), np.uint8)
            assert N.lib.nzgpu_blob_export_chunks(db.handle, freqs.ctypes.data, ptrs, mant.ctypes.data,
                                                  scales.ctypes.data, index.ctypes.data) == 0
            stream = want.stream
            pos = 4
            for c in range(nc):
                assert int.from_bytes(stream[pos:pos + 4], "little") == nsyms[c]
                assert int.from_bytes(stream[pos + 4:pos + 8], "little") == lens[c]
                pos += 8
                assert bufs[c][: lens[c]].tobytes() == stream[pos:pos + int(lens[c])], c
                pos += int(lens[c])
            assert pos == len(stream)
            assert (freqs == want.freqs).all()
            assert (mant[: i.mantissa_len] == want.signmant).all()
            if k != 7:
                assert (scales[: i.scales_len] == want.scales).all()
            assert index[: i.index_len].tobytes() == want.index
        finally:
            db.free()
