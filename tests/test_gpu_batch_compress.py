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
