"""GPU memory-safety checks without compute-sanitizer (closed on this GPU
pool): every decode writes exactly its n bf16 values and nothing around
them.  Outputs sit between guard bands of canary values, for sizes that hit
every boundary case of the kernels (n % 8 tails, partial warp units, partial
chunks, tensors below one unit, one chunk, many chunks), both checkpoint
strides, lossless and lossy, single-tensor and grouped-plan launches, and
both decode schedules; guards must be intact and values equal to the
reference (lossless: the input; lossy: oracle decompress_lossy)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [1, 7, 8, 9, 63, 64, 65, 2047, 2048, 2049, 4095, 4097, 65535, 65536, 65537, 131072 + 13, (1 << 20) + 5]
GUARD = 64  # elements (128 B) of canary on each side
CANARY = 0x7BCD


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


def _guarded(torch, n):
    buf = torch.full((n + 2 * GUARD,), CANARY, dtype=torch.int16, device="cuda")
    return buf, buf[GUARD:GUARD + n]


def _check(torch, buf, n, want, what):
    h = buf.cpu().numpy().view(np.uint16)
    assert (h[:GUARD] == CANARY).all() and (h[GUARD + n:] == CANARY).all(), f"{what}: guard band overwritten"
    assert (h[GUARD:GUARD + n] == want).all(), f"{what}: wrong values"


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("interval", [64, 128])
@pytest.mark.parametrize("k", [7, 3, 0])
def test_gpu_decode_writes_exactly_its_output(nz, port, kernel, interval, k):
    import torch

    N = nz.nzgpu
    N.lib.nzgpu_set_decode_kernel(kernel)
    try:
        vs = [port.gaussian_bf16(port.derive(99, i), n, 0.02) for i, n in enumerate(SIZES)]
        dev = [torch.from_numpy(v.view(np.int16)).cuda() for v in vs]
        blobs = nz.DeviceBlob.compress_batch(dev, precision=k, block_size=512, interval=interval)
        wants = []
        for v, b in zip(vs, blobs):
            if k == 7:
                wants.append(v)
            else:
                f, sc, s, pk = port.compress_lossy(v, k, 512)
                wants.append(port.decompress_lossy(f, sc, s, pk, k, 512, v.size))
        # one launch per blob
        for v, b, want in zip(vs, blobs, wants):
            buf, out = _guarded(torch, v.size)
            b.decompress_into(out)
            b.status()
            _check(torch, buf, v.size, want, f"single n={v.size}")
        # one grouped launch, outputs packed back to back between guards
        bufs = [_guarded(torch, v.size) for v in vs]
        plan = nz.DecodePlan(blobs, [o for _, o in bufs])
        plan.launch()
        plan.status()
        for (buf, _), v, want in zip(bufs, vs, wants):
            _check(torch, buf, v.size, want, f"plan n={v.size}")
    finally:
        N.lib.nzgpu_set_decode_kernel(0)
