"""GPU: seeded random shapes through the host tier -- tensor lengths around
and above the sliced pipeline's 4 Mi-element cut, chunk sizes that are and
are not powers of two, checkpoint strides 64/128, lossy block sizes that do
and do not divide a slice -- each compressed on the GPU, checked byte for
byte against the oracle's compress, and decoded through both host routes
(nzgpu_decompress_host: sliced pipeline into pageable memory; and
nzgpu_decompress_host_batch) against the oracle's decode
(tensorstore.hpp:87-238, ans.hpp:202-347)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


def _cases():
    rng = np.random.default_rng(2410)
    out = []
    for i in range(24):
        n = int(rng.choice([4 << 20, (4 << 20) + 1, 5_000_000 + int(rng.integers(0, 1 << 20)), 9_437_184 - 3]))
        k = int(rng.choice([7, 3, 1, 0]))
        chunk = int(rng.choice([65536, 65536 * 3, 1 << 18, 4096 * 5]))
        interval = int(rng.choice([0, 64, 128]))
        if interval and chunk % interval:
            interval = 64
        block = int(rng.choice([512, 256, 1000, 3, 2048, 777]))
        out.append((i, n, k, chunk, interval, block))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-n{c[1]}-k{c[2]}-S{c[3]}-K{c[4]}-B{c[5]}")
def test_gpu_host_tier_random_shapes(nz, port, case):
    i, n, k, chunk, interval, block = case
    v = port.gaussian_bf16(port.derive(900, i), n, 0.02 if i % 3 else 0.5)
    if k == 7:
        blob = nz.compress_lossless(v, chunk_symbols=chunk, interval=interval)
        f, st, sm = port.compress_lossless(v, chunk)
        assert blob.stream == st and (blob.freqs == f).all() and (blob.signmant == sm).all()
        want = v
        got = nz.decompress_lossless(blob)
    else:
        blob = nz.compress_lossy(v, k, block, chunk_symbols=chunk, interval=interval)
        f, sc, st, pk = port.compress_lossy(v, k, block, chunk)
        assert blob.stream == st and (blob.scales == sc).all() and (blob.signmant == pk).all()
        want = port.decompress_lossy(f, sc, st, pk, k, block, n)
        got = nz.decompress_lossy(blob)
    assert (got == want).all()
    (batched,) = nz.decompress_batch([blob])
    assert (batched == want).all()
