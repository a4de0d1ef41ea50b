"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over every hand-written kernel of the codec: split+histogram,
table build, lossy normalise/pack, rANS encode, stream scan/copy, the
persistent decode (single blob and a grouped multi-tensor plan, lossless and
lossy), the tiled decode (NZGPU_KERNEL=tiles), the sequential decode that
rebuilds the side index of a foreign stream, CRC-32 + NZT I/O and the
entropy histogram.  Inputs are small so the instrumented run stays short.
Dev tool:  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2410_20650_b200 as nz
from tests import inputs


def gauss(n, seed, sigma=0.02):
    u1 = (inputs.words(seed, n, 0) >> np.uint64(11)).astype(np.float64) * 2.0**-53 + 2.0**-53
    u2 = (inputs.words(seed, n, n) >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return inputs.f32_to_bf16((sigma * np.sqrt(-2.0 * np.log(u1)) * np.cos(2 * np.pi * u2)).astype(np.float32))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
    v = gauss(n, 1)
    # host tier: compress (K1 K2 K3 K4) + decode (persist or tiles) + sections path
    b = nz.compress_lossless(v)
    assert (nz.decompress_lossless(b) == v).all()
    for k in (0, 1, 3):
        lb = nz.compress_lossy(v, k, 512)
        out = nz.decompress_lossy(lb)
        assert out.size == v.size
    # foreign stream (no side index): K8 sequential decode rebuilds it
    b_noix = nz.LosslessBlob(b.meta, b.freqs, b.stream, b.signmant, None)
    assert (nz.decompress_lossless(b_noix) == v).all()
    # batch host path
    outs = nz.decompress_batch([b, b_noix])
    assert all((o == v).all() for o in outs)
    # NZT (GPU CRC-32) and entropy histogram
    data = nz.write_nzt(b)
    back = nz.read_nzt(data)
    assert back.stream == b.stream
    nz.analyze_tensor(v)
    # device tier: grouped plan over several tensors, lossless and lossy
    import torch

    ts = [torch.from_numpy(gauss(m, 10 + i).view(np.int16)).cuda() for i, m in enumerate([70_001, 4096, 150_000])]
    ts.append(torch.ones(4096, dtype=torch.int16, device="cuda") * 0x3F80)
    for prec in (7, 3):
        blobs = nz.DeviceBlob.compress_batch(ts, precision=prec)
        outs = [torch.empty(t.numel(), dtype=torch.bfloat16, device="cuda") for t in ts]
        plan = nz.DecodePlan(blobs, outs)
        plan.launch()
        plan.status()
        if prec == 7:
            assert all(torch.equal(o.view(torch.int16), t) for o, t in zip(outs, ts))
    print(f"sanitize workload ok (n={n}, kernel={os.environ.get('NZGPU_KERNEL', 'persist')})")


main()
