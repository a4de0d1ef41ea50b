"""A/B of the two decode schedules (persistent vs tiles) in one process,
interleaved so both see the same clocks/L2 state.  Dev tool.
usage: ab.py [n] [precision] [K] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz
from paper_2410_20650_b200 import nzgpu as N


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 218112000
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    torch.manual_seed(0)
    w = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
    blob = nz.DeviceBlob.compress(w, precision=prec, interval=K)
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    plan = nz.DecodePlan([blob], [out])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    algo = blob.info.payload_bytes + 2 * n
    res = {0: [], 1: []}
    for r in range(rounds + 3):
        for kern in (0, 1):
            N.lib.nzgpu_set_decode_kernel(kern)
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            plan.launch()
            b.record()
            b.synchronize()
            if r >= 3:
                res[kern].append(a.elapsed_time(b) * 1e-3)
            if prec == 7 and r == 0:
                plan.status()
                assert torch.equal(out.view(torch.int16), w.view(torch.int16)), f"kernel {kern} mismatch"
    plan.status()
    for kern, name in ((0, "persist"), (1, "tiles")):
        t = np.array(res[kern])
        print(f"{name:8s} n={n} prec={prec} K={K} median={np.median(t)*1e6:.1f}us min={t.min()*1e6:.1f}us "
              f"GB/s(med)={algo/np.median(t)/1e9:.1f} frac={algo/np.median(t)/6545.6e9:.3f}", flush=True)


main()
