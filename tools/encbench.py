"""Compress timing (dev tool): median wall time of DeviceBlob.compress.
usage: encbench.py [n] [precision] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 58720256
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    torch.manual_seed(0)
    w = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b = nz.DeviceBlob.compress(w, precision=prec)
        torch.cuda.synchronize()
        if r:
            ts.append(time.perf_counter() - t0)
        b.free()
    t = float(np.median(ts))
    if os.environ.get("PROF"):
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                nz.DeviceBlob.compress(w, precision=prec).free()
            torch.cuda.synchronize()
        for ev in sorted(prof.key_averages(), key=lambda e: -e.device_time_total)[:6]:
            print(f"  {ev.key[:60]:60s} calls={ev.count:4d} avg={ev.device_time_total / max(ev.count, 1) / 1e3:.3f} ms")
    print(f"compress n={n} prec={prec} median={t*1e3:.2f} ms  {2*n/t/1e9:.1f} GB/s of bf16 in", flush=True)


main()
