"""Compress throughput (dev tool): Llama-3-8B-shaped tensors compressed
one tensor per call vs batched (nzgpu_compress_batch).  GB/s of bf16 in.
usage: compress_bench.py [layers] [precision]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_20650_b200 as nz

LAYER = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336),
         (4096,), (4096,)]


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    g = torch.Generator(device="cuda")
    ts = []
    for l in range(layers):
        for i, sh in enumerate(LAYER):
            n = sh[0] * (sh[1] if len(sh) > 1 else 1)
            if len(sh) == 1:
                ts.append(torch.ones(n, dtype=torch.bfloat16, device="cuda"))
            else:
                g.manual_seed(1000 * l + i)
                ts.append((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    nbytes = 2 * sum(t.numel() for t in ts)
    res = {"layers": layers, "precision": prec, "bf16_bytes": nbytes}

    def timed(fn, reps=3):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            for b in out:
                b.free()
            best = dt if best is None else min(best, dt)
        return best

    res["per_tensor_s"] = timed(lambda: [nz.DeviceBlob.compress(t, precision=prec) for t in ts])
    per_layer = lambda: [b for l in range(layers)
                         for b in nz.DeviceBlob.compress_batch(ts[9 * l:9 * l + 9], precision=prec)]
    res["batch_per_layer_s"] = timed(per_layer)
    res["batch_all_s"] = timed(lambda: nz.DeviceBlob.compress_batch(ts, precision=prec))
    for k in ("per_tensor_s", "batch_per_layer_s", "batch_all_s"):
        res[k.replace("_s", "_gbs")] = round(nbytes / res[k] / 1e9, 2)
    if os.environ.get("PROF"):
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for b in nz.DeviceBlob.compress_batch(ts, precision=prec):
                b.free()
            torch.cuda.synchronize()
        for ev in sorted(prof.key_averages(), key=lambda e: -e.device_time_total)[:8]:
            print(f"  {ev.key[:60]:60s} calls={ev.count:4d} total={ev.device_time_total / 1e3:.3f} ms")
    print(json.dumps(res), flush=True)


main()
