"""One Llama-3-8B layer (7 projections + 2 norms, 218,112,000 elements) as one
grouped decode launch, timed with CUDA events (L2 flushed between launches).
Dev tool for A/B runs of library variants (NZGPU_LIB=libnzgpu_<tag>.so).
usage: layerbench.py [precisions e.g. 7,3,0] [iters] [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz

H, F, KV = 4096, 14336, 1024
SHAPES = [(H, H), (KV, H), (KV, H), (H, H), (F, H), (F, H), (H, F), (H,), (H,)]


def main():
    precs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "7").split(",")]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    g = torch.Generator(device="cuda")
    ws = []
    for i, s in enumerate(SHAPES):
        n = int(np.prod(s))
        if len(s) == 1:
            ws.append(torch.ones(n, dtype=torch.bfloat16, device="cuda"))
        else:
            g.manual_seed(1000 + i)
            ws.append((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for prec in precs:
        blobs = nz.DeviceBlob.compress_batch(ws, precision=prec, interval=K)
        outs = [torch.empty(b.n, dtype=torch.bfloat16, device="cuda") for b in blobs]
        plan = nz.DecodePlan(blobs, outs)
        for _ in range(3):
            plan.launch()
        plan.status()
        if prec == 7:
            assert os.environ.get("NZ_NOVERIFY") or all(torch.equal(o.view(torch.int16), w.view(torch.int16)) for o, w in zip(outs, ws))
        t = []
        for _ in range(iters):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.launch()
            b.record()
            b.synchronize()
            t.append(a.elapsed_time(b) * 1e-3)
        plan.status()
        algo = sum(int(bb.info.payload_bytes) + 2 * bb.n for bb in blobs)
        med = float(np.median(t))
        print(json.dumps({"lib": os.environ.get("NZGPU_LIB", "libnzgpu.so"), "prec": prec, "us": round(med * 1e6, 1),
                          "min_us": round(min(t) * 1e6, 1), "gbs": round(algo / med / 1e9, 1),
                          "frac": round(algo / med / 6545.6e9, 4), "kernel": plan.kernel}), flush=True)
        plan.free()
        for bb in blobs:
            bb.free()


main()
