"""Compress latency of the single-tensor config (C1: one 4096x4096 bf16
tensor, 256 rANS chunks) and of one Llama-3-8B layer (the bench's per-layer
recompress, nn.hpp:311's cost), host-synchronised wall time around
nzgpu_compress_batch, median of N.  Dev tool for A/B of encoder variants
(NZGPU_LIB=libnzgpu_<tag>.so).  usage: compress_c1.py [iters] [precision] [layers per batch]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz

LAYER = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336),
         (4096,), (4096,)]


def timed(ts, prec, iters, ws):
    out = []
    for _ in range(iters + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bs = nz.DeviceBlob.compress_batch(ts, precision=prec, workspace=ws)
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
        for b in bs:
            b.free()
    return float(np.median(out[2:]))


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    multi = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    g = torch.Generator(device="cuda").manual_seed(42)
    c1 = [(torch.randn(4096 * 4096, device="cuda", generator=g) * 0.02).to(torch.bfloat16)]
    layer = []
    for s in LAYER:
        n = int(np.prod(s))
        layer.append(torch.ones(n, dtype=torch.bfloat16, device="cuda") if len(s) == 1 else
                     (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    ws = torch.empty(nz.DeviceBlob.compress_workspace_bytes([t.numel() for t in layer], prec), dtype=torch.uint8,
                     device="cuda")
    t1 = timed(c1, prec, iters, ws)
    tl = timed(layer, prec, iters, ws)
    n_l = sum(t.numel() for t in layer)
    rec = {"lib": os.environ.get("NZGPU_LIB", "libnzgpu.so"), "prec": prec, "c1_ms": round(t1 * 1e3, 3),
           "layer_ms": round(tl * 1e3, 3), "layer_gbs_bf16_in": round(2 * n_l / tl / 1e9, 1)}
    if multi > 1:  # one batch of `multi` layers: enough chains for the byte-queue encoder
        batch = layer * multi
        ws = torch.empty(nz.DeviceBlob.compress_workspace_bytes([t.numel() for t in batch], prec),
                         dtype=torch.uint8, device="cuda")
        tm = timed(batch, prec, max(3, iters // 4), ws)
        rec.update({"multi": multi, "multi_ms": round(tm * 1e3, 3), "multi_gbs_bf16_in": round(2 * n_l * multi / tm / 1e9, 1)})
    print(json.dumps(rec), flush=True)


main()
