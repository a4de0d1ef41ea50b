"""One batched compress of N Llama-3-8B layers (ncu target for the encode kernel).
usage: encode_one.py [layers]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_20650_b200 as nz

LAYER = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336)]
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = torch.Generator(device="cuda")
ts = []
for l in range(layers):
    for i, (a, b) in enumerate(LAYER):
        g.manual_seed(1000 * l + i)
        ts.append((torch.randn(a * b, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
for _ in range(2):
    for b in nz.DeviceBlob.compress_batch(ts):
        b.free()
torch.cuda.synchronize()
print("ok")
