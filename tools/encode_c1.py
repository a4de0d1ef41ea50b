"""ncu target: compress one 4096x4096 tensor (C1, 256 rANS chains) a few times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_20650_b200 as nz

g = torch.Generator(device="cuda").manual_seed(42)
w = (torch.randn(4096 * 4096, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
for _ in range(3):
    for b in nz.DeviceBlob.compress_batch([w]):
        b.free()
torch.cuda.synchronize()
print("ok")
