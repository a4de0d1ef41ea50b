"""ncu target: decode one 4096x4096 tensor (C1) a few times (L2 flushed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_20650_b200 as nz

g = torch.Generator(device="cuda").manual_seed(42)
w = (torch.randn(4096 * 4096, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
(b,) = nz.DeviceBlob.compress_batch([w])
out = torch.empty_like(w)
plan = nz.DecodePlan([b], [out])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    plan.launch()
plan.status()
assert torch.equal(out.view(torch.int16), w.view(torch.int16))
print("ok")
