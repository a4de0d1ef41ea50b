"""One device CRC-32 of 1 GiB (dev tool for ncu)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_20650_b200 import nzgpu as N

big = torch.randint(0, 256, (1 << 30,), dtype=torch.uint8, device="cuda")
out = C.c_uint32()
for _ in range(3):
    N.check(N.lib.nzgpu_crc32(C.c_void_p(big.data_ptr()), big.numel(), None, C.byref(out)), "crc")
print(hex(out.value))
