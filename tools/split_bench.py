"""K1 (split + exponent histogram) throughput (dev tool): nzgpu_split on one
large bf16 tensor, CUDA-event timed; GB/s of HBM traffic (2 B in + 2 B out
per element).  usage: split_bench.py [n]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_20650_b200 import nzgpu as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
v = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
e = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
m = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
c = torch.zeros(256, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
run = lambda: N.check(N.lib.nzgpu_split(C.c_void_p(v.data_ptr()), n, C.c_void_p(e.data_ptr()),
                                        C.c_void_p(m.data_ptr()), C.c_void_p(c.data_ptr()), C.c_void_p(s)), "split")
for _ in range(3):
    c.zero_()
    run()
ts = []
for _ in range(10):
    c.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 1e3)
t = sorted(ts)[len(ts) // 2]
want = torch.bincount(((v.view(torch.int16).int() >> 7) & 0xFF).flatten(), minlength=256)
assert torch.equal(c.cpu(), want.cpu()), "histogram mismatch"
assert torch.equal(e[:n].int().cpu(), ((v.view(torch.int16).int() >> 7) & 0xFF).to(torch.uint8).int().cpu())
print(f"{os.environ.get('NZGPU_LIB', 'libnzgpu.so')} n={n} {t * 1e3:.3f} ms {4 * n / t / 1e9:.1f} GB/s")
