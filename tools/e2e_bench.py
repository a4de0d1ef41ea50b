"""e2e host-API decode (dev tool): nzgpu_decompress_host_batch over L
Llama-3-8B layers with pinned buffers, against the PCIe ceiling of the same
bytes (H2D alone, D2H alone, both concurrently).  usage: e2e_bench.py [layers]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz
from paper_2410_20650_b200 import nzgpu as N

LAYER = [(4096, 4096), (1024, 4096), (1024, 4096), (4096, 4096), (14336, 4096), (14336, 4096), (4096, 14336),
         (4096,), (4096,)]
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = torch.Generator(device="cuda")
ws = []
for l in range(layers):
    for i, sh in enumerate(LAYER):
        n = sh[0] * (sh[1] if len(sh) > 1 else 1)
        if len(sh) == 1:
            ws.append(torch.ones(n, dtype=torch.bfloat16, device="cuda"))
        else:
            g.manual_seed(1000 * l + i)
            ws.append((torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
blobs = nz.DeviceBlob.compress_batch(ws)
hosts = [b.to_host() for b in blobs]
keep = []


def pin(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    keep.append(t)
    return t


ts, h2d = [], 0
for h in hosts:
    t = N.HostTensor()
    f, s, m, ix = pin(h.freqs), pin(np.frombuffer(h.stream, np.uint8)), pin(h.signmant), pin(np.frombuffer(h.index, np.uint8))
    t.n, t.precision, t.freqs = h.meta.element_count(), h.precision, f.data_ptr()
    t.stream, t.stream_len = s.data_ptr(), s.numel()
    t.mantissas, t.mantissa_len = m.data_ptr(), m.numel()
    t.index, t.index_len = ix.data_ptr(), ix.numel()
    h2d += 512 + s.numel() + m.numel() + ix.numel()
    ts.append(t)
outs = [torch.empty(h.meta.element_count(), dtype=torch.int16).pin_memory() for h in hosts]
arr = (N.HostTensor * len(ts))(*ts)
ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
algo = sum(int(b.info.payload_bytes) + 2 * b.n for b in blobs)
d2h = sum(2 * b.n for b in blobs)
N.check(N.lib.nzgpu_decompress_host_batch(arr, len(ts), ptrs), "warmup")
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    N.check(N.lib.nzgpu_decompress_host_batch(arr, len(ts), ptrs), "e2e")
dt = (time.perf_counter() - t0) / reps
for o, w in zip(outs, ws):
    assert torch.equal(o, w.view(torch.int16).cpu())

# PCIe ceiling for the same bytes
hb = torch.empty(h2d, dtype=torch.uint8).pin_memory()
db = torch.empty(h2d, dtype=torch.uint8, device="cuda")
ho = torch.empty(d2h, dtype=torch.uint8).pin_memory()
do = torch.empty(d2h, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / 3


t_h = timed(lambda: db.copy_(hb, non_blocking=True))
t_d = timed(lambda: ho.copy_(do, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        db.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


t_b = timed(both)
print(f"layers={layers} h2d={h2d/1e9:.3f}GB d2h={d2h/1e9:.3f}GB e2e={dt*1e3:.2f}ms {algo/dt/1e9:.2f}GB/s | "
      f"H2D alone {t_h*1e3:.2f}ms ({h2d/t_h/1e9:.1f}GB/s) D2H alone {t_d*1e3:.2f}ms ({d2h/t_d/1e9:.1f}GB/s) "
      f"both {t_b*1e3:.2f}ms -> e2e ceiling {algo/t_b/1e9:.2f}GB/s")
