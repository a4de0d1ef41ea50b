"""CRC-32 and NZT throughput (dev tool, GPU only).

Device CRC-32 (nzgpu_crc32) of resident buffers 16 MiB .. 2 GiB: GB/s and
fraction of the 6,536 GB/s HBM roofline (bytes read once).  NZT write/read of
a Llama-3-8B-layer-sized tensor through host buffers (includes the PCIe
copies).  One JSON line per measurement."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz
from paper_2410_20650_b200 import nzgpu as N

PEAK = 6545.6  # MEASURED_PEAKS.json hbm_gbs


def dev_crc(t, n):
    out = C.c_uint32()
    N.check(N.lib.nzgpu_crc32(C.c_void_p(t.data_ptr()), n, None, C.byref(out)), "crc32")
    return out.value


def main():
    big = torch.randint(0, 256, (2 << 30,), dtype=torch.uint8, device="cuda")
    for log in (24, 26, 28, 30, 31):
        n = 1 << log
        dev_crc(big, n)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev_crc(big, n)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        print(json.dumps({"what": "crc32_device", "bytes": n, "ms": round(t * 1e3, 3),
                          "gbs": round(n / t / 1e9, 1), "frac": round(n / t / 1e9 / PEAK, 4)}), flush=True)
    del big
    n = 218112000 // 4  # one gate/up/down-sized tensor x 0.93
    w = (torch.randn(58720256, device="cuda") * 0.02).to(torch.bfloat16)
    db = nz.DeviceBlob.compress(w, meta=nz.TensorMeta((14336, 4096)))
    data = db.to_nzt()
    for what, fn in (("write_nzt_device_blob", lambda: db.to_nzt()),
                     ("read_nzt_to_device_blob", lambda: nz.DeviceBlob.from_nzt(data).free())):
        fn()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        print(json.dumps({"what": what, "file_bytes": len(data), "elements": 58720256, "ms": round(t * 1e3, 2),
                          "file_gbs": round(len(data) / t / 1e9, 2)}), flush=True)


main()
