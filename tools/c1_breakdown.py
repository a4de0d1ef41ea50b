"""C1 (one 4096x4096 tensor) decode latency broken down: after an L2 flush
(the bench's c1 probe), back to back without a flush (warm L2), and ten
launches timed as one (launch latency amortised).  Dev tool.
usage: c1_breakdown.py [kernel: persist|tiles]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_20650_b200 as nz


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "tiles":
        nz.nzgpu.lib.nzgpu_set_decode_kernel(1)
    g = torch.Generator(device="cuda").manual_seed(43)
    n = 4096 * 4096
    w = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    blob = nz.DeviceBlob.compress_batch([w])[0]
    out = torch.empty_like(w)
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()

    def once(flush):
        if flush:
            scrub.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        blob.decompress_into(out, s)
        b.record(s)
        b.synchronize()
        return a.elapsed_time(b) * 1e3

    res = {}
    for name, flush in (("flushed_us", True), ("warm_us", False)):
        v = [once(flush) for _ in range(25)][5:]
        res[name] = round(float(np.median(v)), 2)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        blob.decompress_into(out, s)
    a.record(s)
    for _ in range(20):
        blob.decompress_into(out, s)
    b.record(s)
    b.synchronize()
    res["back_to_back_us"] = round(a.elapsed_time(b) * 1e3 / 20, 2)
    blob.status(s)
    assert torch.equal(out.view(torch.int16), w.view(torch.int16))
    res["kernel"] = sys.argv[1] if len(sys.argv) > 1 else "persist"
    print(json.dumps(res))


main()
