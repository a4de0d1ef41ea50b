"""Quick decode timing of one tensor (dev tool, not the contract bench).
usage: quickbench.py [n] [precisions e.g. 7,3,0] [intervals e.g. 64,128,256] [iters]"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_20650_b200 as nz

def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096 * 4096
    precs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "7,3,0").split(",")]
    ks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "64,128,256").split(",")]
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    torch.manual_seed(0)
    w = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for prec in precs:
        for K in ks:
            t0 = time.time()
            blob = nz.DeviceBlob.compress(w, precision=prec, interval=K)
            torch.cuda.synchronize(); tc = time.time() - t0
            out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            plan = nz.DecodePlan([blob], [out])
            for _ in range(3): plan.launch()
            plan.status()
            if prec == 7:
                assert torch.equal(out.view(torch.int16), w.view(torch.int16))
            times = []
            for _ in range(iters):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(); plan.launch(); b.record(); b.synchronize()
                times.append(a.elapsed_time(b) * 1e-3)
            t = float(np.median(times))
            info = blob.info
            algo = info.payload_bytes + 2 * n
            print(f"prec={prec} K={K} n={n} compress={tc*1e3:.1f}ms decode={t*1e6:.1f}us "
                  f"algoGB/s={algo/t/1e9:.1f} frac={algo/t/6545.6e9:.3f} bf16GB/s={2*n/t/1e9:.1f} "
                  f"ratio={2*n/(info.payload_bytes+35+8):.4f} win={info.max_window}", flush=True)
            plan.free(); blob.free()

main()
