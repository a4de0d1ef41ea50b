"""Layer-wise consumer measurement: forward pass of a
Llama-3-8B-FFN-shaped MLP stack (4096 -> 14336 -> 4096, 16 pairs = 32 linear
layers, 1.88 B params) with weights resident compressed (decode of layer l+1
beside layer l's GEMM, decode capped to `ctas` SMs) vs resident raw.
Prints one JSON line per (tokens, ctas)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2410_20650_b200 import layerwise as lw


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    h, f, pairs = 4096, 14336, 16
    g = torch.Generator(device="cuda").manual_seed(0)
    raw_layers = []
    for _ in range(pairs):
        for i, o in ((h, f), (f, h)):
            raw_layers.append(lw.RawLayer((torch.randn(o, i, device="cuda", generator=g) * 0.02).to(torch.bfloat16),
                                          torch.zeros(o, dtype=torch.bfloat16, device="cuda")))
    raw = lw.RawMlp(raw_layers)
    params = sum(l.weight.numel() for l in raw_layers)
    comp = lw.CompressedMlp.from_raw(raw_layers)
    dec_ms = timed(lambda: [p.launch() for p in comp.plans])
    for tokens in (1024, 4096, 16384):
        x = torch.randn(tokens, h, device="cuda", generator=g).to(torch.bfloat16)
        t_raw = timed(lambda: raw.forward(x))
        for ctas in (0, 16, 32, 64):
            comp.decode_ctas = ctas
            for i in range(len(comp.layers)):
                comp._plan(i)
            # status checks of every plan are done once after the timing
            t_cmp = timed(lambda: comp.forward(x, check=False))
            y_raw, y_cmp = raw.forward(x), comp.forward(x)
            assert torch.equal(y_raw.view(torch.int16), y_cmp.view(torch.int16))
            print(json.dumps({"tokens": tokens, "decode_ctas": ctas or "all", "params": params,
                              "raw_forward_ms": round(t_raw, 3), "compressed_forward_ms": round(t_cmp, 3),
                              "overhead": round(t_cmp / t_raw - 1, 4), "decode_only_ms": round(dec_ms, 3),
                              "gemm_tflops": round(2 * tokens * params / t_raw / 1e9, 1)}), flush=True)


main()
