"""SURVEY.md §8(d) CPU-vs-GPU table: compress AND decompress, lossless and lossy,
on BASELINE configs[0] (C1: one 4096x4096 tensor) and one Llama-3-8B layer
(C2/C3: q,k,v,o,gate,up,down + 2 norms), the reference CPU codec and the GPU
codec on the same host-resident tensors of the same box.

CPU: the unmodified reference (oracle/_ref, the shim over
/root/reference/proj/include) -- compress_lossless / compress_lossy (the
shim's copy-out of the blob is included) and decompress_* on a blob parsed
once (only the reference's decompress is timed); median of 3 trials
(`neuzip bench` uses 5, neuzip.cpp:129-149; 3 keeps the lossy layer compress
under a minute); NEUZIP_THREADS = nproc (<= 64, parallel.hpp:24), and 1 for C1.
GPU: nzgpu_compress_batch on device-resident tensors (wall time, host
synchronised, median of 5) and the decode plan (CUDA events, median of 20,
L2 flushed before every C1 iteration: 55 MB fits in the 126 MB L2).
Throughput: compress = (bf16 in + compressed out) / s, decode = algorithmic
bytes (compressed in + bf16 out) / s.

Test / measurement infrastructure: the reference library is the baseline
being timed, never the thing shipped.

usage: codec_table.py [out.jsonl]"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2410_20650_b200 as nz
from oracle.oracle import Oracle, ref_available

PEAK = 6545.6  # MEASURED_PEAKS.json hbm_gbs
H, FFN, KV = 4096, 14336, 1024


def workloads(ref):
    c1 = [ref.gaussian_bf16(42, H * H)]  # the golden config-1 tensor (tests/golden/make_golden.py)
    rng = np.random.default_rng(42)
    layer = []
    for shape in [(H, H), (KV, H), (KV, H), (H, H), (FFN, H), (FFN, H), (H, FFN)]:
        w = (rng.standard_normal(shape[0] * shape[1], dtype=np.float32) * 0.02)
        layer.append((torch.from_numpy(w).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)))
    layer += [np.full(H, 0x3F80, np.uint16), np.full(H, 0x3F80, np.uint16)]
    return [("C1 4096x4096 (configs[0])", c1, True, [2]),
            ("C2 Llama-3-8B layer 0 (configs[1]/[2])", layer, False, [2] * 7 + [1, 1])]


def median_time(fn, trials):
    ts = []
    for _ in range(trials):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def cpu_rows(ref, name, vals, prec, threads):
    os.environ["NEUZIP_THREADS"] = str(threads)
    n = sum(v.size for v in vals)
    blobs = []

    def comp():
        blobs.clear()
        for v in vals:
            blobs.append(ref.compress_lossless(v) if prec == 7 else ref.compress_lossy(v, prec, 512))

    tc = median_time(comp, 3)
    preps, payload = [], 0
    for v, b in zip(vals, blobs):
        if prec == 7:
            f, s, m = b
            payload += len(s) + m.size + 512
            preps.append(ref.prepared(f, s, m, v.size))
        else:
            f, sc, s, pk = b
            payload += len(s) + pk.size + sc.size + 512
            preps.append(ref.prepared(f, s, pk, v.size, prec, sc, 512))
    td = median_time(lambda: [p.decode() for p in preps], 3)
    return {"impl": "reference CPU", "threads": threads, "compress_gbs": (2 * n + payload) / tc / 1e9,
            "compress_s": tc, "decode_gbs": (payload + 2 * n) / td / 1e9, "decode_s": td}, payload


def gpu_rows(vals, prec, flush):
    dev = torch.device("cuda")
    xs = [torch.from_numpy(v.view(np.int16)).to(dev) for v in vals]
    n = sum(x.numel() for x in xs)

    def comp():
        out = nz.DeviceBlob.compress_batch(xs, precision=prec, block_size=512)
        torch.cuda.synchronize()
        return out

    for b in comp():  # warm-up (module load)
        b.free()
    tcs = []
    blobs = None
    for _ in range(5):
        if blobs:
            for b in blobs:
                b.free()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blobs = comp()
        tcs.append(time.perf_counter() - t0)
    tc = statistics.median(tcs)
    payload = sum(int(b.info.payload_bytes) for b in blobs)
    outs = [torch.empty(x.numel() + 1024, dtype=torch.int16, device=dev)[: x.numel()] for x in xs]
    plan = nz.DecodePlan(blobs, outs)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        plan.launch()
    plan.status()
    for x, o in zip(xs, outs):
        if prec == 7:
            assert torch.equal(x, o), "GPU round trip"
    times = []
    for _ in range(20):
        if flush:
            scratch.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.launch()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    plan.status()
    td = statistics.median(times)
    # the reference-facing host API (pageable numpy in/out, copies included)
    hb = [nz.codec.compress_lossless(v) if prec == 7 else nz.codec.compress_lossy(v, prec, 512) for v in vals]
    dec = nz.codec.decompress_lossless if prec == 7 else nz.codec.decompress_lossy
    th = median_time(lambda: [dec(b) for b in hb], 3)
    for b in blobs:
        b.free()
    return {"impl": "B200", "compress_gbs": (2 * n + payload) / tc / 1e9, "compress_s": tc,
            "decode_gbs": (payload + 2 * n) / td / 1e9, "decode_s": td, "decode_frac": (payload + 2 * n) / td / 1e9 / PEAK,
            "host_api_decode_gbs": (payload + 2 * n) / th / 1e9}, payload


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    if not ref_available():
        raise SystemExit("oracle/_ref (the reference library) is not built")
    ref = Oracle("ref")
    nproc = min(os.cpu_count() or 1, 64)
    lines = []
    for name, vals, c1, ndims in workloads(ref):
        n = sum(v.size for v in vals)
        for prec in (7, 3, 0):
            g, gp = gpu_rows(vals, prec, flush=c1)
            rows = [g]
            for th in ([nproc, 1] if c1 else [nproc]):
                c, cp = cpu_rows(ref, name, vals, prec, th)
                assert cp == gp, f"payload bytes differ: reference {cp} vs GPU {gp}"
                rows.append(c)
            line = {"workload": name, "elements": n, "precision": prec, "block_size": 512 if prec != 7 else None,
                    "ratio": round(2 * n / (gp + sum(nz.codec.nzt_header_bytes(d) for d in ndims)), 6),
                    "payload_bytes": gp, "cpu_model_nproc": os.cpu_count(),
                    "rows": [{k: (round(v, 6) if isinstance(v, float) else v) for k, v in r.items()} for r in rows]}
            cpu = rows[1]
            line["gpu_vs_cpu_nproc"] = {"compress": round(g["compress_gbs"] / cpu["compress_gbs"], 1),
                                        "decode": round(g["decode_gbs"] / cpu["decode_gbs"], 1)}
            print(json.dumps(line), flush=True)
            lines.append(line)
    if out_path:
        with open(out_path, "w") as fh:
            for l in lines:
                fh.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()
