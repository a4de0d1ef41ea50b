"""Headline benchmark: NeuZip layer-by-layer decode of Llama-3-8B-shaped
weights on B200 (BASELINE.json configs[1]; metric: decode GB/s of
reconstructed bf16 weights, % of HBM roofline; ratio).

One step = decode every tensor of the model once, layer by layer, each layer
(7 projections + 2 RMSNorms) as ONE grouped kernel launch into a reused
output buffer (the reference's Alg. 1 usage: one uncompressed layer live,
nn.hpp:228-248), plus embed, lm_head and the final norm.

Algorithmic bytes per tensor:
    stream_len + mantissa_len + scale_len + 512-byte table + 2n (bf16 out)
i.e. the reference-format compressed payload read plus the bf16 written.
The checkpoint side index is NOT counted (it is reported as overhead).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision 7|3|1|0]
    python bench.py --impl reference ...   # the reference's CPU codec arm

Multi-GPU (torchrun, one process per GPU): every rank decodes its own
Llama-3-8B-shaped model (weak scaling: per-GPU work fixed, no collective on
the data path); time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent

# Llama-3-8B: hidden 4096, ffn 14336, 32 layers, 32 heads / 8 KV heads, vocab 128256, untied.
LLAMA3_8B = dict(hidden=4096, ffn=14336, layers=32, kv=1024, vocab=128256)
# Llama-3-70B: hidden 8192, ffn 28672, 80 layers, 64 heads / 8 KV heads, vocab 128256 (BASELINE configs[3]).
LLAMA3_70B = dict(hidden=8192, ffn=28672, layers=80, kv=1024, vocab=128256)
MODELS = {"8b": LLAMA3_8B, "70b": LLAMA3_70B}


def llama_layout(cfg=LLAMA3_8B):
    h, f, kv = cfg["hidden"], cfg["ffn"], cfg["kv"]
    groups = []
    for layer in range(cfg["layers"]):
        groups.append((f"layer{layer}", [
            ("q_proj", (h, h), "w"), ("k_proj", (kv, h), "w"), ("v_proj", (kv, h), "w"),
            ("o_proj", (h, h), "w"), ("gate_proj", (f, h), "w"), ("up_proj", (f, h), "w"),
            ("down_proj", (h, f), "w"), ("input_layernorm", (h,), "norm"),
            ("post_attention_layernorm", (h,), "norm")]))
    groups.append(("embed_tokens", [("embed_tokens", (cfg["vocab"], h), "w")]))
    groups.append(("lm_head", [("lm_head", (cfg["vocab"], h), "w"), ("norm", (h,), "norm")]))
    return groups


def workload_name(args, world):
    name = f"Llama-3-{args.model.upper()}-shaped per-layer decode"
    if args.precision != 7:
        name += f" lossy k={args.precision} B={args.block}"
    if args.shard == "lpt":
        name += f", full model LPT-sharded over {world} GPU(s)"
    return name


def numel(shape):
    n = 1
    for d in shape:
        n *= d
    return n


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", HBM_FALLBACK)), "measured"
    return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._first = threading.Event()  # set once a sample exists
        self._t = None

    def _add(self, row):
        self.samples.append(row)
        self._first.set()

    def _run(self):
        try:  # NVML: 10 ms sampling, enough samples even for a short timed region
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self._add([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.01)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self._add(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # NVML / nvidia-smi start-up can outlast a short timed region: wait
        # for the first sample here, before the caller starts its timer
        self._first.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- GPU arm ---
def run_gpu(args):
    import numpy as np
    import torch

    import paper_2410_20650_b200 as nz

    world, rank, local = dist_setup()
    # NZ_BENCH_BACKEND=gloo (test only): ranks may share a GPU (device =
    # local rank mod visible GPUs) to exercise the N>1 harness on a 1-GPU box;
    # the plumbing reductions then run on CPU tensors.  Default: NCCL, one GPU
    # per rank.
    backend = os.environ.get("NZ_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    red_dev = dev if backend == "nccl" else None  # where the timing reductions run
    stream = torch.cuda.current_stream()

    # ---- synthetic model: HF Llama init N(0, 0.02^2) weights, RMSNorm = 1.0.
    # replica (weak scaling): every rank owns a whole model with its own seeds;
    # lpt (strong scaling, C4): one model, whole tensors assigned to ranks by
    # LPT on element count (shard.py) -- each rank compresses and decodes only
    # its tensors, no collective on the data path.
    from paper_2410_20650_b200.shard import lpt_assign

    groups = llama_layout(MODELS[args.model])
    flat = [numel(shape) for _, ts in groups for _, shape, _ in ts]
    owner = lpt_assign(flat, world) if args.shard == "lpt" else [rank] * len(flat)
    blobs, plans_meta = [], []
    t0 = time.time()
    gen = torch.Generator(device=dev)
    tensor_idx = -1
    # Tensors are generated on the GPU and compressed in batches of up to
    # --compress-batch elements (nzgpu_compress_batch: one encode launch over
    # every chunk of the batch); only the compress calls are timed.
    pending, pend_elems, t_comp = [], 0, 0.0
    by_group: dict = {}
    # One workspace for every batch, allocated once (a user keeps it like a
    # plan): bounded by the largest batch plus per-tensor rounding.
    mine = [n for n, o in zip(flat, owner) if o == rank]
    ws_bytes = (nz.DeviceBlob.compress_workspace_bytes([min(args.compress_batch, max(sum(mine), 1))] + [1] * len(mine),
                                                       args.precision)
                + len(mine) * (2 * 65536 + 1024))
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    # untimed warm-up: loads the compress kernels (lazy module loading costs
    # ~30 ms on the first call) so the timed batches measure compression
    for b in nz.DeviceBlob.compress_batch([torch.ones(1 << 20, dtype=torch.bfloat16, device=dev),
                                           (torch.randn(1 << 20, device=dev) * 0.02).to(torch.bfloat16)],
                                          precision=args.precision, block_size=args.block, interval=args.interval):
        b.free()

    def flush():
        nonlocal pending, pend_elems, t_comp
        if not pending:
            return
        torch.cuda.synchronize()
        tc = time.perf_counter()
        out = nz.DeviceBlob.compress_batch([w for _, _, _, _, w in pending], precision=args.precision,
                                           block_size=args.block, interval=args.interval,
                                           metas=[nz.TensorMeta(shape) for _, _, shape, _, _ in pending],
                                           max_batch_elements=1 << 62, workspace=workspace)
        torch.cuda.synchronize()
        t_comp += time.perf_counter() - tc
        if os.environ.get("NZGPU_TRACE"):
            print(f"[bench] compress_batch of {len(pending)} tensors: {(time.perf_counter() - tc) * 1e3:.1f} ms",
                  file=sys.stderr)
        for (gname, tname, shape, tidx, w), blob in zip(pending, out):
            blob.tidx = tidx
            by_group.setdefault(gname, []).append((tname, shape, blob))
        pending, pend_elems = [], 0

    kinds = [kind for _, ts in groups for _, _, kind in ts]

    def regen(tidx):
        """Synthetic weight `tidx` (deterministic: regenerated for the check)."""
        n = flat[tidx]
        if kinds[tidx] == "norm":
            return torch.ones(n, dtype=torch.bfloat16, device=dev)
        salt = rank * 10007 if args.shard == "replica" else 0
        gen.manual_seed(args.seed * 1000003 + salt + tidx)
        return (torch.randn(n, device=dev, generator=gen) * 0.02).to(torch.bfloat16)

    for gname, tensors in groups:
        for tname, shape, kind in tensors:
            tensor_idx += 1
            if owner[tensor_idx] != rank:
                continue
            n = numel(shape)
            if pend_elems and pend_elems + n > args.compress_batch:
                flush()
            pending.append((gname, tname, shape, tensor_idx, regen(tensor_idx)))
            pend_elems += n
    flush()
    del workspace
    for gname, _ in groups:
        if gname in by_group:
            blobs.append((gname, by_group[gname]))
    torch.cuda.synchronize()
    t_compress = time.time() - t0
    comp_elems = sum(b.n for _, gb in blobs for _, _, b in gb)

    # ---- per-layer grouped decode plans into one reused output buffer
    # --overlap 1: consecutive layer plans alternate between two streams and
    # two output buffers (the double buffer of Alg. 1's consumer, nn.hpp:286-318),
    # so layer l+1's CTAs start on the SMs layer l's tail CTAs release; plan
    # k+2 reuses plan k's buffer and follows it on the same stream.
    max_elems = max(sum(b.n for _, _, b in gb) for _, gb in blobs)
    nbuf = 2 if args.overlap else 1
    outbufs = [torch.empty(max_elems + 64 * 16, dtype=torch.bfloat16, device=dev) for _ in range(nbuf)]

    def make_plan(gb, outbuf):
        outs, off = [], 0
        for _, _, b in gb:
            outs.append(outbuf[off:off + b.n])
            off += (b.n + 63) // 64 * 64  # keep every output 128-byte aligned
        return nz.DecodePlan([b for _, _, b in gb], outs), outs

    plans, bytes_algo, total_n, total_fp, index_bytes = [], 0, 0, 0, 0
    for gname, gb in blobs:
        plans.append(make_plan(gb, outbufs[len(plans) % nbuf])[0])
        for _, shape, b in gb:
            i = b.info
            bytes_algo += int(i.payload_bytes) + 2 * b.n
            total_n += b.n
            total_fp += int(i.payload_bytes) + nz.codec.nzt_header_bytes(len(shape))  # footprint().total()
            index_bytes += int(i.index_len)
    launches_per_step = sum(p.launches for p in plans)

    # L2 (126 MB) is far smaller than one step's traffic (~26 GB): no flush needed.
    side = torch.cuda.Stream(device=dev) if args.overlap else stream
    streams = (stream, side)
    # Bounded run-ahead: plan k (stream k % 2) also waits for plan k-3 (the
    # other stream's previous plan), so at most two adjacent layer plans are
    # in flight -- layer l+1 fills layer l's tail; no stream runs whole
    # layers ahead of the other.
    done = [torch.cuda.Event() for _ in range(4)]
    seq = [0]

    def run_plans(ps, events=None, overlap=bool(args.overlap)):
        for k, p in enumerate(ps):
            st = streams[k % 2] if overlap else stream
            q = seq[0]
            if overlap and q >= 3:
                st.wait_event(done[(q - 3) % 4])
            if events is not None:
                events[k][0].record(st)
            p.launch(st)
            if events is not None:
                events[k][1].record(st)
            if overlap:
                done[q % 4].record(st)
            seq[0] += 1

    def join():
        stream.wait_stream(side)
        seq[0] = 0  # the next schedule starts with both streams drained

    def step(events=None, overlap=bool(args.overlap)):
        run_plans(plans, events, overlap)

    side.wait_stream(stream)
    for _ in range(args.warmup):
        step()
        join()
        side.wait_stream(stream)
        step(overlap=False)
        side.wait_stream(stream)
    join()
    for p in plans:
        p.status(stream)
    torch.cuda.synchronize()

    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in plans]
          for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        start.record(stream)
        side.wait_stream(stream)
        for s in range(args.steps):
            step()
        join()
        stop.record(stream)
        torch.cuda.synchronize()
        # roofline pass: the same steps serialised on one stream, each launch
        # bracketed by CUDA events on the stream it runs on
        for s in range(args.steps):
            step(ev[s], overlap=False)
        torch.cuda.synchronize()
    for p in plans:
        p.status(stream)  # every decode passed its checkpoint/desync checks
    elapsed = start.elapsed_time(stop) / 1e3
    kernel_time = sum(a.elapsed_time(b) for row in ev for a, b in row) / 1e3
    from paper_2410_20650_b200.shard import reduce_timing

    t_max, bytes_all = elapsed, bytes_algo  # bytes_all: algorithmic bytes of every rank's tensors
    if dist:
        t_max, bytes_all = reduce_timing(dist, elapsed, bytes_algo, device=red_dev)
    value = bytes_all * args.steps / t_max / 1e9
    peak, peak_kind = load_peaks()
    achieved = bytes_algo * args.steps / kernel_time / 1e9  # per-launch bytes / launch time, aggregated
    traffic = None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            tj = json.load(fh)
        if tj.get("precision") == args.precision:
            # ncu DRAM bytes (read + write) per launch, over the same launch
            # time as `achieved`: directly comparable with it.
            traffic = round(achieved * float(tj["dram_bytes_per_algo_byte"]), 2)

    # ---- output check, outside the timed region: every tensor of the model
    # decoded once more through the same grouped plans on the same two-stream
    # schedule, into distinct buffers, then compared (lossless: with the
    # regenerated source; lossy: with the blob's single-tensor decode; one
    # sampled tensor against the reference codec, oracle/_ref).
    verified, sample = 0, None
    if args.verify:
        verified, sample = verify_outputs(args, nz, torch, blobs, make_plan, run_plans, join, regen, stream, dev,
                                          rank)
        if dist:
            vt = torch.tensor([verified], dtype=torch.int64, device=red_dev)
            dist.all_reduce(vt, op=dist.ReduceOp.SUM)
            verified = int(vt.item())

    # ---- e2e through the reference-facing host API (host buffers in/out)
    e2e = run_e2e(args, nz, blobs, torch, dist, red_dev)
    if dist:
        dist.barrier()

    line = {
        "metric": "decode GB/s of reconstructed bf16 weights (% HBM roofline); ratio",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t_max / args.steps * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak" if args.shard == "replica" else "strong",
        "vs_baseline": None,
        "dtype": "u8" if args.precision == 7 else "u8+bf16",
        "data": "synthetic: random-init N(0,0.02^2) bf16 weights (torch.randn on GPU), RMSNorm=1.0",
        "config": {
            "workload": workload_name(args, world),
            "elements_rank0": total_n,
            "precision": args.precision,
            "block_size": args.block if args.precision != 7 else None,
            "chunk_symbols": 65536,
            "checkpoint_interval": int(blobs[0][1][0][2].info.interval),
            "launches_per_step_rank0": launches_per_step,
            "bytes_algo_per_step": bytes_all,
            "index_bytes_rank0": index_bytes,
            "ratio": round(2 * total_n / total_fp, 6),
            "device_ratio": round(2 * total_n / (total_fp + index_bytes), 6),
            "device_ratio_note": "2n / (footprint + GPU side index): what HBM holds per decoded bf16 byte",
            "verified_tensors": verified,
            "verify": sample,
            "l2": "no flush: one step moves >= 3.4 GB per GPU >> 126 MB L2",
            "schedule": ("layer plans alternate between 2 streams and 2 output buffers (decode of layer l+1 "
                         "starts on the SMs layer l's tail releases); roofline from a separate serialised pass"
                         if args.overlap else "layer plans serialised on one stream, one output buffer"),
            "parallelism": (f"weak dp{world}: one model replica per GPU, no collective" if args.shard == "replica"
                            else f"strong: whole tensors LPT-sharded over {world} GPU(s), no collective"),
            "compress_s": round(t_compress, 2),
            "compress": {"gbs_bf16_in": round(2 * comp_elems / t_comp / 1e9, 2), "s": round(t_comp, 4),
                         "batch_elements": args.compress_batch,
                         "note": "nzgpu_compress_batch wall time (host-synchronised), rank 0, bf16 bytes in, "
                                 "one reused workspace; includes first-touch allocation of the blobs' device "
                                 "memory; compress_s adds tensor generation"},
        },
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                     "kernel": f"{plans[0].kernel} (one launch per layer)",
                     "step_frac": round(value / max(world, 1) / peak, 4),
                     "note": "achieved/frac: per-launch CUDA-event durations of a serialised pass (one stream); "
                             "step_frac: the timed (overlapped) step's per-GPU GB/s over the same peak"},
        "clocks": clocks.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
    }
    if rank == 0:
        if args.c1:
            line["c1"] = run_c1(args, nz, torch, peak, dev)
            if args.precision == 7:
                line["c3"] = run_c3(args, nz, torch, peak, dev)
        if args.dropin and args.model == "8b" and args.precision == 7:
            line["e2e_dropin"] = run_dropin_bench()
        line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_c1(args, nz, torch, peak, dev):
    """configs[0] beside the headline: one 4096x4096 N(0, 0.02^2) tensor
    (rank 0, outside the timed region).  Decode latency with L2 flushed
    before every repetition (a 256 MiB write), CUDA events on the launching
    stream, median of 21; compress wall time (host-synchronised, median of 7).
    The decoded tensor is checked against the source (lossless) or the
    single-blob decode (lossy)."""
    import numpy as np

    g = torch.Generator(device=dev).manual_seed(args.seed + 1)
    n = 4096 * 4096
    w = (torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    ts, blob = [], None
    for i in range(7):
        if blob is not None:
            blob.free()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blob = nz.DeviceBlob.compress_batch([w], precision=args.precision, block_size=args.block,
                                            interval=args.interval)[0]
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out = torch.empty_like(w)
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    us = []
    for i in range(24):
        scrub.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        blob.decompress_into(out, stream)
        b.record(stream)
        b.synchronize()
        if i >= 3:
            us.append(a.elapsed_time(b) * 1e3)
    blob.status(stream)
    ok = bool(torch.equal(out.view(torch.int16), (w if args.precision == 7 else blob.decompress()).view(torch.int16)))
    algo = int(blob.info.payload_bytes) + 2 * n
    dec = float(np.median(us))
    res = {"workload": "C1: one 4096x4096 tensor (configs[0])", "decode_us": round(dec, 2),
           "decode_gbs": round(algo / dec / 1e3, 1), "decode_frac": round(algo / dec / 1e3 / peak, 4),
           "compress_ms": round(float(np.median(ts)) * 1e3, 3), "verified": ok,
           "note": "L2 flushed before each decode; events around the single launch (launch latency included)"}
    blob.free()
    return res


def run_c3(args, nz, torch, peak, dev):
    """configs[2] beside the headline (rank 0, outside the timed region):
    one Llama-3-8B layer (7 projections + 2 norms, N(0, 0.02^2) / 1.0)
    compressed lossy k=3, B=512 with compress_batch, decoded by one grouped
    plan 20 times back to back (each decode writes 436 MB: more than L2),
    CUDA events around each launch, median; the outputs are checked against
    the single-blob decodes."""
    import numpy as np

    cfg = MODELS["8b"]
    h, f, kv = cfg["hidden"], cfg["ffn"], cfg["kv"]
    shapes = [(h, h), (kv, h), (kv, h), (h, h), (f, h), (f, h), (h, f), (h,), (h,)]
    g = torch.Generator(device=dev).manual_seed(args.seed + 2)
    ws = [torch.ones(numel(sh), dtype=torch.bfloat16, device=dev) if len(sh) == 1 else
          (torch.randn(numel(sh), device=dev, generator=g) * 0.02).to(torch.bfloat16) for sh in shapes]
    blobs = nz.DeviceBlob.compress_batch(ws, precision=3, block_size=512, interval=args.interval)
    del ws
    outs = [torch.empty(b.n, dtype=torch.bfloat16, device=dev) for b in blobs]
    plan = nz.DecodePlan(blobs, outs)
    stream = torch.cuda.current_stream()
    us = []
    for i in range(23):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.launch(stream)
        b.record(stream)
        b.synchronize()
        if i >= 3:
            us.append(a.elapsed_time(b) * 1e3)
    plan.status(stream)
    ok = all(torch.equal(o.view(torch.int16), bl.decompress().view(torch.int16)) for o, bl in zip(outs, blobs))
    algo = sum(int(bl.info.payload_bytes) + 2 * bl.n for bl in blobs)
    dec = float(np.median(us))
    res = {"workload": "C3: one Llama-3-8B layer, lossy k=3, B=512 (configs[2])", "decode_us": round(dec, 1),
           "decode_gbs": round(algo / dec / 1e3, 1), "decode_frac": round(algo / dec / 1e3 / peak, 4),
           "ratio": round(sum(2 * bl.n for bl in blobs) / sum(int(bl.info.payload_bytes) for bl in blobs), 4),
           "verified": ok, "note": "one grouped launch per decode, back to back; events around each launch"}
    del plan
    for bl in blobs:
        bl.free()
    return res


def verify_outputs(args, nz, torch, blobs, make_plan, run_plans, join, regen, stream, dev, rank):
    """Decode every tensor once more through the same grouped plans and the
    same two-stream schedule as the timed steps, but into distinct output
    buffers (a window of layers at a time), then check each output:
    lossless -> equal to the regenerated source tensor; lossy -> equal to the
    blob's single-tensor decode.  One sampled tensor (rank 0) is also checked
    against the reference codec (oracle/_ref, else the C restatement): its
    compressed sections and its decoded values.  Returns (count, sample)."""
    import hashlib

    import numpy as np

    def padded(gb):
        return sum((b.n + 63) // 64 * 64 for _, _, b in gb)

    budget = max(max(padded(gb) for _, gb in blobs), args.verify_elems)
    checked, i = 0, 0
    pick = None  # smallest non-norm tensor of this rank: the oracle sample
    while i < len(blobs):
        j, tot = i, 0
        while j < len(blobs) and (j == i or tot + padded(blobs[j][1]) <= budget):
            tot += padded(blobs[j][1])
            j += 1
        buf = torch.empty(tot + 64, dtype=torch.bfloat16, device=dev)
        vplans, off = [], 0
        for _, gb in blobs[i:j]:
            p, outs = make_plan(gb, buf[off:off + padded(gb)])
            off += padded(gb)
            vplans.append((p, gb, outs))
        torch.cuda.synchronize()
        run_plans([p for p, _, _ in vplans])
        join()
        for p, _, _ in vplans:
            p.status(stream)
        torch.cuda.synchronize()
        for _, gb, outs in vplans:
            for (tname, shape, b), o in zip(gb, outs):
                if args.precision == 7:
                    want = regen(b.tidx)
                else:
                    want = torch.empty(b.n, dtype=torch.bfloat16, device=dev)
                    b.decompress_into(want)
                    b.status()
                if not torch.equal(o.view(torch.int16), want.view(torch.int16)):
                    raise AssertionError(f"decoded {tname} (tensor {b.tidx}) differs from its reference")
                checked += 1
                if b.n > 4096 and (pick is None or b.n < pick[2].n):
                    pick = (tname, shape, b)
        del vplans, buf
        i = j
    sample = None
    if rank == 0 and pick is not None:
        tname, shape, b = pick
        ref, kind = reference_lib()
        src = regen(b.tidx).view(torch.int16).cpu().numpy().view(np.uint16)
        host = b.to_host()
        got = torch.empty(b.n, dtype=torch.bfloat16, device=dev)
        b.decompress_into(got)
        b.status()
        got = got.view(torch.int16).cpu().numpy().view(np.uint16)
        if args.precision == 7:
            f, st, m = ref.compress_lossless(src)
            ok = host.stream == st and (host.freqs == f).all() and (host.signmant == m).all() and (got == src).all()
        else:
            f, sc, st, pk = ref.compress_lossy(src, args.precision, args.block)
            want = ref.decompress_lossy(f, sc, st, pk, args.precision, args.block, src.size)
            ok = (host.stream == st and (host.freqs == f).all() and (host.signmant == pk).all()
                  and (host.scales == sc).all() and (got == want).all())
        if not ok:
            raise AssertionError(f"sampled tensor {tname} differs from the reference codec ({kind})")
        sample = {"tensor": f"{tname} {tuple(shape)} (tensor {b.tidx})", "oracle": kind,
                  "stream_sha256": hashlib.sha256(host.stream).hexdigest()[:16],
                  "checks": "sections (table, stream, mantissas, scales) and decoded values equal the oracle's"}
    return checked, sample


def run_e2e(args, nz, blobs, torch, dist=None, red_dev="cuda"):
    """Same metric through nzgpu_decompress_host_batch: compressed sections
    H2D from pinned host memory, GPU decode, bf16 D2H to pinned memory, every
    step.  Bounded to the first `--e2e-layers` layers to cap host memory."""
    import ctypes as C

    import numpy as np

    from paper_2410_20650_b200 import nzgpu as N

    sel = [b for _, gb in blobs[: args.e2e_layers] for _, _, b in gb]
    hosts = [b.to_host() for b in sel]
    pinned = []

    def pin(a):
        a = np.ascontiguousarray(a)
        t = torch.from_numpy(a if a.flags.writeable else a.copy()).pin_memory()
        pinned.append(t)
        return t

    ts = []
    h2d = 0
    for h in hosts:
        t = N.HostTensor()
        f = pin(h.freqs)
        s = pin(np.frombuffer(h.stream, np.uint8))
        m = pin(h.signmant)
        ix = pin(np.frombuffer(h.index, np.uint8)) if h.index else None
        t.n = h.meta.element_count()
        t.precision = h.precision
        t.freqs = f.data_ptr()
        t.stream, t.stream_len = s.data_ptr(), s.numel()
        t.mantissas, t.mantissa_len = m.data_ptr(), m.numel()
        if h.precision != 7:
            sc = pin(h.scales)
            t.block_size, t.scales, t.scales_len = h.block_size, sc.data_ptr(), sc.numel()
            h2d += sc.numel()
        if ix is not None:
            t.index, t.index_len = ix.data_ptr(), ix.numel()
            h2d += ix.numel()
        h2d += 512 + s.numel() + m.numel()
        ts.append(t)
    outs = [torch.empty(h.meta.element_count(), dtype=torch.int16).pin_memory() for h in hosts]
    arr = (N.HostTensor * len(ts))(*ts)
    ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    algo = sum(int(b.info.payload_bytes) + 2 * b.n for b in sel)
    d2h = sum(2 * b.n for b in sel)
    N.check(N.lib.nzgpu_decompress_host_batch(arr, len(ts), ptrs), "e2e warmup")
    steps = max(1, min(args.steps, 5))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        N.check(N.lib.nzgpu_decompress_host_batch(arr, len(ts), ptrs), "e2e")
    dt = time.perf_counter() - t0
    # every rank decodes its own tensors through its own PCIe link: whole-job
    # bytes over the slowest rank's time
    if dist:
        t = torch.tensor([dt, float(algo), float(h2d), float(d2h)], dtype=torch.float64, device=red_dev)
        dt_max = t[:1].clone()
        dist.all_reduce(dt_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dt, algo, h2d, d2h = float(dt_max.item()), int(t[1].item()), int(t[2].item()), int(t[3].item())
    return {"value": round(algo * steps / dt / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "sample": f"first {args.e2e_layers} layers of each rank "
            f"({len(sel)} tensors on rank 0), {steps} steps, nzgpu_decompress_host_batch (pinned host "
            f"buffers), all ranks concurrently: sum of bytes / max time"}


def run_dropin_bench():
    """The reference-signature C++ API (include/neuzip/tensorstore.hpp) on
    one Llama-3-8B layer, host vectors in and out (tools/dropin_bench.cpp):
    `fresh` = std::vector<Bf16> decompress_lossless(blob) as the reference
    declares it (a new value-initialised vector per call); `reused` =
    decompress_lossless_into(blob, vec) into vectors kept across calls."""
    exe = os.path.join(ROOT, "paper_2410_20650_b200", "dropin_bench")
    try:
        out = subprocess.run([exe, "3"], capture_output=True, text=True, timeout=600)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        return {"value": d["fresh_gbs"], "unit": "GB/s", "reused": d["reused_gbs"], "ok": d["ok"],
                "compress": d.get("compress_gbs"),
                "sample": "Llama-3-8B layer projections q,k,v,o,gate,up,down ("
                          f"{d['elements']} elements), C++ drop-in decompress_lossless per tensor, median of "
                          f"{d['reps']}; value = fresh std::vector per call (the reference signature), reused = "
                          "decompress_lossless_into a kept vector; compress = compress_lossless of the same tensors "
                          "(host vector in, LosslessBlob out), same algorithmic bytes"}
    except Exception as e:  # reported, never required
        return {"value": None, "unit": "GB/s", "error": repr(e)[:200]}


# ------------------------------------------------------ CPU reference arm ---
def cpu_sample(args):
    """Bounded sample of the workload for the CPU: the first layer's tensors
    (same shapes and N(0,0.02^2) init via the reference's own RNG)."""
    from oracle.oracle import Oracle

    gen = Oracle("port")
    cfg = MODELS[args.model]
    h, f, kv = cfg["hidden"], cfg["ffn"], cfg["kv"]
    shapes = [(h, h), (kv, h), (kv, h), (h, h), (f, h), (f, h), (h, f)][: args.cpu_tensors]
    vals = [gen.gaussian_bf16(gen.derive(42, i), numel(s), 0.02) for i, s in enumerate(shapes)]
    return shapes, vals


def reference_lib():
    from oracle.oracle import Oracle, ref_available

    if ref_available():
        return Oracle("ref"), "reference"
    return Oracle("port"), "port"


def cpu_decoders(ref, kind, vals, args):
    """[(decode_callable, algorithmic_bytes)] for each sample tensor.  With
    the reference library the blob is parsed once and only the reference's
    decompress_lossless / decompress_lossy is timed."""
    out = []
    for v in vals:
        if args.precision == 7:
            f, s, m = ref.compress_lossless(v)
            algo = len(s) + m.size + 512 + 2 * v.size
            if kind == "reference":
                out.append((ref.prepared(f, s, m, v.size).decode, algo))
            else:
                out.append((lambda f=f, s=s, m=m, n=v.size: ref.decompress_lossless(f, s, m, n), algo))
        else:
            f, sc, s, pk = ref.compress_lossy(v, args.precision, args.block)
            algo = len(s) + pk.size + sc.size + 512 + 2 * v.size
            if kind == "reference":
                out.append((ref.prepared(f, s, pk, v.size, args.precision, sc, args.block).decode, algo))
            else:
                out.append((lambda f=f, sc=sc, s=s, pk=pk, n=v.size: ref.decompress_lossy(
                    f, sc, s, pk, args.precision, args.block, n), algo))
    return out


def cpu_baseline(args):
    """The reference CPU codec on the GPU box's host cores (rank 0, N=1 only)."""
    try:
        ref, kind = reference_lib()
        shapes, vals = cpu_sample(args)
        cores = min(os.cpu_count() or 1, 64) if kind == "reference" else 1
        os.environ["NEUZIP_THREADS"] = str(cores)
        decs = cpu_decoders(ref, kind, vals, args)

        def timed(seconds):
            algo, reps, t0 = 0, 0, time.perf_counter()
            while True:
                for fn, a in decs:
                    fn()
                    algo += a
                reps += 1
                if time.perf_counter() - t0 > seconds or reps >= 50:
                    break
            return algo / (time.perf_counter() - t0) / 1e9, reps

        value, reps = timed(args.cpu_seconds)
        one = None
        if kind == "reference" and cores > 1:  # also NEUZIP_THREADS=1 (read per call)
            os.environ["NEUZIP_THREADS"] = "1"
            one, _ = timed(args.cpu_seconds / 2)
            os.environ["NEUZIP_THREADS"] = str(cores)
        return {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": kind,
                "value_1thread": round(one, 4) if one is not None else None,
                "sample": f"decompress of layer-0 tensors {shapes}, {reps} reps, NEUZIP_THREADS={cores} "
                          f"(reference caps workers at 64, parallel.hpp:24); host nproc={os.cpu_count()}; "
                          f"value_1thread: the same with NEUZIP_THREADS=1"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "unavailable", "sample": repr(e)}


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    ref, kind = reference_lib()
    cores = min(os.cpu_count() or 1, 64) if kind == "reference" else 1
    os.environ["NEUZIP_THREADS"] = str(cores)
    shapes, vals = cpu_sample(args)
    decs = cpu_decoders(ref, kind, vals, args)

    def step():
        algo = 0
        for fn, a in decs:
            fn()
            algo += a
        return algo

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    algo = sum(step() for _ in range(args.steps))
    dt = time.perf_counter() - t0
    value = algo / dt / 1e9
    sample = f"decompress of Llama-3-{args.model.upper()} layer-0 tensors {shapes} per step, NEUZIP_THREADS={cores}"
    print(json.dumps({
        "impl": "reference",
        "metric": "decode GB/s of reconstructed bf16 weights (% HBM roofline); ratio",
        "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak" if args.shard == "replica" else "strong",
        "vs_baseline": None, "dtype": "u8" if args.precision == 7 else "u8+f64", "data": "synthetic (reference rng.hpp)",
        # same workload as the B200 arm; the per-step CPU sample is named in
        # cpu_baseline.sample (the metric is per algorithmic byte, so the
        # rates compare directly)
        "config": {"workload": workload_name(args, world), "precision": args.precision,
                   "block_size": args.block if args.precision != 7 else None, "chunk_symbols": 65536},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--precision", type=int, default=7, choices=[7, 3, 1, 0])
    ap.add_argument("--model", choices=sorted(MODELS), default=None,
                    help="8b: BASELINE configs[1] (default at N=1); 70b: configs[3] (default at N>1, LPT-sharded)")
    ap.add_argument("--shard", choices=["replica", "lpt"], default=None,
                    help="replica: a model per GPU (weak, 8b default); lpt: one model sharded (strong, 70b default)")
    ap.add_argument("--block", type=int, default=512)
    ap.add_argument("--interval", type=int, default=0, help="checkpoint stride K (0 = auto)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--e2e-layers", type=int, default=8)
    ap.add_argument("--dropin", type=int, default=1, help="also time the C++ drop-in host API (rank 0, 8B lossless)")
    ap.add_argument("--c1", type=int, default=1, help="also time configs[0] (one 4096x4096 tensor), rank 0")
    ap.add_argument("--cpu-tensors", type=int, default=7)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--verify", type=int, default=1,
                    help="after the timed region, check every decoded tensor (and one against oracle/_ref)")
    ap.add_argument("--verify-elems", type=int, default=1 << 32,
                    help="elements decoded per verification window (distinct output buffers)")
    ap.add_argument("--overlap", type=int, default=1, choices=[0, 1],
                    help="1: consecutive layer decodes on two streams / two output buffers")
    ap.add_argument("--compress-batch", type=int, default=1 << 31,
                    help="max elements per nzgpu_compress_batch call (temporaries ~3 B/element)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun
        sys.exit(spawn_local_ranks(args.gpus))
    if world is not None and int(world) != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.model is None:
        # N=1: BASELINE configs[1] (Llama-3-8B per-layer decode on 1 B200);
        # N>1: configs[3] (Llama-3-70B sharded across 2/4/8 B200 by LPT)
        args.model = "70b" if args.gpus > 1 else "8b"
    if args.shard is None:
        args.shard = "lpt" if args.model == "70b" else "replica"
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


def spawn_local_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: the same command as N local
    ranks (torch.distributed.run, rendezvous on 127.0.0.1).  Only rank 0
    prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


if __name__ == "__main__":
    main()
