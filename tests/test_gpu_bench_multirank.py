"""GPU: the N>1 bench harness end to end on a one-GPU box.  Two ranks under
torchrun share cuda:0 (NZ_BENCH_BACKEND=gloo: NCCL refuses two ranks on one
device; the data path has no collective anyway), the Llama-3-8B model is
LPT-sharded over them (each rank compresses, decodes and verifies only its
tensors), timing is the max over ranks and bytes / verified tensors are
summed.  Checks the one JSON line rank 0 prints; the throughput of two
ranks sharing one GPU means nothing and is not asserted."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpu_bench_two_ranks_lpt_one_line():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, NZ_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--model", "8b", "--shard", "lpt", "--steps", "2", "--warmup", "3", "--dropin", "0",
           "--e2e-layers", "1", "--cpu-seconds", "0.5", "--cpu-tensors", "1"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["verified_tensors"] == 291  # every tensor, each decoded by its owner
    assert d["config"]["bytes_algo_per_step"] > 26e9  # whole model summed over the ranks
    assert d["value"] > 0 and d["e2e"]["value"] > 0
