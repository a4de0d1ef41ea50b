"""bench.py's one-JSON-line contract: the reference arm on CPU (it times the
unmodified reference codec, oracle/_ref, on host cores) and the B200 arm on
the GPU (roofline, cpu_baseline, e2e, clocks, gpu_launches present and sane)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    from oracle.oracle import ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.3",
                  "--cpu-tensors", "1", timeout=300)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_b200_arm_line():
    d = run_bench("--steps", "3", "--warmup", "3", "--cpu-seconds", "0.3", "--cpu-tensors", "1",
                  "--e2e-layers", "1")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("Llama-3-8B")
    assert d["config"]["ratio"] == pytest.approx(1.5165, abs=2e-4)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], abs=1e-3)
    assert 0 < r["step_frac"] < 1
    assert d["gpu_launches"] == 34 * 3
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert "sm_mhz" in d["clocks"]
    # configs[0] probe: one 4096x4096 tensor, decoded and verified
    c1 = d["c1"]
    assert c1["verified"] is True and c1["decode_us"] > 0 and 0 < c1["decode_frac"] < 1 and c1["compress_ms"] > 0
    c3 = d["c3"]  # configs[2] probe: a lossy layer, decoded and checked
    assert c3["verified"] is True and 0 < c3["decode_frac"] < 1 and c3["ratio"] > 2
    # throughput = algorithmic bytes over the timed steps
    bytes_step = d["config"]["bytes_algo_per_step"]
    assert d["value"] == pytest.approx(bytes_step / (d["ms_per_step"] / 1e3) / 1e9, rel=0.01)


def test_reference_arm_under_torchrun_prints_one_line():
    """N>1 reference arm: rank 0 alone runs and prints, the other ranks exit 0."""
    from oracle.oracle import ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29537", os.path.join(ROOT, "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-tensors", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_gpus_flag_spawns_local_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 local ranks
    (the reference arm here, so it runs on CPU): one JSON line, n_gpus == 2,
    and N>1 defaults to configs[3] (Llama-3-70B, LPT strong scaling)."""
    from oracle.oracle import ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = run_bench("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-tensors", "1",
                  timeout=300)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == "strong" and "70B" in d["config"]["workload"]


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
