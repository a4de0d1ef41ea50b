"""GPU: the `neuzip` CLI (proj/tools/neuzip.cpp analyze / compress /
decompress / bench) built on the drop-in headers: same CSV output, same files,
same exit codes (2 usage/format, 3 NaN/Inf, 4 checksum)."""
import os
import struct
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2410_20650_b200", "neuzip")


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    assert os.path.exists(CLI), "run __graft_entry__.build() first"
    return nz


def bft(values, shape):
    return b"BFT1" + struct.pack("<B", len(shape)) + b"".join(struct.pack("<Q", d) for d in shape) + \
        np.ascontiguousarray(values, "<u2").tobytes()


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


def fmt6(x):
    return "%.6g" % x


def test_gpu_cli_compress_decompress_analyze(nz, port, tmp_path):
    v = port.gaussian_bf16(5, 300 * 1000, 0.02)
    src = tmp_path / "w.bft"
    src.write_bytes(bft(v, (300, 1000)))
    out = tmp_path / "w.nzt"
    r = run("compress", str(src), str(out))
    assert r.returncode == 0, r.stderr
    blob = nz.compress_lossless(v, nz.TensorMeta((300, 1000)))
    assert out.read_bytes() == nz.write_nzt(blob)
    fp = nz.footprint(blob)
    lines = r.stdout.splitlines()
    assert lines[0] == "section,bytes" and f"total,{fp.total()}" in lines and f"raw,{2 * v.size}" in lines
    assert f"ratio,{fmt6(2 * v.size / fp.total())}" in lines
    back = tmp_path / "back.bft"
    r = run("decompress", str(out), str(back))
    assert r.returncode == 0, r.stderr
    assert back.read_bytes() == src.read_bytes()
    r = run("analyze", str(src), "--hist")
    assert r.returncode == 0, r.stderr
    rep = nz.analyze_tensor(v)
    lines = r.stdout.splitlines()
    assert lines[:6] == ["component,entropy_bits,capacity_bits", f"sign,{fmt6(rep.h_sign)},1",
                         f"exponent,{fmt6(rep.h_exp)},8", f"mantissa,{fmt6(rep.h_mant)},7",
                         f"ideal_ratio,{fmt6(rep.ideal_ratio)},", f"exponent_only_ratio,{fmt6(rep.exponent_only_ratio)},"]
    assert len(lines) == 6 + 2 + 256 + 128


def test_gpu_cli_lossy_and_exit_codes(nz, port, tmp_path):
    v = port.gaussian_bf16(6, 70000, 0.02)
    src = tmp_path / "w.bft"
    src.write_bytes(bft(v, (70000,)))
    out = tmp_path / "w.nzt"
    assert run("compress", str(src), str(out), "-p", "3", "--block-size", "64").returncode == 0
    blob = nz.compress_lossy(v, 3, 64)
    assert out.read_bytes() == nz.write_nzt(blob)
    back = tmp_path / "back.bft"
    assert run("decompress", str(out), str(back)).returncode == 0
    got = np.frombuffer(back.read_bytes()[13 + 8 * 0:], "<u2")[-v.size:]
    assert (got == nz.decompress_lossy(blob)).all()
    bad = bytearray(out.read_bytes())
    bad[len(bad) // 2] ^= 1
    (tmp_path / "bad.nzt").write_bytes(bytes(bad))
    assert run("decompress", str(tmp_path / "bad.nzt"), str(back)).returncode == 4  # ChecksumError
    (tmp_path / "magic.nzt").write_bytes(b"NZT9" + bytes(bad[4:]))
    assert run("decompress", str(tmp_path / "magic.nzt"), str(back)).returncode == 2  # FormatError
    nan = v.copy()
    nan[7] = 0x7FC0
    (tmp_path / "nan.bft").write_bytes(bft(nan, (70000,)))
    assert run("compress", str(tmp_path / "nan.bft"), str(out), "-p", "0").returncode == 3  # NonFiniteError
    assert run("compress", str(src), str(out), "-p", "2").returncode == 2  # usage
    assert run("frobnicate").returncode == 2


def test_gpu_cli_bench(nz):
    r = run("bench", "--sizes", "100000,1000000", "--trials", "2")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "direction,size_bytes,gib_per_s" and len(lines) == 5
    assert all(float(l.split(",")[2]) > 0 for l in lines[1:])
