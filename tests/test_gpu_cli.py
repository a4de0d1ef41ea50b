"""GPU: the `neuzip` CLI (tools/neuzip_cli.cpp) against text and files the
REFERENCE codec produces (oracle/_ref: the unmodified reference headers;
the C restatement where it is not built) -- not against this repo's own API.

Pinned per subcommand of proj/tools/neuzip.cpp:
  analyze     CSV = the reference's analyze_tensor doubles (entropy.hpp:89-94)
              formatted %.6g, histogram bins = numpy counts (neuzip.cpp:40-65);
  compress    the .nzt file is byte-identical to the reference's write_nzt,
              and the footprint CSV is the reference blob's section sizes
              (tensorstore.hpp:242-287, neuzip.cpp:67-96);
  decompress  lossless: the original .bft back; lossy: the reference's
              decompress_lossy values (neuzip.cpp:98-115);
  exit codes  2 usage / FormatError, 3 NonFiniteError, 4 ChecksumError
              (neuzip.cpp:324-339)."""
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


@pytest.fixture(scope="module")
def refc():
    from oracle.oracle import Oracle, ref_available

    return Oracle("ref") if ref_available() else Oracle("port")


def bft(values, shape):
    return b"BFT1" + struct.pack("<B", len(shape)) + b"".join(struct.pack("<Q", d) for d in shape) + \
        np.ascontiguousarray(values, "<u2").tobytes()


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


def g6(x):
    return "%.6g" % x


def footprint_lines(n, stream_len, mant_len, scales_len, ndim):
    header = 35 + 8 * ndim
    total = stream_len + mant_len + scales_len + 512 + header
    return ["section,bytes", f"exponent,{stream_len}", f"mantissa,{mant_len}", f"scales,{scales_len}", "table,512",
            f"header,{header}", f"total,{total}", f"raw,{2 * n}", f"ratio,{g6(2 * n / total)}"]


def test_gpu_cli_lossless_against_reference(nz, port, refc, tmp_path):
    shape = (300, 1000)
    v = port.gaussian_bf16(5, 300 * 1000, 0.02)
    src = tmp_path / "w.bft"
    src.write_bytes(bft(v, shape))
    out = tmp_path / "w.nzt"
    r = run("compress", str(src), str(out))
    assert r.returncode == 0, r.stderr
    assert out.read_bytes() == refc.write_nzt_lossless(v, shape)
    f, s, m = refc.compress_lossless(v)
    assert r.stdout.splitlines() == footprint_lines(v.size, len(s), m.size, 0, 2)
    back = tmp_path / "back.bft"
    r = run("decompress", str(out), str(back))
    assert r.returncode == 0, r.stderr
    assert back.read_bytes() == src.read_bytes()


def test_gpu_cli_analyze_against_reference(nz, refc, port, tmp_path):
    v = port.gaussian_bf16(9, 65536 * 3 + 11, 0.05)
    src = tmp_path / "a.bft"
    src.write_bytes(bft(v, (v.size,)))
    r = run("analyze", str(src), "--hist")
    assert r.returncode == 0, r.stderr
    hs, he, hm, ideal, exp_only = refc.entropy_report(v)
    want = ["component,entropy_bits,capacity_bits", f"sign,{g6(hs)},1", f"exponent,{g6(he)},8",
            f"mantissa,{g6(hm)},7", f"ideal_ratio,{g6(ideal)},", f"exponent_only_ratio,{g6(exp_only)},"]
    sign = np.bincount(v >> 15, minlength=2)
    exp = np.bincount((v >> 7) & 0xFF, minlength=256)
    mant = np.bincount(v & 0x7F, minlength=128)
    want += [f"hist_sign_{i},{c}," for i, c in enumerate(sign)]
    want += [f"hist_exp_{i},{c}," for i, c in enumerate(exp)]
    want += [f"hist_mant_{i},{c}," for i, c in enumerate(mant)]
    assert r.stdout.splitlines() == want


@pytest.mark.parametrize("k,block", [(3, 64), (0, 512), (1, 100)])
def test_gpu_cli_lossy_against_reference(nz, port, refc, tmp_path, k, block):
    v = port.gaussian_bf16(6 + k, 70000, 0.02)
    src = tmp_path / "w.bft"
    src.write_bytes(bft(v, (70000,)))
    out = tmp_path / "w.nzt"
    r = run("compress", str(src), str(out), "-p", str(k), "--block-size", str(block))
    assert r.returncode == 0, r.stderr
    assert out.read_bytes() == refc.write_nzt_lossy(v, (70000,), k, block)
    f, sc, s, pk = refc.compress_lossy(v, k, block)
    assert r.stdout.splitlines() == footprint_lines(v.size, len(s), pk.size, sc.size, 1)
    back = tmp_path / "back.bft"
    assert run("decompress", str(out), str(back)).returncode == 0
    got = np.frombuffer(back.read_bytes()[5 + 8:], "<u2")
    assert (got == refc.decompress_lossy(f, sc, s, pk, k, block, v.size)).all()


def test_gpu_cli_exit_codes(nz, port, refc, tmp_path):
    v = port.gaussian_bf16(6, 70000, 0.02)
    src = tmp_path / "w.bft"
    src.write_bytes(bft(v, (70000,)))
    good = refc.write_nzt_lossy(v, (70000,), 3, 64)  # a file the REFERENCE wrote
    back = tmp_path / "back.bft"
    (tmp_path / "good.nzt").write_bytes(good)
    assert run("decompress", str(tmp_path / "good.nzt"), str(back)).returncode == 0
    bad = bytearray(good)
    bad[len(bad) // 2] ^= 1
    (tmp_path / "bad.nzt").write_bytes(bytes(bad))
    assert run("decompress", str(tmp_path / "bad.nzt"), str(back)).returncode == 4  # ChecksumError
    (tmp_path / "magic.nzt").write_bytes(b"NZT9" + bytes(bad[4:]))
    assert run("decompress", str(tmp_path / "magic.nzt"), str(back)).returncode == 2  # FormatError
    (tmp_path / "short.nzt").write_bytes(good[:100])
    assert run("decompress", str(tmp_path / "short.nzt"), str(back)).returncode == 2
    nan = v.copy()
    nan[7] = 0x7FC0
    (tmp_path / "nan.bft").write_bytes(bft(nan, (70000,)))
    out = tmp_path / "o.nzt"
    assert run("compress", str(tmp_path / "nan.bft"), str(out), "-p", "0").returncode == 3  # NonFiniteError
    assert run("compress", str(src), str(out), "-p", "2").returncode == 2  # not in {0,1,3,7}
    assert run("compress", str(src), str(out), "--block-size", "0", "-p", "3").returncode == 2
    assert run("compress", str(src)).returncode == 2
    (tmp_path / "trunc.bft").write_bytes(bft(v, (70001,)))
    assert run("compress", str(tmp_path / "trunc.bft"), str(out)).returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("analyze", str(src), "--bogus").returncode == 2
    assert run("train-demo").returncode == 2
    assert run("--help").returncode == 0


def test_gpu_cli_bench(nz):
    r = run("bench", "--sizes", "100000,1000000", "--trials", "2")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "direction,size_bytes,gib_per_s" and len(lines) == 5
    assert [l.split(",")[:2] for l in lines[1:]] == [["compress", "100000"], ["decompress", "100000"],
                                                       ["compress", "1000000"], ["decompress", "1000000"]]
    assert all(float(l.split(",")[2]) > 0 for l in lines[1:])
    assert run("bench", "--sizes", "100").returncode == 2
    assert run("bench", "--trials", "0").returncode == 2
