"""CPU tests of the product boundary: libnzgpu.so loads, exports every
symbol include/nzgpu.h declares, the ctypes mirror binds all of them, and
without a GPU the data path fails loudly instead of falling back to the CPU."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nzgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(nzgpu_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_2410_20650_b200 as nz

    syms = declared_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", nz.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r" T (nzgpu_\w+)", out.stdout))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    from paper_2410_20650_b200 import nzgpu

    assert sorted(nzgpu.SIGNATURES) == syms


def test_library_is_sm100a_cubin():
    import paper_2410_20650_b200 as nz

    out = subprocess.run(["cuobjdump", "--list-elf", nz.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_sass_uses_tma_bulk_copy():
    """The decode kernel stages payload + LUT with cp.async.bulk (UBLKCP)."""
    import paper_2410_20650_b200 as nz

    sass = subprocess.run(["cuobjdump", "-sass", nz.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass and "SYNCS.PHASECHK.TRANS64.TRYWAIT" in sass


def test_status_strings_and_version():
    from paper_2410_20650_b200 import nzgpu

    assert nzgpu.lib.nzgpu_version() >= 100
    assert b"desynchronization" in nzgpu.lib.nzgpu_status_string(3)


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and os.path.exists("/dev/nvidia0"),
                    reason="a GPU is present")
def test_no_gpu_means_loud_failure_not_cpu_fallback():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(nz.nzgpu.NoDeviceError):
        nz.compress_lossless(np.ones(16, np.uint16))
    with pytest.raises(nz.nzgpu.NoDeviceError):
        nz.build_table(np.ones(256, np.uint64))


def test_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2410_20650_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert not re.search(r"import oracle|from oracle|liboracle|neuzip_oracle|libneuzip_ref", text), f


def test_shannon_entropy_is_the_reference_sum():
    """nzgpu_shannon_entropy (host math behind the drop-in's shannon_entropy,
    entropy.hpp:41-55) sums -p log2 p over the nonzero bins in bin order with
    p = c / total in double -- the reference's exact order, so the result is
    bit-identical to the same loop in Python (both call libm's log2).  Empty
    histograms are invalid_argument.  Host-only: runs without a GPU."""
    import ctypes as C
    import math

    from paper_2410_20650_b200 import nzgpu as N

    rng = np.random.default_rng(5)
    for bins in (1, 2, 7, 128, 256, 1000):
        for _ in range(5):
            c = rng.integers(0, 1 << 40, size=bins).astype(np.uint64)
            c[rng.random(bins) < 0.3] = 0
            if c.sum() == 0:
                c[0] = 1
            h = C.c_double()
            assert N.lib.nzgpu_shannon_entropy(c.ctypes.data, bins, C.byref(h)) == 0
            n = float(int(c.sum()))
            want = 0.0
            for x in c.tolist():
                if x:
                    p = float(x) / n
                    want -= p * math.log2(p)
            want = 0.0 if want < 0.0 else want
            assert h.value == want
    h = C.c_double()
    z = np.zeros(4, np.uint64)
    assert N.lib.nzgpu_shannon_entropy(z.ctypes.data, 4, C.byref(h)) == N.INVALID_ARGUMENT
    assert N.lib.nzgpu_shannon_entropy(None, 0, C.byref(h)) == N.INVALID_ARGUMENT


def test_host_tier_entry_points_reject_bad_arguments_without_a_device():
    """The chunk-export and sections entry points validate their arguments
    before any CUDA call (so these run on a GPU-less machine too)."""
    import ctypes as C

    from paper_2410_20650_b200 import nzgpu as N

    lens = (C.c_uint32 * 4)()
    assert N.lib.nzgpu_blob_chunks(None, lens, lens) == N.INVALID_ARGUMENT
    assert N.lib.nzgpu_blob_export_chunks(None, None, None, None, None, None) == N.INVALID_ARGUMENT
    assert N.lib.nzgpu_decompress_host_sections(None, None) == N.INVALID_ARGUMENT
    t = N.HostSections() if hasattr(N, "HostSections") else None
    if t is not None:
        t.n, t.precision = 10, 5  # invalid precision
        assert N.lib.nzgpu_decompress_host_sections(C.byref(t), None) == N.INVALID_ARGUMENT
