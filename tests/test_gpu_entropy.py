"""GPU: component histograms and the entropy report (entropy.hpp:17-94,
SURVEY §8(f) rank 3) against numpy counts, the unmodified reference (exact
doubles) and the reference's checked-in golden CSV."""
import os

import numpy as np
import pytest

from tests import inputs

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def nz():
    import paper_2410_20650_b200 as nz

    if nz.nzgpu.device_count() == 0:
        pytest.fail("no CUDA device visible to a gpu-marked test")
    return nz


def _cases(port):
    pats = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    return {
        "gauss_1m": port.gaussian_bf16(42, 1 << 20),
        "gauss_odd": port.gaussian_bf16(3, 100003, 0.3),
        "patterns": pats,
        "const": np.full(777, 0x3F80, np.uint16),
        "uniform": inputs.bf16_uniform(50001, 4, 0.05),
        "one": np.array([0xC0A0], np.uint16),
    }


def test_gpu_component_histogram_matches_numpy(nz, port):
    import torch

    for name, v in _cases(port).items():
        t = torch.from_numpy(v.view(np.int16)).cuda()
        s, e, m = nz.component_histogram(t)
        assert (s == np.bincount(v >> 15, minlength=2)).all(), name
        assert (e == np.bincount((v >> 7) & 0xFF, minlength=256)).all(), name
        assert (m == np.bincount(v & 0x7F, minlength=128)).all(), name


def test_gpu_entropy_report_matches_reference(nz, port, ref):
    import torch

    for name, v in _cases(port).items():
        want = ref.entropy_report(v)
        got = nz.analyze_tensor(v)
        assert [got.h_sign, got.h_exp, got.h_mant, got.ideal_ratio, got.exponent_only_ratio] == list(want), name
        got_d = nz.analyze_tensor(torch.from_numpy(v.view(np.int16)).cuda())
        assert got_d == got, name


def test_gpu_entropy_golden_csv(nz, port):
    """gen_golden.cpp:22-33: the reference's checked-in gaussian_entropy.csv."""
    r = nz.analyze_tensor(port.gaussian_bf16(42, 1 << 20))
    text = ("sign,%.6g\nexponent,%.6g\nmantissa,%.6g\nideal_ratio,%.6g\nexponent_only_ratio,%.6g\n"
            % (r.h_sign, r.h_exp, r.h_mant, r.ideal_ratio, r.exponent_only_ratio))
    with open(os.path.join(HERE, "golden", "gaussian_entropy.csv")) as fh:
        assert text == fh.read()


def test_gpu_entropy_empty_raises(nz):
    with pytest.raises(ValueError):
        nz.analyze_tensor(np.zeros(0, np.uint16))
