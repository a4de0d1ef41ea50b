"""Golden case catalogue: deterministic inputs whose reference outputs are
frozen in tests/golden/golden.json by tests/golden/make_golden.py (run where
the reference is mounted; it uses oracle/_ref = the unmodified reference
headers).  The CPU tests pin the C restatement against these fixtures, and
the GPU tests pin the CUDA path against the same fixtures.

Each case names the reference test it mirrors (proj/tests/...)."""
from __future__ import annotations

import numpy as np

from tests import inputs

CHUNK = 65536


def _patterns():
    return np.arange(65536, dtype=np.uint32).astype(np.uint16)


# (name, generator(oracle) -> bf16 values, chunk_symbols, mirrors)
def lossless_cases():
    g = lambda seed, n, sigma=0.02: (lambda o: o.gaussian_bf16(seed, n, sigma))
    return [
        ("gauss_n1", g(42, 1), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_n2", g(42, 2), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_n999", g(42, 999), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_n65535", g(42, 65535), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_n65536", g(42, 65536), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_n65537", g(42, 65537), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_n200000", g(42, 200000), CHUNK, "test_ans.cpp:195-218 lengths"),
        ("gauss_1m_seed42", g(42, 1 << 20), CHUNK, "test_tensorstore.cpp:69-82, acceptance crit 3"),
        ("gauss_5000_s3_sigma01", g(3, 5000, 0.1), CHUNK, "test_tensorstore.cpp:84-93"),
        ("all_patterns", lambda o: _patterns(), CHUNK, "test_tensorstore.cpp:40-53"),
        ("nan_inf", lambda o: np.array([0x7FC1, 0xFF80, 0x7F80, 0x0001, 0x8000], np.uint16), CHUNK,
         "test_tensorstore.cpp:55-60"),
        ("const_1m", lambda o: np.full(1 << 20, 0x3F80, np.uint16), CHUNK, "test_tensorstore.cpp:62-67"),
        ("const16", lambda o: np.full(16, 0x3F80, np.uint16), CHUNK, "gen_golden.cpp:34-41"),
        ("uniform_bf16_300k", lambda o: inputs.bf16_uniform(300000, 5, 0.02 * 3 ** 0.5), CHUNK, "C5 uniform"),
        ("laplace_bf16_300k", lambda o: inputs.bf16_laplace(300000, 6, 0.02 / 2 ** 0.5), CHUNK, "C5 heavy-tailed"),
        # chunk-size sweep (C5 / probe P10): ans_encode_chunk composed over S-spans
        ("gauss_1m_S1024", g(42, 1 << 20), 1024, "C5 chunk sweep"),
        ("gauss_1m_S16384", g(42, 1 << 20), 16384, "C5 chunk sweep"),
        ("gauss_1m_S131072", g(42, 1 << 20), 131072, "C5 chunk sweep"),
        ("gauss_1m_S1048576", g(42, 1 << 20), 1 << 20, "C5 chunk sweep"),
        ("gauss_300k_S100000", g(9, 300000), 100000, "C5 chunk sweep, S not a power of two"),
    ]


def coder_cases():
    """Symbol streams for the raw coder (ans_encode / ans_decode)."""
    return [
        ("uniform_1m", lambda: inputs.uniform_bytes(1 << 20, 99), "test_ans.cpp:172-181"),
        ("zipf_1m", lambda: inputs.zipf_bytes(1 << 20, 6), "test_ans.cpp:183-193"),
        ("const31_1m", lambda: np.full(1 << 20, 31, np.uint8), "test_ans.cpp:183-193"),
        ("const7_100k", lambda: np.full(100000, 7, np.uint8), "test_ans.cpp:156-162"),
        ("zipf_200k", lambda: inputs.zipf_bytes(200000, 8), "test_ans.cpp:220-229"),
        ("zipf_1000000", lambda: inputs.zipf_bytes(1000000, 44), "test_ans.cpp:213-216"),
        ("zipf2_200k", lambda: inputs.zipf_bytes(200000, 12, power=2.0), "probe P6b: 2-byte renorms"),
        ("uniform_150001", lambda: inputs.uniform_bytes(150001, 13), "probe P6b: partial last chunk"),
        ("zipf3_70000", lambda: inputs.zipf_bytes(70000, 14, power=3.0), "many tiny frequencies"),
    ]


def lossy_cases():
    g = lambda seed, n, sigma=0.02: (lambda o: o.gaussian_bf16(seed, n, sigma))
    f = lambda vals: (lambda o: inputs.f32_to_bf16(np.array(vals, np.float32)))
    cases = []
    for k in (0, 1, 3):
        cases += [
            (f"gauss100k_k{k}_B512", g(7, 100000), k, 512, "test_tensorstore.cpp:141-169"),
            (f"gauss2048_s11_k{k}_B64", g(11, 2048, 0.3), k, 64, "test_tensorstore.cpp:171-185"),
            (f"gauss1000_k{k}_B1", g(5, 1000, 0.05), k, 1, "test_tensorstore.cpp:133-139"),
            (f"one_half_k{k}", f([1.0, 0.5]), k, 512, "test_tensorstore.cpp:104-112"),
            (f"gauss70000_k{k}_B100", g(21, 70000), k, 100, "block not dividing chunk"),
            (f"patterns_finite_k{k}_B37", lambda o: _finite_patterns(), k, 37, "all finite bf16"),
        ]
    cases += [
        ("m175_03_k0", f([-1.75, 0.3]), 0, 512, "test_tensorstore.cpp:114-131"),
        ("zeros2000_k1", lambda o: np.zeros(2000, np.uint16), 1, 512, "test_tensorstore.cpp:187-191"),
        ("gauss65536_k1_B32", g(17, 1 << 16), 1, 32, "test_tensorstore.cpp:217-240"),
        ("gauss65536_k3_B512", g(13, 1 << 16), 3, 512, "test_tensorstore.cpp:205-215"),
    ]
    return cases


def _finite_patterns():
    p = _patterns()
    return p[(p & 0x7F80) != 0x7F80]


def table_cases():
    """(name, counts u64[256]) for build_table (test_ans.cpp:48-117)."""
    out = []
    c = np.zeros(256, np.uint64); c[42] = 4096; out.append(("single42", c))
    out.append(("uniform1000", np.full(256, 1000, np.uint64)))
    c = np.zeros(256, np.uint64); c[0] = 3; c[1] = 1; out.append(("three_one", c))
    c = np.zeros(256, np.uint64); c[0] = 4095; c[1] = 1; out.append(("split4095_1", c))
    c = np.zeros(256, np.uint64); c[9] = 5; c[200] = 11; out.append(("nine_200", c))
    out.append(("uniform7", np.full(256, 7, np.uint64)))
    w = inputs.words(3, 256 * 60)
    for t in range(50):  # test_ans.cpp:78-89 shape: 100 + r % 1000
        out.append((f"rand_dense_{t}", (np.uint64(100) + w[t * 256:(t + 1) * 256] % np.uint64(1000)).astype(np.uint64)))
    w = inputs.words(17, 4096 * 100)
    for t in range(100):  # test_ans.cpp:92-117 shape: huge and tiny counts mixed
        r = w[t * 4096:(t + 1) * 4096]
        c = np.zeros(256, np.uint64)
        present = 1 + int(r[0] % np.uint64(256))
        for i in range(present):
            s = int(r[1 + 3 * i] % np.uint64(256))
            c[s] += np.uint64(1) if int(r[2 + 3 * i]) & 1 else r[3 + 3 * i] % np.uint64(1000000)
            if c[s] == 0:
                c[s] = 1
        out.append((f"rand_repair_{t}", c))
    return out


# NZT containers (tensorstore.hpp:289-477): (name, generator, shape, precision, block)
def nzt_cases():
    g = lambda seed, n, sigma=0.02: (lambda o: o.gaussian_bf16(seed, n, sigma))
    return [
        ("const16_k7", lambda o: np.full(16, 0x3F80, np.uint16), (16,), 7, 0),
        ("gauss_4x4096_k7", g(42, 4 * 4096), (4, 4096), 7, 0),
        ("gauss_300k_k7", g(8, 300000), (300, 1000), 7, 0),
        ("gauss_2x3x7x1000_k7", g(9, 42000), (2, 3, 7, 1000), 7, 0),
        ("gauss_70000_k3_B512", g(10, 70000), (70000,), 3, 512),
        ("gauss_70000_k1_B100", g(11, 70000), (700, 100), 1, 100),
        ("gauss_70000_k0_B37", g(12, 70000), (70000,), 0, 37),
    ]
