"""Deterministic synthetic inputs shared by tests, the golden-fixture
generator and bench.py.

Everything is built on the reference's counter RNG (rng.hpp:21-51:
splitmix64 of seed + (i+1)*golden), restated here in vectorised numpy
uint64 arithmetic (wrapping multiply) so byte streams are reproducible
without any library RNG.  Gaussian bf16 tensors need the reference's libm
Box-Muller, so they come from the oracle (``Oracle.gaussian_bf16``)."""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(0xBF58476D1CE4E5B9)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return z


def words(seed: int, n: int, start: int = 0) -> np.ndarray:
    """rng::word(seed, counter) for counter in [start, start+n) (rng.hpp:30-32)."""
    with np.errstate(over="ignore"):
        c = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        return _mix64(np.uint64(seed) + c * GOLDEN)


def uniform(seed: int, n: int) -> np.ndarray:
    """rng::uniform (rng.hpp:40-42): top 53 bits * 2^-53."""
    return (words(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def uniform_bytes(n: int, seed: int) -> np.ndarray:
    return (words(seed, n) & np.uint64(0xFF)).astype(np.uint8)


def zipf_bytes(n: int, seed: int, power: float = 1.0) -> np.ndarray:
    """Symbols with P(s) ~ 1/(1+s)^power over 256 symbols (test_ans.cpp:27-35
    shape), inverse-CDF sampled from rng::uniform."""
    w = 1.0 / (1.0 + np.arange(256, dtype=np.float64)) ** power
    cdf = np.cumsum(w) / w.sum()
    return np.minimum(np.searchsorted(cdf, uniform(seed, n), side="right"), 255).astype(np.uint8)


def counts_of(symbols: np.ndarray) -> np.ndarray:
    return np.bincount(np.asarray(symbols, dtype=np.int64), minlength=256).astype(np.uint64)


def bf16_uniform(n: int, seed: int, half_width: float) -> np.ndarray:
    """U(-a, a) rounded to bf16 (RNE via float32)."""
    x = ((uniform(seed, n) * 2.0 - 1.0) * half_width).astype(np.float32)
    return f32_to_bf16(x)


def bf16_laplace(n: int, seed: int, b: float) -> np.ndarray:
    """Laplace(0, b) by inverse CDF of rng::uniform, rounded to bf16."""
    u = uniform(seed, n) - 0.5
    x = (-b * np.sign(u) * np.log1p(-2.0 * np.abs(u))).astype(np.float32)
    return f32_to_bf16(x)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Bf16::from_float (bitfloat.hpp:25-32) for finite inputs."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (r & np.uint64(0xFFFF)).astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
