"""Counter-based random numbers shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the DeepInverse method.  It only turns
(stream, index) pairs into uniform / normal numbers so that every input of a
run -- measurement matrix Phi, network weights Omega, synthetic images -- is a
pure function of the seed and of the *global* element index.  That makes the
inputs identical on any machine, for any batch sharding over GPUs (SURVEY.md
§8(d) "Seeding"; SPEC.md:181 asks for seeded ensembles).

Generator: splitmix64 (Steele, Lea, Flood 2014) applied to ``key + index``,
53-bit mantissa uniforms, Box-Muller for normals.  Vectorised with numpy
uint64 arithmetic (wrap-around multiplication is the intended semantics).
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 1701
# stream ids: Phi = +1, Omega = +2, images = +3, noise = +4
STREAM_PHI = 1
STREAM_OMEGA = 2
STREAM_IMAGES = 3
STREAM_NOISE = 4

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def stream_key(stream: int, sub: int = 0, seed: int = BASE_SEED) -> np.uint64:
    """64-bit key of a named stream (and an optional sub-stream, e.g. a layer)."""
    with np.errstate(over="ignore"):
        z = np.array([seed], dtype=np.uint64) * _GOLDEN
        z = _mix(z + np.uint64(stream))
        z = _mix(z ^ (np.uint64(sub) * _M1 + np.uint64(0x632BE59BD9B4E019)))
    return np.uint64(z[0])


def bits(key: np.uint64, index: np.ndarray) -> np.ndarray:
    """splitmix64 output for counters ``index`` (uint64 array) under ``key``."""
    index = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (index + np.uint64(1)) * _GOLDEN
    return _mix(z)


def uniform(key: np.uint64, index: np.ndarray) -> np.ndarray:
    """U[0,1) doubles with 53 random bits."""
    return (bits(key, index) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(key: np.uint64, start: int, count: int, chunk: int = 1 << 24) -> np.ndarray:
    """``count`` standard normals for counters start..start+count-1 (fp64).

    Normal i uses the two uniforms at counters 2i and 2i+1 (Box-Muller, cosine
    branch only), so element i never depends on how the range is split.
    """
    out = np.empty(count, dtype=np.float64)
    for s in range(0, count, chunk):
        n = min(chunk, count - s)
        i = np.arange(start + s, start + s + n, dtype=np.uint64)
        u1 = 1.0 - uniform(key, i * np.uint64(2))          # (0, 1]
        u2 = uniform(key, i * np.uint64(2) + np.uint64(1))  # [0, 1)
        out[s:s + n] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return out
