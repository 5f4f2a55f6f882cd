"""Measurement noise of the sensing model (TEST INFRASTRUCTURE, see oracle/__init__.py).

add_noise  y + w, w i.i.d. N(0, sigma^2) per image with 10 log10(||y||^2 / E||w||^2) = snr_db, i.e.
           sigma^2 = ||y||^2 / (M * 10^(snr_db / 10)).  Measurement-domain noise (
           SPEC.md:163-171 add_noise; Table 3 "20 dB noise").
           The standard normals are the counter-based stream synth.rng.normal(noise_key(seed), b*M + i): the
           shared seeded generator (no method arithmetic), which the CUDA path re-implements bit for bit.
"""
from __future__ import annotations

import math

import numpy as np

from synth import rng

STREAM_MEAS_NOISE = 5   # synth.rng stream id of the measurement noise


def noise_key(seed: int) -> np.uint64:
    return rng.stream_key(STREAM_MEAS_NOISE, seed=seed)


def add_noise(y, snr_db: float, seed: int) -> np.ndarray:
    """y [B][M] -> y + w (fp64).  snr_db = +inf returns y unchanged (the noiseless flag)."""
    y = np.asarray(y, np.float64)
    y2 = np.atleast_2d(y)
    if math.isinf(snr_db) and snr_db > 0:
        return y.copy()
    b, m = y2.shape
    energy = np.sum(y2 * y2, axis=1)
    if np.any(energy == 0.0):
        raise ValueError("zero-energy measurement vector (SPEC.md:167 domain error)")
    sigma = np.sqrt(energy / (m * 10.0 ** (snr_db / 10.0)))
    z = rng.normal(noise_key(seed), 0, b * m).reshape(b, m)
    return (y2 + sigma[:, None] * z).reshape(y.shape)
