"""Quality metrics of PAPER.md §5, fp64 (TEST INFRASTRUCTURE, see oracle/__init__.py).

psnr    PAPER.md:165 footnote: PSNR = 10 log10(max_Image^2 / MSE); max_Image is
        the maximum of the ground-truth image, MSE is the
        mean over the N pixels, +inf when MSE = 0.
success PAPER.md:160: phi = 1(||x_hat - x||^2 / ||x||^2 <= 0.1), inclusive.
nmse    ||x_hat - x||^2 / ||x||^2 (the quantity inside success).
rel_l2  ||a - b||_2 / ||b||_2 -- the parity statistic of BASELINE.json north_star.
"""
from __future__ import annotations

import math

import numpy as np


def psnr(xhat, x) -> float:
    xhat = np.asarray(xhat, np.float64).ravel()
    x = np.asarray(x, np.float64).ravel()
    mse = float(np.mean((xhat - x) ** 2))
    peak = float(np.max(x))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(peak * peak / mse)


def nmse(xhat, x) -> float:
    xhat = np.asarray(xhat, np.float64).ravel()
    x = np.asarray(x, np.float64).ravel()
    return float(np.sum((xhat - x) ** 2) / np.sum(x ** 2))


def success(xhat, x) -> int:
    return int(nmse(xhat, x) <= 0.1)


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = float(np.linalg.norm(b))
    d = float(np.linalg.norm(a - b))
    if nb == 0.0:
        return 0.0 if d == 0.0 else math.inf
    return d / nb
