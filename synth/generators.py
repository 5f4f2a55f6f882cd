"""Seeded synthetic inputs with the shapes of the paper's workloads.

Everything here is *input generation*: the measurement matrix Phi, the random
network parameters Omega, piecewise-smooth test images x and their
measurements y = Phi x (the problem statement, §1).  None of the
DeepInverse computation y -> x_hat (§4) lives here; the CUDA
path and the oracle each implement that on their own.

Recipes (BASELINE.json configs):
  * Phi: i.i.d. N(0, 1/M) (variance 1/M), row-major [M][N].
  * Omega: He-normal N(0, 2/fan_in), fan_in = C_in*k*k; biases zero unless a
    test asks for U[-0.1, 0.1] biases.
  * images: Gaussian blobs (added) + constant rectangles (painted over) +
    optional N(0, 0.01) texture noise, clipped to [0, 1], fp32.  ImageNet
     is not available; these stand in for its 64x64 crops.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import rng
from .dtypes import round_bf16

KSIZE = 11                     # PAPER.md:149-151 (§5): every filter is 11x11
WIDTHS = (1, 64, 32, 1)        # channels: x_tilde -> 64 -> 32 -> 1


# --------------------------------------------------------------------------- Phi
def make_phi(m: int, n: int, dtype: str = "f32", seed: int = rng.BASE_SEED,
             rows: tuple[int, int] | None = None) -> np.ndarray:
    """Phi [m][n] fp32, entries N(0, 1/m); ``dtype='bf16'`` rounds them (RNE) to bf16 values.

    ``rows=(r0, r1)`` generates only rows r0..r1-1 (same values as the full matrix).
    """
    r0, r1 = rows if rows is not None else (0, m)
    key = rng.stream_key(rng.STREAM_PHI, seed=seed)
    out = np.empty((r1 - r0, n), dtype=np.float32)
    scale = 1.0 / math.sqrt(m)
    step = max(1, (1 << 24) // max(n, 1))
    for a in range(r0, r1, step):
        b = min(r1, a + step)
        z = rng.normal(key, a * n, (b - a) * n)
        out[a - r0:b - r0] = (z * scale).astype(np.float32).reshape(b - a, n)
    if dtype == "bf16":
        out = round_bf16(out)
    return out


# ------------------------------------------------------------------------ Omega
@dataclass
class Params:
    """Omega = {W_l, b_l}.  W_l: [C_out][C_in][k][k] fp32 taps in the
    true-convolution convention of Eq. (1); b_l: [C_out] (per-channel) or
    [C_out][n1+k-1][n2+k-1] (full map)."""
    w: list
    b: list
    fullmap_bias: bool = False

    def rounded(self, dtype: str) -> "Params":
        if dtype != "bf16":
            return self
        return Params([round_bf16(w) for w in self.w], [np.asarray(b, np.float32) for b in self.b],
                      self.fullmap_bias)


def make_params(widths=WIDTHS, k: int = KSIZE, bias: str = "zero", n1: int = 0, n2: int = 0,
                seed: int = rng.BASE_SEED) -> Params:
    """He-normal weights (BASELINE.json configs), biases 'zero' | 'channel' | 'fullmap'."""
    ws, bs = [], []
    for l in range(len(widths) - 1):
        cin, cout = widths[l], widths[l + 1]
        key = rng.stream_key(rng.STREAM_OMEGA, sub=2 * l, seed=seed)
        sd = math.sqrt(2.0 / (cin * k * k))
        w = (rng.normal(key, 0, cout * cin * k * k) * sd).astype(np.float32)
        ws.append(w.reshape(cout, cin, k, k))
        bkey = rng.stream_key(rng.STREAM_OMEGA, sub=2 * l + 1, seed=seed)
        if bias == "zero":
            bs.append(np.zeros(cout, np.float32))
        elif bias == "channel":
            bs.append((rng.uniform(bkey, np.arange(cout, dtype=np.uint64)) * 0.2 - 0.1).astype(np.float32))
        elif bias == "fullmap":
            h, w_ = n1 + k - 1, n2 + k - 1
            u = rng.uniform(bkey, np.arange(cout * h * w_, dtype=np.uint64))
            bs.append((u * 0.2 - 0.1).astype(np.float32).reshape(cout, h, w_))
        else:
            raise ValueError(bias)
    return Params(ws, bs, fullmap_bias=(bias == "fullmap"))


# ----------------------------------------------------------------------- images
_SLOTS = 8  # uniforms reserved per blob / rectangle


def make_images(n: int, start: int, count: int, n_blobs: int, n_rects: int,
                texture_var: float = 0.0, seed: int = rng.BASE_SEED) -> np.ndarray:
    """``count`` n x n images with global indices start..start+count-1, fp32 in [0,1].

    Blob: centre U[0,n)^2, sigma U[n/16, n/4], amplitude U[0.2, 1.0], added.
    Rectangle: corner U{0..n-1}^2, sides U{ceil(n/16)..ceil(n/3)} (clipped at the
    border), intensity U[0,1], painted over.  Texture: N(0, texture_var) added.
    Then clipped to [0,1].
    """
    key = rng.stream_key(rng.STREAM_IMAGES, seed=seed)
    per_img = (n_blobs + n_rects) * _SLOTS
    g = np.arange(start, start + count, dtype=np.uint64)[:, None]
    yy = np.arange(n, dtype=np.float64)[None, :, None]
    xx = np.arange(n, dtype=np.float64)[None, None, :]
    img = np.zeros((count, n, n), dtype=np.float64)

    def u(slot):
        return rng.uniform(key, g * np.uint64(per_img) + np.uint64(slot))[:, 0][:, None, None]

    for j in range(n_blobs):
        s = j * _SLOTS
        cy, cx = u(s) * n, u(s + 1) * n
        sig = n / 16.0 + u(s + 2) * (n / 4.0 - n / 16.0)
        amp = 0.2 + 0.8 * u(s + 3)
        img += amp * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2.0 * sig * sig))
    lo, hi = math.ceil(n / 16), math.ceil(n / 3)
    for j in range(n_rects):
        s = (n_blobs + j) * _SLOTS
        r0 = np.floor(u(s) * n)
        c0 = np.floor(u(s + 1) * n)
        h = lo + np.floor(u(s + 2) * (hi - lo + 1))
        w = lo + np.floor(u(s + 3) * (hi - lo + 1))
        val = u(s + 4)
        mask = (yy >= r0) & (yy < r0 + h) & (xx >= c0) & (xx < c0 + w)
        img = np.where(mask, val, img)
    if texture_var > 0.0:
        nkey = rng.stream_key(rng.STREAM_NOISE, seed=seed)
        z = rng.normal(nkey, start * n * n, count * n * n).reshape(count, n, n)
        img += math.sqrt(texture_var) * z
    return np.clip(img, 0.0, 1.0).astype(np.float32)


# ------------------------------------------------------------------ measurement
def measure(phi: np.ndarray, x: np.ndarray, dtype: str = "f32", chunk: int = 1024) -> np.ndarray:
    """y = Phi x for every image, fp64 accumulation, then rounded once
    to the path storage type.  x: [B][n1][n2] (row-major vectorisation j = r*n2 + c,
    SURVEY.md §8(c) Q8).  Returns fp32 values [B][M] (bf16-representable if dtype='bf16')."""
    b = x.shape[0]
    xf = x.reshape(b, -1)
    y = np.empty((b, phi.shape[0]), dtype=np.float32)
    phi64 = phi.astype(np.float64) if phi.size * 8 <= (4 << 30) else None
    for a in range(0, b, chunk):
        e = min(b, a + chunk)
        xs = xf[a:e].astype(np.float64)
        if phi64 is not None:
            y[a:e] = (xs @ phi64.T).astype(np.float32)
        else:  # very large Phi: stream it in row blocks to bound host memory
            for r in range(0, phi.shape[0], 2048):
                s = min(phi.shape[0], r + 2048)
                y[a:e, r:s] = (xs @ phi[r:s].astype(np.float64).T).astype(np.float32)
    if dtype == "bf16":
        y = round_bf16(y)
    return y
