"""Shared helpers for the GPU parity tests: seeded inputs (synth), the CUDA path through the C ABI, and the
oracle on the same input bits."""
from __future__ import annotations

import numpy as np

import oracle
import synth

# BASELINE.json north_star tolerances
TOL_REL_L2 = {"f32": 1e-5, "tf32": 2e-2, "bf16": 2e-2}
TOL_DPSNR = 0.05


class Case:
    """Inputs of one workload in the exact values both sides consume."""

    def __init__(self, n1, n2, m, batch, precision, n_blobs=8, n_rects=4, texture=0.0, bias="zero", start=0,
                 params=None):
        self.n1, self.n2, self.m, self.batch, self.precision = n1, n2, m, batch, precision
        st = "bf16" if precision == "bf16" else "f32"
        self.phi = synth.make_phi(m, n1 * n2, st)
        n = max(n1, n2)
        self.x = synth.make_images(n, start, batch, n_blobs, n_rects, texture)[:, :n1, :n2].copy()
        self.y = synth.measure(self.phi, self.x, st)
        p = params if params is not None else synth.make_params(bias=bias, n1=n1, n2=n2)
        self.params = p.rounded(st)

    def oracle(self, idx, final_relu=False, xcorr=False):
        return oracle.forward(self.y[idx], self.phi, self.params, self.n1, self.n2, final_relu=final_relu,
                              xcorr=xcorr)


def make_ctx(case: Case, flags=0, max_batch=None, device=0):
    from paper_1701_03891_b200 import DeepInverse
    return DeepInverse(case.phi, case.params, case.n1, case.n2, case.precision, flags=flags, device=device,
                       max_batch=max_batch or case.batch)


def y_device(case: Case, ctx, rows=None):
    import torch
    y = case.y if rows is None else case.y[rows]
    return torch.from_numpy(np.ascontiguousarray(y)).to(device="cuda", dtype=ctx.storage_dtype)


def run(case: Case, ctx, rows=None) -> np.ndarray:
    import torch
    y = y_device(case, ctx, rows)
    out = ctx.recover(y)
    torch.cuda.synchronize()
    return out.cpu().numpy()


# Element-wise bound on the whole path (on top of the per-image rel-L2 of north_star): max |gpu - ref| over the pixels
# of an image, relative to max |ref| of that image.  A single wrong output pixel (|ref_p| ~ rms ~ max/3) fails it at
# every image size, where rel-L2 dilutes it by 1/sqrt(N).  Calibrated on the green B200 run r02a over every
# compare() call of the suite (profiles/r02_parity_calibration.json): observed maxima bf16 7.2e-3, tf32 5.7e-3,
# fp32 1.1e-6 -- about 2x (bf16/tf32) and 5x (fp32) below these bounds.
TOL_PIX = {"f32": 5e-6, "tf32": 1.5e-2, "bf16": 1.5e-2}


def compare(gpu, ref, x, precision):
    """Per image rel-L2 and |dPSNR| (PAPER.md:165 PSNR, peak = max of ground truth); asserts the element-wise bound
    TOL_PIX.  Returns (max rel-L2, max |dPSNR|, mean dPSNR)."""
    import json
    import os
    rel = [oracle.rel_l2(g, r) for g, r in zip(gpu, ref)]
    pix = [float(np.max(np.abs(np.asarray(g, np.float64) - r)) / max(float(np.max(np.abs(r))), 1e-30))
           for g, r in zip(gpu, ref)]
    dps = [abs(oracle.psnr(g, t) - oracle.psnr(r, t)) for g, r, t in zip(gpu, ref, x)]
    if os.environ.get("DI_PARITY_LOG"):
        with open(os.environ["DI_PARITY_LOG"], "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "?"), "precision": precision,
                                "rel_l2": max(rel), "pix": max(pix), "dpsnr": max(dps)}) + "\n")
    worst = int(np.argmax(pix))
    assert pix[worst] <= TOL_PIX[precision], (f"image {worst}: max |gpu - ref| = {pix[worst]:.3g} x max|ref| > "
                                              f"{TOL_PIX[precision]}")
    return max(rel), max(dps), float(np.mean([oracle.psnr(g, t) for g, t in zip(gpu, x)]) -
                                     np.mean([oracle.psnr(r, t) for r, t in zip(ref, x)]))


def sample_rows(batch, k):
    """Deterministic sample: the first k/2 and last k/2 images (and all when batch <= k)."""
    if batch <= k:
        return np.arange(batch)
    h = k // 2
    return np.concatenate([np.arange(h), np.arange(batch - h, batch)])
