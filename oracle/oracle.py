"""ctypes wrapper over oracle/di_oracle.c (TEST INFRASTRUCTURE, see oracle/__init__.py).

Inputs are upcast to fp64 from the exact values the GPU path received, so the
oracle evaluates the same mathematical function on the same input bits.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "di_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O3 -fopenmp, no intrinsics) if missing or stale."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib_path() -> str:
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER(ctypes.c_double)
        I = ctypes.c_int
        lib.dio_proxy.argtypes = [I, I, I, P, P, P]
        lib.dio_measure.argtypes = [I, I, I, P, P, P]
        lib.dio_train_grad.argtypes = [I, I, I, I, I, ctypes.POINTER(I), I, P, P, P, P, P, I, ctypes.c_double, P, P,
                                       P, I]
        lib.dio_conv_layer.argtypes = [I, I, I, I, I, P, P, P, I, I, I, P]
        lib.dio_forward.argtypes = [I, I, I, I, I, ctypes.POINTER(I), I, P, P, P, P, I, I, I, P, I]
        for f in (lib.dio_proxy, lib.dio_measure, lib.dio_conv_layer, lib.dio_forward, lib.dio_train_grad):
            f.restype = I
        _lib = lib
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def measure(phi, x) -> np.ndarray:
    """y = Phi x for x [B][n1][n2] (or [B][N]) -> [B][M]."""
    phi = _d(phi)
    m, n = phi.shape
    x = _d(np.asarray(x).reshape(-1, n))
    out = np.empty((x.shape[0], m), np.float64)
    rc = _load().dio_measure(m, n, x.shape[0], _p(phi), _p(x), _p(out))
    if rc:
        raise ValueError(f"dio_measure status {rc}")
    return out


def proxy(phi, y) -> np.ndarray:
    """x_tilde = Phi^T y for y [B][M] -> [B][N]."""
    phi, y = _d(phi), _d(np.atleast_2d(y))
    m, n = phi.shape
    out = np.empty((y.shape[0], n), np.float64)
    rc = _load().dio_proxy(m, n, y.shape[0], _p(phi), _p(y), _p(out))
    if rc:
        raise ValueError(f"dio_proxy status {rc}")
    return out


def conv_layer(x, w, b=None, relu=True, xcorr=False, fullmap_bias=False) -> np.ndarray:
    """Eq. (1) layer on X [C_in][n1][n2] with W [C_out][C_in][k][k]."""
    x, w = _d(x), _d(w)
    cin, n1, n2 = x.shape
    cout, cin2, k, k2 = w.shape
    if cin2 != cin or k2 != k:
        raise ValueError("shape mismatch")
    bb = _d(b) if b is not None else None
    out = np.empty((cout, n1, n2), np.float64)
    rc = _load().dio_conv_layer(cin, cout, n1, n2, k, _p(x), _p(w), _p(bb), int(fullmap_bias),
                                int(relu), int(xcorr), _p(out))
    if rc:
        raise ValueError(f"dio_conv_layer status {rc}")
    return out


def forward(y, phi, params, n1, n2, final_relu=False, xcorr=False, threads=None) -> np.ndarray:
    """x_hat = M(y, Omega) for y [B][M]; returns [B][n1][n2] fp64.

    params: synth.Params-like (w: list of [C_out][C_in][k][k], b: list, fullmap_bias)."""
    y = _d(np.atleast_2d(y))
    phi = _d(phi)
    m = phi.shape[0]
    ws = [np.asarray(w) for w in params.w]
    widths = [ws[0].shape[1]] + [w.shape[0] for w in ws]
    k = ws[0].shape[-1]
    w_all = _d(np.concatenate([w.ravel() for w in ws]))
    has_bias = params.b is not None and any(np.any(np.asarray(b) != 0) for b in params.b)
    b_all = _d(np.concatenate([np.asarray(b).ravel() for b in params.b])) if has_bias else None
    wid = (ctypes.c_int * len(widths))(*widths)
    out = np.empty((y.shape[0], n1, n2), np.float64)
    if threads is None:
        threads = os.cpu_count() or 1
    rc = _load().dio_forward(y.shape[0], m, n1, n2, len(ws), wid, k, _p(phi), _p(y), _p(w_all),
                             _p(b_all), int(bool(params.fullmap_bias)), int(final_relu), int(xcorr),
                             _p(out), int(threads))
    if rc:
        raise ValueError(f"dio_forward status {rc}")
    return out


def train_grad(y, x, phi, params, n1, n2, scale=None, final_relu=False, threads=None):
    """Loss scale * sum_b ||M(y_b) - x_b||^2 (scale defaults to 1/batch) and its gradient with respect
    to the weights ([C_out][C_in][k][k] per layer, true-convolution orientation) and per-channel biases.
    Returns (loss, [dW1, dW2, dW3], [db1, db2, db3])."""
    y = _d(np.atleast_2d(y))
    x = _d(np.asarray(x).reshape(y.shape[0], -1))
    phi = _d(phi)
    ws = [np.asarray(w) for w in params.w]
    widths = [ws[0].shape[1]] + [w.shape[0] for w in ws]
    k = ws[0].shape[-1]
    w_all = _d(np.concatenate([w.ravel() for w in ws]))
    b_all = _d(np.concatenate([np.asarray(b).ravel() for b in params.b])) if params.b is not None else None
    if params.b is not None and b_all.size != sum(widths[1:]):
        raise ValueError("training gradients need per-channel biases")
    gw = np.empty_like(w_all)
    gb = np.empty(sum(widths[1:]), np.float64)
    loss = np.zeros(1, np.float64)
    wid = (ctypes.c_int * len(widths))(*widths)
    if scale is None:
        scale = 1.0 / y.shape[0]
    if threads is None:
        threads = os.cpu_count() or 1
    rc = _load().dio_train_grad(y.shape[0], phi.shape[0], n1, n2, len(ws), wid, k, _p(phi), _p(y), _p(x), _p(w_all),
                                _p(b_all), int(final_relu), float(scale), _p(gw), _p(gb), _p(loss), int(threads))
    if rc:
        raise ValueError(f"dio_train_grad status {rc}")
    dws, dbs, o, ob = [], [], 0, 0
    for w in ws:
        dws.append(gw[o:o + w.size].reshape(w.shape))
        dbs.append(gb[ob:ob + w.shape[0]])
        o += w.size
        ob += w.shape[0]
    return float(loss[0]), dws, dbs
