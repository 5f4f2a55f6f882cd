"""Pins for oracle.forward, x_hat = M(y, Omega) -- CPU only."""
import json
import math
import os

import numpy as np
import pytest
import scipy.signal

import oracle
import synth

RNG = np.random.default_rng(5)
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _torch_pipeline(y, phi, params, n1, n2, final_relu):
    """Independent fp64 composition with torch library ops (matmul + conv2d)."""
    torch = pytest.importorskip("torch")
    t = torch.from_numpy(np.asarray(y, np.float64)) @ torch.from_numpy(np.asarray(phi, np.float64))
    a = t.reshape(-1, 1, n1, n2)
    L = len(params.w)
    for l, (w, b) in enumerate(zip(params.w, params.b)):
        wt = torch.from_numpy(np.asarray(w, np.float64)).flip(-1, -2)
        a = torch.nn.functional.conv2d(a, wt, torch.from_numpy(np.asarray(b, np.float64)), padding=w.shape[-1] // 2)
        if l < L - 1 or final_relu:
            a = a.relu()
    return a[:, 0].numpy()


@pytest.mark.parametrize("n1,n2,m", [(16, 16, 64), (9, 13, 40), (5, 5, 25)])
@pytest.mark.parametrize("final_relu", [False, True])
def test_forward_vs_torch_composition(n1, n2, m, final_relu):
    phi = synth.make_phi(m, n1 * n2).astype(np.float64)
    params = synth.make_params(bias="channel")
    x = synth.make_images(max(n1, n2), 0, 3, 4, 1)[:, :n1, :n2]
    y = phi @ x.reshape(3, -1).T
    got = oracle.forward(y.T, phi, params, n1, n2, final_relu=final_relu)
    ref = _torch_pipeline(y.T, phi, params, n1, n2, final_relu)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


def test_forward_equals_layer_composition_fullmap_bias():
    n = 12
    phi = synth.make_phi(50, n * n).astype(np.float64)
    params = synth.make_params(bias="fullmap", n1=n, n2=n)
    y = RNG.standard_normal((2, 50))
    got = oracle.forward(y, phi, params, n, n)
    for i in range(2):
        a = oracle.proxy(phi, y[i]).reshape(1, n, n)
        for l in range(3):
            a = oracle.conv_layer(a, params.w[l], params.b[l], relu=(l < 2), fullmap_bias=True)
        assert np.array_equal(got[i], a[0])


def test_zero_omega_and_zero_y():
    n = 8
    phi = synth.make_phi(20, n * n).astype(np.float64)
    p0 = synth.Params([np.zeros_like(w) for w in synth.make_params().w], [np.zeros(c) for c in (64, 32, 1)])
    assert np.all(oracle.forward(RNG.standard_normal((2, 20)), phi, p0, n, n) == 0)
    assert np.all(oracle.forward(np.zeros((2, 20)), phi, synth.make_params(), n, n) == 0)


def test_positive_homogeneity_bitwise():
    """With zero biases M(2y) = 2 M(y) exactly: scaling by 2 is exact in binary floating point."""
    n = 16
    phi = synth.make_phi(64, n * n).astype(np.float64)
    params = synth.make_params()
    y = RNG.standard_normal((2, 64))
    assert np.array_equal(oracle.forward(2 * y, phi, params, n, n), 2 * oracle.forward(y, phi, params, n, n))


def _gauss(k=11, s=1.5):
    a = np.arange(k) - k // 2
    g = np.exp(-(a[:, None] ** 2 + a[None, :] ** 2) / (2 * s * s))
    return g / g.sum()


def structured_params():
    """W1[0] = normalised Gaussian, W2[0][0] = delta, W3[0][0] = delta, all else 0."""
    ws = [np.zeros_like(w, dtype=np.float64) for w in synth.make_params().w]
    ws[0][0, 0] = _gauss()
    ws[1][0, 0, 5, 5] = 1.0
    ws[2][0, 0, 5, 5] = 1.0
    return synth.Params(ws, [np.zeros(64), np.zeros(32), np.zeros(1)])


def test_structured_weights_reduce_to_blur_of_backprojection():
    """Closed form: x_hat = ReLU(G * Phi^T y), G a symmetric Gaussian (textbook blur, scipy)."""
    n, m = 32, 256
    phi = synth.make_phi(m, n * n).astype(np.float64)
    x = synth.make_images(n, 0, 2, 8, 4)
    y = (phi @ x.reshape(2, -1).T).T
    got = oracle.forward(y, phi, structured_params(), n, n)
    for i in range(2):
        xt = (y[i] @ phi).reshape(n, n)
        ref = np.maximum(scipy.signal.convolve2d(xt, _gauss(), mode="same"), 0)
        np.testing.assert_allclose(got[i], ref, rtol=0, atol=1e-12)
        assert -20 < oracle.psnr(got[i], x[i]) < 40


@pytest.mark.parametrize("m", [1, 7, 256])
def test_output_shape_is_image_for_every_m(m):
    n1, n2 = 16, 16
    phi = synth.make_phi(m, n1 * n2).astype(np.float64)
    out = oracle.forward(RNG.standard_normal((1, m)), phi, synth.make_params(), n1, n2)
    assert out.shape == (1, n1, n2) and np.all(np.isfinite(out))


def test_m_greater_than_n_is_domain_error():
    with pytest.raises(ValueError):
        oracle.forward(np.zeros((1, 5)), np.zeros((5, 4)), synth.make_params(), 2, 2)


def test_metrics_golden():
    for c in GOLD["psnr"]["cases"]:
        x = np.zeros(100)
        x[0] = c["peak"]
        xh = x.copy()
        xh[1:] += math.sqrt(c["mse"] * 100 / 99) if c["mse"] else 0.0
        want = math.inf if c["db"] == "inf" else c["db"]
        assert oracle.psnr(xh, x) == pytest.approx(want, abs=1e-9)
    for c in GOLD["success"]["cases"]:
        x = np.ones(10)                   # ||x||^2 = 10
        xh = x.copy()
        xh[0] += math.sqrt(10 * c["nmse"])  # ||x_hat - x||^2 = 10 * nmse (exact at 0 and 0.1)
        assert oracle.success(xh, x) == c["phi"]
    x = RNG.standard_normal(50)
    for c in GOLD["nmse"]["cases"]:
        assert oracle.nmse(c["scale"] * x, x) == pytest.approx(c["nmse"], abs=1e-15)


@pytest.mark.parametrize("bias", ["zero", "channel"])
def test_forward_xcorr_flag(bias):
    """DI_FLAG_XCORR at the forward level: taps T given in cross-correlation
    convention.  Pinned two ways: (1) forward(T, xcorr) == forward(flip(T)) bitwise -- the flip is an index
    relabelling, same products in the same order; (2) torch conv2d (itself a cross-correlation) with T unflipped."""
    torch = pytest.importorskip("torch")
    n1, n2, m = 13, 10, 60
    phi = synth.make_phi(m, n1 * n2).astype(np.float64)
    p = synth.make_params(bias=bias)
    y = RNG.standard_normal((2, m))
    got = oracle.forward(y, phi, p, n1, n2, xcorr=True)
    flipped = synth.Params([np.ascontiguousarray(np.asarray(w)[:, :, ::-1, ::-1]) for w in p.w], p.b)
    assert np.array_equal(got, oracle.forward(y, phi, flipped, n1, n2))
    a = (torch.from_numpy(y) @ torch.from_numpy(phi)).reshape(-1, 1, n1, n2)
    for l, (w, b) in enumerate(zip(p.w, p.b)):
        a = torch.nn.functional.conv2d(a, torch.from_numpy(np.asarray(w, np.float64)),
                                       torch.from_numpy(np.asarray(b, np.float64)), padding=5)
        if l < 2:
            a = a.relu()
    ref = a[:, 0].numpy()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
    # and the flag matters: the He-normal taps are not symmetric
    assert not np.allclose(got, oracle.forward(y, phi, p, n1, n2))
