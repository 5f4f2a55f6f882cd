"""Pins for oracle.conv_layer (Eq. (1)) -- CPU only.

Each pin is independent of the oracle's own loop nest: library routines
(scipy.signal.convolve2d, torch conv2d in fp64), an im2col+matmul brute force,
closed forms (delta kernel, delta image, zero input), worked examples
(tests/golden/spec_examples.json) and invariants (linearity, translation
equivariance).  A dropped term, wrong flip, wrong crop offset or transposed
channel index fails at least one of them.
"""
import json
import os

import numpy as np
import pytest
import scipy.signal

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
RNG = np.random.default_rng(1701)


def _im2col_full_then_crop(x, w, b, relu, fullmap):
    """Brute force: full true convolution as one matrix product over an explicit
    zero-padded copy, then bias, ReLU and the centred crop."""
    cin, n1, n2 = x.shape
    cout, _, k, _ = w.shape
    h, wd = n1 + k - 1, n2 + k - 1
    xp = np.zeros((cin, n1 + 2 * (k - 1), n2 + 2 * (k - 1)))
    xp[:, k - 1:k - 1 + n1, k - 1:k - 1 + n2] = x
    cols = np.empty((h * wd, cin * k * k))
    for i in range(h):
        for j in range(wd):
            # element (c, u, v) = X[c][i-u][j-v]
            patch = xp[:, i:i + k, j:j + k][:, ::-1, ::-1]
            cols[i * wd + j] = patch.ravel()
    f = (cols @ w.reshape(cout, -1).T).T.reshape(cout, h, wd)
    if b is not None:
        f = f + (b if fullmap else b[:, None, None])
    if relu:
        f = np.maximum(f, 0.0)
    p = (k - 1) // 2
    return f[:, p:p + n1, p:p + n2]


@pytest.mark.parametrize("cin,cout,n1,n2,k", [(1, 3, 5, 5, 3), (3, 2, 7, 4, 5), (2, 2, 1, 1, 11),
                                              (4, 3, 11, 6, 11), (1, 1, 16, 17, 11)])
@pytest.mark.parametrize("fullmap", [False, True])
def test_conv_vs_im2col_bruteforce(cin, cout, n1, n2, k, fullmap):
    x = RNG.standard_normal((cin, n1, n2))
    w = RNG.standard_normal((cout, cin, k, k))
    b = RNG.uniform(-0.1, 0.1, (cout, n1 + k - 1, n2 + k - 1) if fullmap else (cout,))
    for relu in (False, True):
        got = oracle.conv_layer(x, w, b, relu=relu, fullmap_bias=fullmap)
        ref = _im2col_full_then_crop(x, w, b, relu, fullmap)
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * (1 + np.abs(ref).max()))


@pytest.mark.parametrize("cin,n", [(1, 5), (3, 11), (64, 16)])
def test_conv_vs_scipy_convolve2d(cin, n):
    """Special case reducing to a library routine: scipy's full 2-D convolution, summed
    over input channels, then the centred crop."""
    k = 11
    x = RNG.standard_normal((cin, n, n))
    w = RNG.standard_normal((2, cin, k, k))
    got = oracle.conv_layer(x, w, None, relu=False)
    for o in range(2):
        full = sum(scipy.signal.convolve2d(x[c], w[o, c], mode="full") for c in range(cin))
        ref = full[5:5 + n, 5:5 + n]
        np.testing.assert_allclose(got[o], ref, rtol=0, atol=1e-11 * (1 + np.abs(ref).max()))


def test_conv_vs_torch_fp64_same_padding():
    """torch conv2d is a cross-correlation: true conv + crop == xcorr with the flipped kernel,
    'same' zero padding (k-1)/2 (SURVEY.md §8(c) equivalent fast form)."""
    torch = pytest.importorskip("torch")
    x = RNG.standard_normal((64, 13, 9))
    w = RNG.standard_normal((32, 64, 11, 11)) * 0.02
    b = RNG.uniform(-0.1, 0.1, 32)
    got = oracle.conv_layer(x, w, b, relu=True)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x)[None], torch.from_numpy(w).flip(-1, -2),
                                     torch.from_numpy(b), padding=5).relu()[0].numpy()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    # the XCORR flag takes taps in torch's convention directly
    got2 = oracle.conv_layer(x, w, b, relu=True, xcorr=True)
    ref2 = torch.nn.functional.conv2d(torch.from_numpy(x)[None], torch.from_numpy(w),
                                      torch.from_numpy(b), padding=5).relu()[0].numpy()
    np.testing.assert_allclose(got2, ref2, rtol=0, atol=1e-12)


def test_golden_scalar_conv():
    g = GOLD["conv_scalar"]
    got = oracle.conv_layer(np.array(g["input"]), np.array(g["filter"]), None, relu=False)
    assert got.tolist() == g["output"]


def test_golden_relu():
    g = GOLD["relu"]
    x = np.array(g["input"]).reshape(1, 1, 3)
    got = oracle.conv_layer(x, np.ones((1, 1, 1, 1)), None, relu=True)
    assert got.ravel().tolist() == g["output"]


def test_golden_crop_window_fullmap_bias():
    """S keeps the centred window: with a zero input only the full-map bias
    reaches the output, and exactly its rows/cols p..p+n-1 do."""
    g = GOLD["crop"]
    k = g["n_in"] - g["n_out"] + 1       # 5 = 3 + k - 1  ->  k = 3
    b = np.arange(25, dtype=np.float64).reshape(1, 5, 5)
    got = oracle.conv_layer(np.zeros((1, 3, 3)), np.zeros((1, 1, k, k)), b, relu=False, fullmap_bias=True)
    f = g["first"]
    assert np.array_equal(got[0], b[0, f:f + 3, f:f + 3])


@pytest.mark.parametrize("k", [1, 3, 11])
def test_delta_kernel_is_identity(k):
    x = RNG.standard_normal((1, 9, 7))
    w = np.zeros((1, 1, k, k))
    w[0, 0, k // 2, k // 2] = 1.0
    got = oracle.conv_layer(x, w, None, relu=False)
    assert np.array_equal(got, x)


@pytest.mark.parametrize("p,q", [(10, 10), (0, 0), (3, 19), (20, 2)])
def test_delta_image_reproduces_taps(p, q):
    """True convolution (Q2): a unit impulse at (p,q) gives out[p+a][q+b] = W[5+a][5+b]
    (the taps un-flipped, centred at the impulse); XCORR gives the flipped taps."""
    n, k = 21, 11
    x = np.zeros((1, n, n))
    x[0, p, q] = 1.0
    w = RNG.standard_normal((1, 1, k, k))
    got = oracle.conv_layer(x, w, None, relu=False)[0]
    gotx = oracle.conv_layer(x, w, None, relu=False, xcorr=True)[0]
    for a in range(-5, 6):
        for b in range(-5, 6):
            r, s = p + a, q + b
            if 0 <= r < n and 0 <= s < n:
                assert got[r, s] == w[0, 0, 5 + a, 5 + b]
                assert gotx[r, s] == w[0, 0, 5 - a, 5 - b]
    mask = np.ones((n, n), bool)
    mask[max(0, p - 5):p + 6, max(0, q - 5):q + 6] = False
    assert np.all(got[mask] == 0)


@pytest.mark.parametrize("fullmap", [False, True])
def test_zero_input_gives_bias_response(fullmap):
    n, k = 8, 11
    b = RNG.uniform(-0.1, 0.1, (3, n + k - 1, n + k - 1) if fullmap else (3,))
    w = RNG.standard_normal((3, 2, k, k))
    got = oracle.conv_layer(np.zeros((2, n, n)), w, b, relu=True, fullmap_bias=fullmap)
    ref = np.maximum(b[:, 5:5 + n, 5:5 + n], 0) if fullmap else np.broadcast_to(np.maximum(b, 0)[:, None, None], (3, n, n))
    assert np.array_equal(got, ref)


def test_linearity_before_relu():
    x1, x2 = RNG.standard_normal((2, 3, 12, 12))
    w = RNG.standard_normal((4, 3, 11, 11))
    a, c = 0.7, -1.3
    lhs = oracle.conv_layer(a * x1 + c * x2, w, None, relu=False)
    rhs = a * oracle.conv_layer(x1, w, None, relu=False) + c * oracle.conv_layer(x2, w, None, relu=False)
    np.testing.assert_allclose(lhs, rhs, rtol=0, atol=1e-10 * np.abs(rhs).max())


def test_translation_equivariance_exact():
    """Input supported >= 5+|shift| px from every border: the output shifts exactly
    (same products, same order)."""
    n = 40
    x = np.zeros((2, n, n))
    x[:, 12:22, 11:20] = RNG.standard_normal((2, 10, 9))
    w = RNG.standard_normal((3, 2, 11, 11))
    b = RNG.uniform(-0.1, 0.1, 3)
    y0 = oracle.conv_layer(x, w, b, relu=True)
    xs = np.roll(x, (3, -2), axis=(1, 2))
    y1 = oracle.conv_layer(xs, w, b, relu=True)
    assert np.array_equal(np.roll(y0, (3, -2), axis=(1, 2))[:, 8:32, 8:32], y1[:, 8:32, 8:32])


def test_relu_idempotent_and_shape():
    x = RNG.standard_normal((2, 6, 9))
    w = RNG.standard_normal((3, 2, 3, 3))
    y = oracle.conv_layer(x, w, None, relu=True)
    assert y.shape == (3, 6, 9)
    assert np.array_equal(np.maximum(y, 0), y)


def test_even_kernel_rejected():
    with pytest.raises(ValueError):
        oracle.conv_layer(np.zeros((1, 4, 4)), np.zeros((1, 1, 2, 2)))
