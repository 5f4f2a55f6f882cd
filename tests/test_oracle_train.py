"""Pins for oracle.train_grad: the MSE loss of PAPER.md:136 and its gradient -- CPU only.

The gradient is checked against central finite differences of the loss (SPEC.md:81-89 grad_check idea), against
the closed forms of a zero residual and of the loss scale, and for additivity over images (the data-parallel
all-reduce relies on it)."""
import numpy as np
import pytest

import oracle
import synth


def _tiny(seed=0, widths=(1, 3, 2, 1), k=3, n1=6, n2=5, m=17, batch=2):
    r = np.random.default_rng(seed)
    phi = r.standard_normal((m, n1 * n2)) / np.sqrt(m)
    ws = [r.standard_normal((widths[l + 1], widths[l], k, k)) * 0.6 for l in range(len(widths) - 1)]
    bs = [r.uniform(-0.1, 0.1, widths[l + 1]) for l in range(len(widths) - 1)]
    y = r.standard_normal((batch, m))
    x = r.uniform(0, 1, (batch, n1, n2))
    return phi, synth.Params(ws, bs), y, x, n1, n2


def _loss(phi, p, y, x, n1, n2):
    xh = oracle.forward(y, phi, p, n1, n2)
    return float(np.sum((xh - x) ** 2)) / y.shape[0]


@pytest.mark.parametrize("seed", [0, 1])
def test_gradient_vs_central_differences(seed):
    phi, p, y, x, n1, n2 = _tiny(seed)
    loss, dws, dbs = oracle.train_grad(y, x, phi, p, n1, n2)
    assert loss == pytest.approx(_loss(phi, p, y, x, n1, n2), rel=1e-12)
    r = np.random.default_rng(seed + 10)
    eps = 1e-6
    for l in range(3):
        for _ in range(6):                                     # random weights of layer l
            idx = tuple(int(r.integers(0, s)) for s in p.w[l].shape)
            wp = [w.copy() for w in p.w]
            wm = [w.copy() for w in p.w]
            wp[l][idx] += eps
            wm[l][idx] -= eps
            fd = (_loss(phi, synth.Params(wp, p.b), y, x, n1, n2) - _loss(phi, synth.Params(wm, p.b), y, x, n1, n2)) / (2 * eps)
            assert dws[l][idx] == pytest.approx(fd, rel=1e-5, abs=1e-8), (l, idx)
        for o in range(p.b[l].size):                           # every bias of layer l
            bp = [b.copy() for b in p.b]
            bm = [b.copy() for b in p.b]
            bp[l][o] += eps
            bm[l][o] -= eps
            fd = (_loss(phi, synth.Params(p.w, bp), y, x, n1, n2) - _loss(phi, synth.Params(p.w, bm), y, x, n1, n2)) / (2 * eps)
            assert dbs[l][o] == pytest.approx(fd, rel=1e-5, abs=1e-8), (l, o)


def test_zero_residual_gives_zero_gradient():
    phi, p, y, _, n1, n2 = _tiny(3)
    x = oracle.forward(y, phi, p, n1, n2)
    loss, dws, dbs = oracle.train_grad(y, x, phi, p, n1, n2)
    assert loss == 0.0
    assert all(np.all(g == 0) for g in dws + dbs)


def test_scale_and_additivity_over_images():
    """grad(scale 2s) = 2 grad(s) exactly; grad over a batch = sum of the grads of its halves (the DP all-reduce)."""
    phi, p, y, x, n1, n2 = _tiny(4, batch=4)
    l1, g1, b1 = oracle.train_grad(y, x, phi, p, n1, n2, scale=0.25, threads=1)
    l2, g2, b2 = oracle.train_grad(y, x, phi, p, n1, n2, scale=0.5, threads=1)
    assert l2 == 2 * l1
    assert all(np.array_equal(2 * a, b) for a, b in zip(g1 + b1, g2 + b2))
    la, ga, ba = oracle.train_grad(y[:2], x[:2], phi, p, n1, n2, scale=0.25)
    lb, gb, bb = oracle.train_grad(y[2:], x[2:], phi, p, n1, n2, scale=0.25)
    assert la + lb == pytest.approx(l1, rel=1e-13)
    for full, a, b in zip(g1 + b1, ga + ba, gb + bb):
        assert np.allclose(full, a + b, rtol=1e-12, atol=1e-15)


def test_paper_widths_single_image_runs_and_final_relu_flag():
    c = synth.CONFIGS["tiny"]
    phi = synth.make_phi(c.m, c.N)
    x = synth.make_images(c.n, 0, 1, c.n_blobs, c.n_rects)
    y = synth.measure(phi, x)
    p = synth.make_params(bias="channel")
    loss, dws, dbs = oracle.train_grad(y, x, phi, p, c.n, c.n)
    assert loss > 0 and [g.shape for g in dws] == [w.shape for w in p.w]
    loss_r, dws_r, _ = oracle.train_grad(y, x, phi, p, c.n, c.n, final_relu=True)
    assert np.isfinite(loss_r) and dws_r[2].shape == p.w[2].shape


def _loss_fr(phi, p, y, x, n1, n2):
    xh = oracle.forward(y, phi, p, n1, n2, final_relu=True)
    return float(np.sum((xh - x) ** 2)) / y.shape[0]


@pytest.mark.parametrize("seed", [5, 6])
def test_final_relu_gradient_vs_central_differences(seed):
    """PAPER.md:118 ("each convolutional layer applies a ReLU") read literally: the layer-3 ReLU mask must reach the
    gradient.  The case has layer-3 pre-activations on both sides of zero (checked), so a gradient that ignored the
    mask (or masked with the wrong sign) differs from the finite differences of the masked loss."""
    phi, p, y, x, n1, n2 = _tiny(seed)
    xh = oracle.forward(y, phi, p, n1, n2, final_relu=True)
    lin = oracle.forward(y, phi, p, n1, n2, final_relu=False)
    assert np.any(lin < -1e-3) and np.any(lin > 1e-3)          # both sides of the kink
    assert np.array_equal(xh, np.maximum(lin, 0.0))
    loss, dws, dbs = oracle.train_grad(y, x, phi, p, n1, n2, final_relu=True)
    assert loss == pytest.approx(_loss_fr(phi, p, y, x, n1, n2), rel=1e-12)
    _, dws0, dbs0 = oracle.train_grad(y, x, phi, p, n1, n2, final_relu=False)
    assert not np.allclose(dbs[2], dbs0[2])                    # the flag changes the gradient
    r = np.random.default_rng(seed + 20)
    eps = 1e-6
    for l in range(3):
        for _ in range(6):
            idx = tuple(int(r.integers(0, s)) for s in p.w[l].shape)
            wp = [w.copy() for w in p.w]
            wm = [w.copy() for w in p.w]
            wp[l][idx] += eps
            wm[l][idx] -= eps
            fd = (_loss_fr(phi, synth.Params(wp, p.b), y, x, n1, n2) -
                  _loss_fr(phi, synth.Params(wm, p.b), y, x, n1, n2)) / (2 * eps)
            assert dws[l][idx] == pytest.approx(fd, rel=1e-5, abs=1e-8), (l, idx)
        for o in range(p.b[l].size):
            bp = [b.copy() for b in p.b]
            bm = [b.copy() for b in p.b]
            bp[l][o] += eps
            bm[l][o] -= eps
            fd = (_loss_fr(phi, synth.Params(p.w, bp), y, x, n1, n2) -
                  _loss_fr(phi, synth.Params(p.w, bm), y, x, n1, n2)) / (2 * eps)
            assert dbs[l][o] == pytest.approx(fd, rel=1e-5, abs=1e-8), (l, o)
