"""Input generators: determinism, sharding invariance, distributions (CPU only)."""
import numpy as np

import synth
from synth import rng


def test_phi_deterministic_and_row_slices():
    a = synth.make_phi(64, 256)
    b = synth.make_phi(64, 256)
    assert np.array_equal(a, b)
    assert np.array_equal(synth.make_phi(64, 256, rows=(10, 30)), a[10:30])
    assert not np.array_equal(a, synth.make_phi(64, 256, seed=7))


def test_phi_column_norms_near_one():
    """mean squared column norm in [0.9, 1.1] for m >= 200 (variance 1/m)."""
    phi = synth.make_phi(410, 4096).astype(np.float64)
    msq = float(np.mean(np.sum(phi ** 2, axis=0)))
    assert 0.9 <= msq <= 1.1
    assert abs(float(phi.mean())) < 1e-3


def test_images_shard_invariant_and_range():
    full = synth.make_images(64, 0, 12, 8, 4)
    part = synth.make_images(64, 5, 4, 8, 4)
    assert np.array_equal(full[5:9], part)
    assert full.dtype == np.float32 and full.min() >= 0 and full.max() <= 1
    tex = synth.make_images(32, 0, 3, 4, 2, texture_var=0.01)
    assert tex.min() >= 0 and tex.max() <= 1


def test_bf16_round_to_nearest_even():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e38, 1e-40], np.float32)
    b = synth.f32_to_bf16_bits(x)
    assert b[0] == 0x3F80
    assert b[1] == 0x3F80          # tie -> even
    assert b[2] == 0x3F82          # tie -> even (up)
    assert b[3] == 0xC020
    r = synth.round_bf16(x)
    assert np.all(np.abs(r[:4] - x[:4]) <= np.abs(x[:4]) * 2.0 ** -8)


def test_params_he_normal():
    p = synth.make_params()
    for w, cin in zip(p.w, (1, 64, 32)):
        sd = np.sqrt(2.0 / (cin * 121))
        assert abs(w.std() / sd - 1) < 0.1
    assert [w.shape for w in p.w] == [(64, 1, 11, 11), (32, 64, 11, 11), (1, 32, 11, 11)]


def test_normals_split_invariant():
    key = rng.stream_key(9)
    a = rng.normal(key, 0, 1000, chunk=64)
    b = rng.normal(key, 500, 500)
    assert np.array_equal(a[500:], b)
    assert abs(a.mean()) < 0.15 and abs(a.std() - 1) < 0.1


def test_measure_is_phi_x():
    phi = synth.make_phi(20, 64)
    x = synth.make_images(8, 0, 3, 2, 1)
    y = synth.measure(phi, x)
    np.testing.assert_allclose(y, (phi.astype(np.float64) @ x.reshape(3, -1).T.astype(np.float64)).T, rtol=1e-6)
