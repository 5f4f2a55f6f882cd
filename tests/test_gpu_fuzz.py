"""GPU parity on seeded random shapes: the three precisions over image sizes that land on and off every geometry
boundary of the kernels (64-column segments, 6/7-row conv2 blocks, 11-row conv3 units, 256-position tiles, odd
widths that force the gather paths), random M and batch, zero or per-channel biases.  Each case compares 2 + 2
sampled images element-wise against the fp64 oracle (gpu_helpers.compare) and the north_star rel-L2 / dPSNR bars.
The case list is fixed by its seed, so a failure names a reproducible shape."""
import numpy as np
import pytest

from gpu_helpers import TOL_DPSNR, TOL_REL_L2, Case, compare, make_ctx, run, sample_rows

pytestmark = pytest.mark.gpu

_EDGES = [1, 2, 5, 6, 7, 11, 12, 13, 21, 22, 23, 42, 43, 59, 63, 64, 65, 69, 70, 74, 75, 77, 96, 127, 128, 129, 133,
          140]


def _cases(seed=20260420, n=36):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        prec = ("f32", "tf32", "bf16")[i % 3]
        n1 = int(rng.choice(_EDGES)) if rng.random() < 0.6 else int(rng.integers(1, 141))
        n2 = int(rng.choice(_EDGES)) if rng.random() < 0.6 else int(rng.integers(1, 141))
        N = n1 * n2
        m = int(max(1, min(N, round(N * rng.uniform(0.05, 1.0)))))
        batch = int(rng.choice([1, 2, 3, 5, 17, 64, 129, 257, 300]))
        bias = "channel" if rng.random() < 0.5 else "zero"
        out.append((prec, n1, n2, m, batch, bias))
    return out


@pytest.mark.parametrize("prec,n1,n2,m,batch,bias", _cases())
def test_random_shape_parity(prec, n1, n2, m, batch, bias):
    case = Case(n1, n2, m, batch, prec, 5, 3, bias=bias, start=7 * n1 + n2)
    ctx = make_ctx(case)
    out = run(case, ctx)
    assert out.shape == (batch, n1, n2)
    assert np.all(np.isfinite(out))
    idx = sample_rows(batch, 4)
    ref = case.oracle(idx)
    rel, dps, dmean = compare(out[idx], ref, case.x[idx], prec)
    assert rel <= TOL_REL_L2[prec], f"rel-L2 {rel:.3g}"
    assert dps <= TOL_DPSNR and abs(dmean) <= TOL_DPSNR, f"dPSNR {dps:.3g} mean {dmean:.3g}"
