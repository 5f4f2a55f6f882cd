"""GPU parity of the sensing model and metrics around the path: di_measure (y = Phi x,
PAPER.md:27), di_add_noise (Table 3's SNR rule, Q14) and di_metrics (PSNR PAPER.md:165, NMSE and
success PAPER.md:160) against the fp64 oracle on the same input bits."""
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import Case, make_ctx

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "tf32": 2e-2, "bf16": 2e-2}


@pytest.mark.parametrize("precision", ["f32", "bf16", "tf32"])
@pytest.mark.parametrize("n1,n2,m,batch", [(64, 64, 410, 300), (9, 13, 40, 3), (16, 16, 64, 4), (40, 72, 300, 130)])
def test_measure_matches_oracle(precision, n1, n2, m, batch):
    import torch
    case = Case(n1, n2, m, batch, precision, 6, 3)
    ctx = make_ctx(case)
    st = "bf16" if precision == "bf16" else "f32"
    xs = synth.round_bf16(case.x) if st == "bf16" else case.x     # the GPU reads x in the storage type
    xd = torch.from_numpy(case.x).cuda()
    y = ctx.measure(xd).float().cpu().numpy()
    ref = oracle.measure(case.phi, xs)
    rel = max(oracle.rel_l2(a, r) for a, r in zip(y, ref))
    assert rel <= (1e-5 if precision == "f32" else 1e-2), rel
    # measuring then recovering on the GPU equals recovering the host-generated measurements (same tolerance)
    out = ctx.recover(ctx.measure(xd)).cpu().numpy()
    ref_x = oracle.forward(ref, case.phi, case.params, n1, n2)
    assert max(oracle.rel_l2(a, r) for a, r in zip(out, ref_x)) <= TOL[precision]


@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_noise_matches_oracle_generator(precision):
    import torch
    case = Case(64, 64, 410, 17, precision)
    ctx = make_ctx(case)
    y0 = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
    for snr, seed in [(20.0, 3), (5.0, 4), (40.0, 1701)]:
        y = y0.clone()
        ctx.add_noise(y, snr, seed)
        got = y.float().cpu().numpy()
        ref = oracle.add_noise(y0.float().cpu().numpy().astype(np.float64), snr, seed)
        w_got, w_ref = got - y0.float().cpu().numpy(), ref - y0.float().cpu().numpy()
        # noise itself (not only y + w): same stream, same scale
        assert oracle.rel_l2(w_got, w_ref) <= (1e-5 if precision == "f32" else 0.05 * 10 ** (snr / 20)), snr
        assert oracle.rel_l2(got, ref) <= (1e-6 if precision == "f32" else 5e-3)
    y = y0.clone()
    ctx.add_noise(y, math.inf, 9)
    assert torch.equal(y, y0), "+inf dB = noiseless"


def test_metrics_match_oracle():
    import torch
    case = Case(64, 64, 410, 33, "bf16")
    ctx = make_ctx(case)
    xhat = ctx.recover(torch.from_numpy(case.y).cuda().to(torch.bfloat16))
    x = torch.from_numpy(case.x).cuda()
    got = ctx.metrics(xhat, x)
    xh = xhat.cpu().numpy()
    for b in range(case.batch):
        assert abs(got[0, b] - oracle.psnr(xh[b], case.x[b])) <= 1e-9
        assert abs(got[1, b] - oracle.nmse(xh[b], case.x[b])) <= 1e-12 * max(1.0, got[1, b])
        assert got[2, b] == oracle.success(xh[b], case.x[b])
    # exact case: x_hat = x -> PSNR = inf, NMSE = 0, success = 1
    same = ctx.metrics(x, x)
    assert np.all(np.isinf(same[0])) and np.all(same[1] == 0) and np.all(same[2] == 1)


@pytest.mark.parametrize("precision,n1,n2,batch", [("bf16", 64, 64, 300), ("bf16", 40, 130, 5), ("bf16", 9, 13, 3),
                                                   ("bf16", 64, 64, 1), ("tf32", 32, 32, 6), ("f32", 16, 16, 4)])
@pytest.mark.parametrize("fused", [True, False])
def test_recover_metrics_fused(monkeypatch, fused, precision, n1, n2, batch):
    """di_recover_metrics: the metrics fused into conv layer 3's epilogue (BF16 with DI_EXP_FUSED_METRICS=1; items =
    whole image columns, several column segments at n2 = 130, split columns at batch 1) or the separate pass equal
    the oracle's metrics of the GPU's own x_hat, the x_hat is bitwise the di_recover result, and the result is
    bitwise repeatable (fixed-order reduction)."""
    import torch
    case = Case(n1, n2, max(1, n1 * n2 // 8), batch, precision, 6, 3)
    if fused:
        monkeypatch.setenv("DI_EXP_FUSED_METRICS", "1")
    ctx = make_ctx(case)
    monkeypatch.delenv("DI_EXP_FUSED_METRICS", raising=False)
    y = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
    x = torch.from_numpy(case.x).cuda()
    xhat, got = ctx.recover_metrics(y, x)
    xh = xhat.cpu().numpy()
    assert np.array_equal(xh, ctx.recover(y).cpu().numpy())
    for b in range(batch):
        assert abs(got[0, b] - oracle.psnr(xh[b], case.x[b])) <= 1e-9
        assert abs(got[1, b] - oracle.nmse(xh[b], case.x[b])) <= 1e-12 * max(1.0, got[1, b])
        assert got[2, b] == oracle.success(xh[b], case.x[b])
    _, again = ctx.recover_metrics(y, x)
    assert np.array_equal(again, got)
