"""GPU parity of the training step: loss and gradients of di_train_grad against the fp64
oracle (oracle.train_grad, pinned by finite differences), SGD consistency and a decreasing loss."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import Case, make_ctx

pytestmark = pytest.mark.gpu

# fp32 forward (<= 1e-5) and fp32 gradient sums (per 256-pixel tile in fp32, then fp64 across tiles); TF32: the
# forward's 10-bit-mantissa products (the 2e-2 bar of the TF32 path)
TOL_GRAD = {"f32": 1e-4, "tf32": 2e-2, "bf16": 2e-2}


def _grads_ok(ctx, case, scale=None, final_relu=False, xcorr=False):
    tol = TOL_GRAD[case.precision]
    import torch
    from paper_1701_03891_b200 import split_params
    y = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
    x = torch.from_numpy(case.x).cuda()
    loss, g = ctx.train_grad(y, x, scale)
    torch.cuda.synchronize()
    ws, bs = split_params(g.cpu().numpy().astype(np.float64))
    p = case.params
    if xcorr:   # the oracle works in the true-convolution orientation
        p = synth.Params([w[:, :, ::-1, ::-1].copy() for w in p.w], p.b)
    rl, rw, rb = oracle.train_grad(case.y, case.x, case.phi, p, case.n1, case.n2, scale=scale, final_relu=final_relu)
    if xcorr:
        rw = [w[:, :, ::-1, ::-1] for w in rw]
    assert abs(float(loss.item()) - rl) <= (1e-5 if case.precision == "f32" else 1e-2) * abs(rl)
    for l in range(3):
        assert oracle.rel_l2(ws[l], rw[l]) <= tol, ("W", l, oracle.rel_l2(ws[l], rw[l]))
        assert oracle.rel_l2(bs[l], rb[l]) <= tol, ("b", l, oracle.rel_l2(bs[l], rb[l]))


@pytest.mark.parametrize("precision", ["f32", "tf32"])
@pytest.mark.parametrize("n1,n2,m,batch", [(16, 16, 64, 4), (40, 72, 300, 3), (9, 13, 40, 2)])
def test_gradients_match_oracle(precision, n1, n2, m, batch):
    case = Case(n1, n2, m, batch, precision, 6, 3, bias="channel")
    _grads_ok(make_ctx(case), case)


@pytest.mark.parametrize("n1,n2,m,batch", [(16, 16, 64, 4), (40, 72, 300, 3), (64, 64, 410, 4)])
def test_gradients_match_oracle_bf16(n1, n2, m, batch):
    """BF16 contexts train on the bf16 forward (x_tilde, h1, h2 stored in bf16) and the bf16 / TF32 tensor-core
    backward; the oracle runs on the same bf16-rounded Phi, y and Omega."""
    case = Case(n1, n2, m, batch, "bf16", 6, 3, bias="channel")
    _grads_ok(make_ctx(case), case)


def test_bf16_training_needs_n2_multiple_of_4():
    import torch
    from paper_1701_03891_b200 import DiError
    case = Case(9, 13, 40, 2, "bf16", 6, 3, bias="channel")
    ctx = make_ctx(case)
    with pytest.raises(DiError):
        ctx.train_grad(torch.from_numpy(case.y).cuda().to(torch.bfloat16), torch.from_numpy(case.x).cuda())


@pytest.mark.parametrize("final_relu,xcorr", [(True, False), (False, True)])
def test_gradients_flags(final_relu, xcorr):
    from paper_1701_03891_b200 import DI_FLAG_FINAL_RELU, DI_FLAG_XCORR
    case = Case(24, 24, 128, 3, "f32", 6, 3, bias="channel")
    flags = (DI_FLAG_FINAL_RELU if final_relu else 0) | (DI_FLAG_XCORR if xcorr else 0)
    _grads_ok(make_ctx(case, flags=flags), case, final_relu=final_relu, xcorr=xcorr)


@pytest.mark.parametrize("precision", ["f32", "tf32", "bf16"])
def test_sgd_updates_the_forward_and_lowers_the_loss(precision):
    import torch
    case = Case(32, 32, 256, 8, precision, 6, 3, bias="channel")
    ctx = make_ctx(case)
    y = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
    x = torch.from_numpy(case.x).cuda()
    losses, lr = [], None
    for _ in range(6):
        loss, g = ctx.train_grad(y, x)
        losses.append(float(loss.item()))
        if lr is None:   # a step small against the curvature: first-order decrease 5 % of the loss
            lr = 0.05 * losses[0] / float((g.double() ** 2).sum())
        ctx.sgd_step(g, lr=lr, momentum=0.5)
    assert all(np.isfinite(losses)) and losses[-1] < 0.9 * losses[0], losses
    # the updated parameters drive the forward: GPU recovery == oracle forward with the read-back parameters
    ws, bs = ctx.params()
    if precision == "bf16":   # BF16 contexts run the forward on the RNE-rounded fp32 master weights (deepinverse.h)
        ws = [synth.round_bf16(w) for w in ws]
    p = synth.Params([w.astype(np.float64) for w in ws], [b.astype(np.float64) for b in bs])
    out = ctx.recover(y).cpu().numpy()
    ref = oracle.forward(case.y, case.phi, p, case.n1, case.n2)
    assert max(oracle.rel_l2(a, r) for a, r in zip(out, ref)) <= (1e-5 if precision == "f32" else 2e-2)
    # one SGD step without momentum is exactly params - lr * grads
    _, g = ctx.train_grad(y, x)
    before = np.concatenate([w.ravel() for w in ctx.params()[0]] + [b for b in ctx.params()[1]])
    ctx.sgd_step(g, lr=1e-3, momentum=0.0)
    after = np.concatenate([w.ravel() for w in ctx.params()[0]] + [b for b in ctx.params()[1]])
    # (the momentum buffer from the loop above persists: vel = 0 * vel + g)
    assert np.allclose(after, before - np.float32(1e-3) * g.cpu().numpy(), rtol=0, atol=1e-7)


def test_training_rejects_fullmap_bias_contexts():
    import torch
    from paper_1701_03891_b200 import DiError
    case = Case(16, 16, 64, 2, "f32", bias="fullmap")
    ctx = make_ctx(case)
    with pytest.raises(DiError):
        ctx.train_grad(torch.from_numpy(case.y).cuda(), torch.from_numpy(case.x).cuda())


@pytest.mark.parametrize("final_relu,xcorr", [(True, False), (False, True)])
def test_gradients_flags_tf32(final_relu, xcorr):
    """The tensor-core backward honours the flags: FINAL_RELU masks dG3, XCORR changes the tap orientation of
    every repacked bank (forward, dgrad2, dgrad3) and of the weight-gradient reduction."""
    from paper_1701_03891_b200 import DI_FLAG_FINAL_RELU, DI_FLAG_XCORR
    case = Case(24, 24, 128, 3, "tf32", 6, 3, bias="channel")
    flags = (DI_FLAG_FINAL_RELU if final_relu else 0) | (DI_FLAG_XCORR if xcorr else 0)
    _grads_ok(make_ctx(case, flags=flags), case, final_relu=final_relu, xcorr=xcorr)


def test_gradients_paper_geometry_tf32():
    """64x64 images (the paper config's geometry: 11 row blocks of 6 with a partial last block, full-width units)
    on the tensor-core backward, 6 images."""
    case = Case(64, 64, 1024, 6, "tf32", 8, 4, bias="channel")
    _grads_ok(make_ctx(case), case)


def test_gradients_column_segments_tf32():
    """96-wide images: two column segments per row block, so the wgrad strips zero their halo columns in shared
    memory (k_wgrad2_tc) and the thin-layer operands are cut at the segment edge (k_wgrad13_tc)."""
    case = Case(20, 96, 400, 2, "tf32", 6, 3, bias="channel")
    _grads_ok(make_ctx(case), case)


@pytest.mark.parametrize("precision", ["f32", "tf32"])
def test_gradients_are_deterministic(precision):
    """Every reduction is two-level in a fixed order (no atomics): repeated calls give identical bits, and the
    gradient of a batch is independent of the batch capacity of the context."""
    import torch
    case = Case(32, 32, 200, 5, precision, 6, 3, bias="channel")
    y = torch.from_numpy(case.y).cuda()
    x = torch.from_numpy(case.x).cuda()
    a = make_ctx(case)
    b = make_ctx(case, max_batch=16)
    l1, g1 = a.train_grad(y, x, 0.2)
    g1 = g1.clone()
    l2, g2 = a.train_grad(y, x, 0.2)
    l3, g3 = b.train_grad(y, x, 0.2)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and float(l1.item()) == float(l2.item())
    assert torch.equal(g1, g3) and float(l1.item()) == float(l3.item())
