"""Custom layer stacks ("DeepInverses with larger capacities"): deeper and
wider stacks of Eq. (1) layers through di_create_args.layers, against the fp64 oracle's forward pass over the same
layer list (oracle.forward takes any stack).  FP32 runs the SIMT kernels, TF32 the tensor-core kernels (first layer
on the conv1 machinery, interior layers on k_conv_tf32<C_in, C_out>, last layer on the conv3 kernel), BF16 the bf16
tensor-core kernels (k_conv1_tc, k_conv2_tc<C_in, C_out>, k_conv3_r4) on bf16 activations; the oracle takes the same
bf16-rounded weights and measurements (gpu_helpers.Case)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import TOL_REL_L2, Case, compare

pytestmark = pytest.mark.gpu


def stack_params(widths, seed=5, bias=True):
    """He-normal taps (reading Q9) and U[-0.1, 0.1] per-channel biases for the layer widths."""
    r = np.random.default_rng(seed)
    ws, bs = [], []
    for cin, cout in zip(widths[:-1], widths[1:]):
        ws.append((r.standard_normal((cout, cin, 11, 11)) * np.sqrt(2.0 / (cin * 121))).astype(np.float32))
        bs.append(r.uniform(-0.1, 0.1, cout).astype(np.float32) if bias else np.zeros(cout, np.float32))
    return synth.Params(ws, bs)


def run_stack(widths, precision, n1, n2, m, batch, flags=0, final_relu=False):
    import torch
    from paper_1701_03891_b200 import DeepInverse
    case = Case(n1, n2, m, batch, precision, 6, 3, params=stack_params(widths))
    ctx = DeepInverse(case.phi, case.params, n1, n2, precision, flags=flags, max_batch=batch)
    assert ctx.custom
    out = ctx.recover(torch.from_numpy(case.y).to(device="cuda", dtype=ctx.storage_dtype)).cpu().numpy()
    ref = oracle.forward(case.y, case.phi, case.params, n1, n2, final_relu=final_relu)
    ctx.close()
    return compare(out, ref, case.x, precision)


@pytest.mark.parametrize("precision", ["f32", "tf32", "bf16"])
@pytest.mark.parametrize("widths", [(1, 64, 64, 32, 1), (1, 32, 32, 32, 32, 1), (1, 32, 64, 32, 1), (1, 32, 1),
                                    (1, 64, 32, 64, 64, 32, 1)])
def test_stack_matches_oracle(precision, widths):
    rel, dps, _ = run_stack(widths, precision, 32, 32, 200, 3)
    assert rel <= TOL_REL_L2[precision], (widths, rel)


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
def test_stack_column_segments_and_ragged_rows(precision):
    """72-wide, 40-row images: two column segments per row block and a partial last row block in every layer."""
    rel, _, _ = run_stack((1, 64, 64, 32, 32, 64, 32, 1), precision, 40, 72, 300, 2)
    assert rel <= TOL_REL_L2[precision], rel


def test_stack_bf16_odd_width_gather_path():
    """n2 = 20 (not a multiple of 8): the bf16 first layer gathers its strip with plain loads instead of TMA."""
    rel, _, _ = run_stack((1, 32, 64, 32, 1), "bf16", 24, 20, 150, 3)
    assert rel <= TOL_REL_L2["bf16"], rel


def test_stack_final_relu_f32():
    from paper_1701_03891_b200 import DI_FLAG_FINAL_RELU
    rel, _, _ = run_stack((1, 32, 32, 1), "f32", 24, 24, 100, 2, flags=DI_FLAG_FINAL_RELU, final_relu=True)
    assert rel <= TOL_REL_L2["f32"], rel


@pytest.mark.parametrize("precision", ["tf32", "bf16"])
def test_stack_batch_invariance(precision):
    """Image i of a batch equals the same image recovered alone (every kernel is per-image independent)."""
    import torch
    from paper_1701_03891_b200 import DeepInverse
    case = Case(32, 32, 200, 4, precision, 6, 3, params=stack_params((1, 64, 64, 32, 1)))
    ctx = DeepInverse(case.phi, case.params, 32, 32, precision, max_batch=4)
    y = torch.from_numpy(case.y).to(device="cuda", dtype=ctx.storage_dtype)
    full = ctx.recover(y).cpu().numpy()
    one = ctx.recover(y[2:3].contiguous()).cpu().numpy()
    assert np.array_equal(full[2], one[0])
    ctx.close()


@pytest.mark.parametrize("precision", ["f32", "bf16"])
@pytest.mark.parametrize("widths,n1,n2", [((1, 64, 128, 32, 1), 32, 32), ((1, 32, 128, 128, 64, 32, 1), 24, 40),
                                          ((1, 64, 128, 64, 32, 1), 40, 72), ((1, 64, 128, 32, 1), 13, 130)])
def test_width_128_interior_layers(precision, widths, n1, n2):
    """Width 128 ("larger capacity"): interior 128-channel layers.  BF16 runs k_conv2_tc with
    C_out = 128 (one column tap x 128 filters in M) and C_in = 128 as two 64-channel strips accumulated into the same
    TMEM tile; FP32 the SIMT kernels.  Column segments (n2 = 72, 130) and partial row blocks included."""
    rel, _, _ = run_stack(widths, precision, n1, n2, max(1, n1 * n2 // 6), 2)
    assert rel <= TOL_REL_L2[precision], (widths, rel)


@pytest.mark.parametrize("widths,precision", [((1, 16, 1), "tf32"), ((1, 64, 128, 1), "f32"), ((1, 64, 1), "tf32"),
                                               ((1, 64, 1), "bf16"), ((1, 16, 32, 1), "bf16"),
                                               ((1, 64, 128, 32, 1), "tf32"), ((1, 128, 32, 1), "bf16"),
                                               ((1, 64, 256, 32, 1), "f32")])
def test_stack_unsupported_shapes_are_rejected(widths, precision):
    from paper_1701_03891_b200 import DeepInverse, DiError
    case = Case(16, 16, 64, 1, "f32", params=stack_params(widths))
    with pytest.raises(DiError):
        DeepInverse(case.phi, case.params, 16, 16, precision, max_batch=1)


# ---------------------------------------------------------------------------------------------------- training
TOL_GRAD = {"f32": 1e-4, "tf32": 2e-2, "bf16": 2e-2}


def _stack_case(widths, precision, n1, n2, m, batch):
    return Case(n1, n2, m, batch, precision, 6, 3, params=stack_params(widths))


@pytest.mark.parametrize("precision", ["f32", "tf32", "bf16"])
@pytest.mark.parametrize("widths", [(1, 32, 64, 32, 1), (1, 64, 32, 32, 32, 1), (1, 32, 1), (1, 64, 128, 32, 1)])
def test_stack_gradients_match_oracle(precision, widths):
    """Training custom stacks (NEXT-3): loss and every layer's weight / bias gradient against oracle.train_grad (the
    reverse mode of the literal forward, pinned by central finite differences for arbitrary widths --
    tests/test_oracle_train.py) on the same (bf16-rounded) inputs; 4- and 5-layer stacks and the minimal 2-layer one,
    a ragged 40 x 36 image (TF32 needs n2 % 4 == 0)."""
    import torch
    from paper_1701_03891_b200 import DeepInverse
    if precision == "tf32" and 128 in widths:
        pytest.skip("width 128 runs in FP32 and BF16 contexts")
    case = _stack_case(widths, precision, 40, 36, 250, 3)
    ctx = DeepInverse(case.phi, case.params, case.n1, case.n2, precision, max_batch=case.batch)
    assert ctx.num_params() == sum(w.size + w.shape[0] for w in case.params.w)
    y = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
    x = torch.from_numpy(case.x).cuda()
    loss, g = ctx.train_grad(y, x)
    torch.cuda.synchronize()
    ws, bs = ctx.split(g.cpu().numpy().astype(np.float64))
    rl, rw, rb = oracle.train_grad(case.y, case.x, case.phi, case.params, case.n1, case.n2)
    # the north_star 2e-2 bar is per forward of the paper's 3 layers; in TF32 / BF16 every stored activation adds its
    # rounding to the masks and operands of the backward, so the bar scales with the depth (reading Q15):
    # measured on B200, 5 bf16 layers reach 2.6e-2 on W_0 (fp32: 2e-7)
    tol = TOL_GRAD[precision] * max(1.0, (len(widths) - 1) / 3.0)
    assert abs(float(loss.item()) - rl) <= (1e-5 if precision == "f32" else 1e-2) * abs(rl)
    errs = [(oracle.rel_l2(ws[l], rw[l]), oracle.rel_l2(bs[l], rb[l])) for l in range(len(widths) - 1)]
    print("grad rel-L2 per layer", precision, widths, errs)
    assert max(max(e) for e in errs) <= tol, errs
    ctx.close()


def test_stack_gradients_final_relu_and_xcorr():
    import torch
    from paper_1701_03891_b200 import DI_FLAG_FINAL_RELU, DI_FLAG_XCORR, DeepInverse
    case = _stack_case((1, 32, 32, 1), "f32", 24, 24, 120, 2)
    ctx = DeepInverse(case.phi, case.params, 24, 24, "f32", flags=DI_FLAG_FINAL_RELU | DI_FLAG_XCORR, max_batch=2)
    loss, g = ctx.train_grad(torch.from_numpy(case.y).cuda(), torch.from_numpy(case.x).cuda())
    ws, bs = ctx.split(g.cpu().numpy().astype(np.float64))
    p = synth.Params([w[:, :, ::-1, ::-1].copy() for w in case.params.w], case.params.b)   # oracle: true convolution
    rl, rw, rb = oracle.train_grad(case.y, case.x, case.phi, p, 24, 24, final_relu=True)
    for l in range(3):
        assert oracle.rel_l2(ws[l], rw[l][:, :, ::-1, ::-1]) <= 1e-4, l
        assert oracle.rel_l2(bs[l], rb[l]) <= 1e-4, l
    ctx.close()


@pytest.mark.parametrize("precision", ["f32", "tf32", "bf16"])
def test_stack_sgd_updates_the_forward(precision):
    """di_sgd_step on a custom stack: the parameters move by -lr * grad (momentum 0), the forward runs on the new
    weights (its output matches the oracle's forward over the updated parameters), and the loss decreases."""
    import torch
    from paper_1701_03891_b200 import DeepInverse
    case = _stack_case((1, 32, 64, 32, 1), precision, 32, 32, 200, 4)
    ctx = DeepInverse(case.phi, case.params, 32, 32, precision, max_batch=4)
    y = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
    x = torch.from_numpy(case.x).cuda()
    losses, lr = [], None
    for _ in range(4):
        loss, g = ctx.train_grad(y, x)
        losses.append(float(loss.item()))
        if lr is None:
            lr = 0.05 * losses[0] / float((g.double() ** 2).sum())
            before = ctx.params()
            gflat = g.cpu().numpy()
        ctx.sgd_step(g, lr, 0.0)
        if len(losses) == 1:
            after = ctx.params()
            gw, gb = ctx.split(gflat)
            for l in range(4):
                np.testing.assert_allclose(after[0][l], before[0][l] - np.float32(lr) * gw[l], rtol=0, atol=1e-6)
                np.testing.assert_allclose(after[1][l], before[1][l] - np.float32(lr) * gb[l], rtol=0, atol=1e-6)
            newp = synth.Params([w.copy() for w in after[0]], [b.copy() for b in after[1]]).rounded(
                "bf16" if precision == "bf16" else "f32")
            out = ctx.recover(y).cpu().numpy()
            ref = oracle.forward(case.y, case.phi, newp, 32, 32)
            assert max(oracle.rel_l2(a, r) for a, r in zip(out, ref)) <= TOL_REL_L2[precision]
    assert losses[-1] < losses[0], losses
    ctx.close()
