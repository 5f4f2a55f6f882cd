"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): max per-image rel-L2 <= 1e-5 (fp32 path), <= 2e-2 (bf16 / TF32
tensor-core paths), |dPSNR| <= 0.05 dB per image and for the batch mean.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import TOL_DPSNR, TOL_REL_L2, Case, compare, make_ctx, run, sample_rows, y_device

pytestmark = pytest.mark.gpu


def _check(case, gpu, idx, **kw):
    ref = case.oracle(idx, **kw)
    rel, dps, dmean = compare(gpu[idx], ref, case.x[idx], case.precision)
    assert rel <= TOL_REL_L2[case.precision], f"rel-L2 {rel:.3g}"
    assert dps <= TOL_DPSNR and abs(dmean) <= TOL_DPSNR, f"dPSNR {dps:.3g} mean {dmean:.3g}"
    return rel, dps


# ----------------------------------------------------------------------------- the five configs
@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_tiny(precision):
    """configs[0]: 16x16, M=64, batch 4 (all images checked)."""
    c = synth.CONFIGS["tiny"]
    case = Case(c.n, c.n, c.m, c.batch, precision, c.n_blobs, c.n_rects)
    ctx = make_ctx(case)
    out = run(case, ctx)
    _check(case, out, np.arange(c.batch))


@pytest.mark.parametrize("precision", ["f32", "tf32"])
def test_paper_scale(precision):
    """configs[1]: 64x64, M=1024, batch 256, fp32 and TF32; 32 sampled images."""
    c = synth.CONFIGS["paper"]
    case = Case(c.n, c.n, c.m, c.batch, precision, c.n_blobs, c.n_rects)
    ctx = make_ctx(case)
    out = run(case, ctx)
    _check(case, out, sample_rows(c.batch, 32))


def test_lowrate_full_batch():
    """configs[2]: 64x64, M=410, batch 4096 (the bench launch), bf16; 64 sampled images."""
    c = synth.CONFIGS["lowrate"]
    case = Case(c.n, c.n, c.m, c.batch, "bf16", c.n_blobs, c.n_rects)
    ctx = make_ctx(case)
    out = run(case, ctx)
    assert np.all(np.isfinite(out))
    _check(case, out, sample_rows(c.batch, 64))


def test_larger():
    """configs[3]: 128x128, M=4096, batch 1024, bf16; 16 sampled images."""
    c = synth.CONFIGS["larger"]
    case = Case(c.n, c.n, c.m, c.batch, "bf16", c.n_blobs, c.n_rects)
    ctx = make_ctx(case)
    out = run(case, ctx)
    _check(case, out, sample_rows(c.batch, 16))


@pytest.mark.slow
def test_stress():
    """configs[4] at its full per-GPU batch: 256x256, M=16384 (Phi 2.1 GB bf16), texture noise, batch 256 (the
    bench launch configuration of that config); 4 sampled images against the oracle."""
    c = synth.CONFIGS["stress"]
    case = Case(c.n, c.n, c.m, c.batch, "bf16", c.n_blobs, c.n_rects, c.texture_var)
    ctx = make_ctx(case)
    out = run(case, ctx)
    assert np.all(np.isfinite(out))
    _check(case, out, sample_rows(c.batch, 4))


# ----------------------------------------------------------------------------- edges / flags
@pytest.mark.parametrize("precision", ["f32", "bf16", "tf32"])
@pytest.mark.parametrize("n1,n2,m,batch", [(9, 13, 40, 3), (40, 72, 300, 130), (64, 64, 410, 1), (23, 64, 100, 129),
                                           (70, 150, 700, 5)])
def test_ragged_shapes(precision, n1, n2, m, batch):
    case = Case(n1, n2, m, batch, precision, 6, 3)
    ctx = make_ctx(case)
    out = run(case, ctx)
    _check(case, out, sample_rows(batch, 8))


@pytest.mark.parametrize("precision", ["f32", "bf16", "tf32"])
@pytest.mark.parametrize("bias", ["channel", "fullmap"])
@pytest.mark.parametrize("final_relu,xcorr", [(False, False), (True, True)])
def test_flags_and_biases(precision, bias, final_relu, xcorr):
    from paper_1701_03891_b200 import DI_FLAG_FINAL_RELU, DI_FLAG_XCORR
    case = Case(32, 32, 256, 6, precision, bias=bias)
    flags = (DI_FLAG_FINAL_RELU if final_relu else 0) | (DI_FLAG_XCORR if xcorr else 0)
    ctx = make_ctx(case, flags=flags)
    out = run(case, ctx)
    _check(case, out, np.arange(6), final_relu=final_relu, xcorr=xcorr)


def test_structured_weights_psnr_parity():
    """Closed-form fixture (tests/test_oracle_forward.py): blur of the back-projection; PSNR vs truth is
    meaningful here (7-15 dB), so |dPSNR| is a real check of the bf16 path."""
    from test_oracle_forward import structured_params
    p = structured_params()
    p = synth.Params([w.astype(np.float32) for w in p.w], [b.astype(np.float32) for b in p.b])
    case = Case(64, 64, 410, 8, "bf16", params=p)
    ctx = make_ctx(case)
    out = run(case, ctx)
    rel, dps = _check(case, out, np.arange(8))
    assert 5 < oracle.psnr(out[0], case.x[0]) < 30


# ----------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("precision", ["f32", "bf16"])
def test_invariants_bitwise(precision):
    import torch
    case = Case(64, 64, 410, 20, precision)
    ctx = make_ctx(case, max_batch=20)
    y = y_device(case, ctx)
    a = ctx.recover(y).cpu().numpy()
    b = ctx.recover(y).cpu().numpy()
    assert np.array_equal(a, b), "repeat-run determinism"
    one = ctx.recover(y[7:8].contiguous()).cpu().numpy()
    assert np.array_equal(one[0], a[7]), "batch invariance"
    two = ctx.recover((2 * y).contiguous()).cpu().numpy()
    assert np.array_equal(two, 2 * a), "positive homogeneity (zero biases)"
    zero = ctx.recover(torch.zeros_like(y)).cpu().numpy()
    assert np.all(zero == 0), "y = 0 -> x_hat = 0"


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_shard_outputs_bitwise_identical(precision):
    """SURVEY.md §8(e) check: the batch-sharded path (rank r recovers images [r B/G, (r+1) B/G))
    gives bitwise the outputs of the unsharded batch for G = 1, 2, 4, 8 -- per-image arithmetic does not depend on
    the batch size or on which persistent CTA a unit lands on."""
    case = Case(64, 64, 410, 512, precision)
    ctx = make_ctx(case, max_batch=512)
    y = y_device(case, ctx)
    whole = ctx.recover(y).cpu().numpy()
    for g in (2, 4, 8):
        per = 512 // g
        parts = [ctx.recover(y[r * per:(r + 1) * per].contiguous()).cpu().numpy() for r in range(g)]
        assert np.array_equal(np.concatenate(parts), whole), f"G = {g}"


def test_weight_multicast_and_tile_width_are_bitwise_neutral(monkeypatch):
    """Schedule choices that must not change a single bit: the CTA-pair weight multicast of conv2 (
    DI_EXP_NO_MC=1 at di_create switches it off for that context) and the lifting GEMM's pixel-tile width / batch
    tiles per CTA, which di_create picks from max_batch (224-pixel tiles for max_batch 256, 256-pixel tiles for
    4096 at 64x64)."""
    case = Case(64, 64, 410, 256, "bf16")
    ctx = make_ctx(case, max_batch=256)
    y = y_device(case, ctx)
    mc = ctx.recover(y).cpu().numpy()
    monkeypatch.setenv("DI_EXP_NO_MC", "1")
    ctx_nomc = make_ctx(case, max_batch=256)
    monkeypatch.delenv("DI_EXP_NO_MC")
    nomc = ctx_nomc.recover(y).cpu().numpy()
    assert np.array_equal(mc, nomc), "weight multicast changed the result"
    assert np.array_equal(ctx.recover(y).cpu().numpy(), mc), "the setting is per context"
    monkeypatch.setenv("DI_EXP_C2_CLUSTER", "4")
    ctx4 = make_ctx(case, max_batch=256)
    monkeypatch.delenv("DI_EXP_C2_CLUSTER")
    assert np.array_equal(ctx4.recover(y).cpu().numpy(), mc), "4-CTA weight multicast changed the result"
    big = make_ctx(case, max_batch=4096)
    assert np.array_equal(big.recover(y).cpu().numpy(), mc), "proxy tile width changed the result"


@pytest.mark.parametrize("n1,n2,batch", [(64, 64, 256), (64, 64, 37), (61, 64, 20), (50, 40, 24), (20, 20, 9)])
def test_mixed_row_blocks_are_bitwise_neutral(monkeypatch, n1, n2, batch):
    """conv2's mixed row-block heights (7- and 6-row units where they cut the MMA tiles per image, e.g. 20 instead
    of 22 at 64 x 64) only regroup outputs into tiles: every output still accumulates the same 33
    K-blocks in the same order, so the result equals the uniform 6-row schedule (DI_EXP_C2_MIXED=0) bit for bit."""
    case = Case(n1, n2, max(1, n1 * n2 // 10), batch, "bf16")
    ctx = make_ctx(case)
    y = y_device(case, ctx)
    mixed = ctx.recover(y).cpu().numpy()
    monkeypatch.setenv("DI_EXP_C2_MIXED", "0")
    uni = make_ctx(case)
    monkeypatch.delenv("DI_EXP_C2_MIXED")
    assert np.array_equal(uni.recover(y).cpu().numpy(), mixed)
    idx = np.array([0, batch - 1])
    compare(mixed[idx], case.oracle(idx), case.x[idx], "bf16")


def test_zero_weights_give_bias_only():
    p = synth.make_params(bias="channel")
    p0 = synth.Params([np.zeros_like(w) for w in p.w], p.b)
    case = Case(32, 32, 100, 3, "bf16", params=p0)
    out = run(case, make_ctx(case))
    ref = case.oracle(np.arange(3))
    assert np.allclose(out, ref, atol=1e-6)


def test_host_e2e_matches_device():
    case = Case(64, 64, 410, 33, "bf16")
    ctx = make_ctx(case)
    dev = run(case, ctx)
    import torch
    yh = torch.from_numpy(case.y).to(torch.bfloat16).pin_memory()
    host = ctx.recover_host(yh)
    assert np.array_equal(host, dev)


def test_host_e2e_multichunk_bitwise():
    """di_recover_host's chunked branch (batch >= 512: chunks shrinking 4x: 3072 + 768 + 260 at 4100, y split between the compute and the copy
    stream, per-chunk D2H on the copy stream) gives bitwise the device-resident di_recover result: batch 512, 515
    (ragged last chunk), 4096 (the bench's e2e call) and max_batch, with pinned and pageable y, repeated on the same
    context (workspace reuse, y staging regrown)."""
    import torch
    maxb = 4100
    case = Case(64, 64, 410, maxb, "bf16", 4, 2)
    ctx = make_ctx(case, max_batch=maxb)
    yd = y_device(case, ctx)
    dev = ctx.recover(yd).cpu().numpy()
    ypin = torch.from_numpy(case.y).to(torch.bfloat16).pin_memory()
    ypage = torch.from_numpy(case.y).to(torch.bfloat16)
    for b in (512, 515, 4096, maxb, 515):
        for yh in (ypin, ypage):
            host = ctx.recover_host(yh[:b])
            assert np.array_equal(host, dev[:b]), f"batch {b} pinned={yh.is_pinned()}"
    out = torch.empty((600, 64, 64), dtype=torch.float32).pin_memory()
    ctx.recover_host(ypin[100:700], out)
    assert np.array_equal(out.numpy(), dev[100:700])


def test_host_e2e_fp32_numpy_and_validation():
    """FP32 context through numpy host buffers (pageable), chunked; wrong dtypes / shapes raise TypeError."""
    import torch
    case = Case(32, 32, 200, 520, "f32", 3, 1)
    ctx = make_ctx(case)
    dev = run(case, ctx)
    assert np.array_equal(ctx.recover_host(case.y), dev)
    with pytest.raises(TypeError):
        ctx.recover_host(case.y.astype(np.float64))
    with pytest.raises(TypeError):
        ctx.recover_host(case.y, np.empty((520, 32, 33), np.float32))
    bctx = make_ctx(Case(32, 32, 200, 4, "bf16", 3, 1))
    with pytest.raises(TypeError):
        bctx.recover_host(case.y[:4])                                 # float32 numpy into a bf16 context
    with pytest.raises(TypeError):
        bctx.recover(torch.zeros((4, 200), dtype=torch.float32, device="cuda"))
    with pytest.raises(TypeError):
        bctx.recover(torch.zeros((200, 4), dtype=torch.bfloat16, device="cuda").t())   # column stride != 1


def test_device_phi_is_rne_bf16():
    case = Case(16, 16, 64, 2, "bf16")
    ctx = make_ctx(case)
    assert np.array_equal(ctx.phi_device_copy(), synth.f32_to_bf16_bits(case.phi))


def test_misaligned_ldy_staging():
    import torch
    case = Case(64, 64, 410, 9, "bf16")
    ctx = make_ctx(case)
    ref = run(case, ctx)
    big = torch.zeros((9, 413), dtype=torch.bfloat16, device="cuda")
    big[:, :410] = torch.from_numpy(case.y).to(torch.bfloat16)
    view = big[:, :410]
    out = ctx.recover(view)          # ldy = 413 -> 826-B rows: staged copy path
    assert np.array_equal(out.cpu().numpy(), ref)


def test_error_codes():
    from paper_1701_03891_b200 import DiError
    import torch
    case = Case(16, 16, 64, 2, "bf16")
    ctx = make_ctx(case, max_batch=2)
    y = torch.zeros((3, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(DiError) as e:
        ctx.recover(y)
    assert e.value.status == 1
    from paper_1701_03891_b200 import di_recover
    y63 = torch.zeros((2, 63), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(TypeError):                       # the binding checks the shape first
        ctx.recover(y63)
    with pytest.raises(DiError) as e:                    # the C ABI: ldy < m is DI_ERR_DIM
        di_recover(ctx.ctx, y63, 63, 2, torch.empty((2, 16, 16), device="cuda"))
    assert e.value.status == 2


# ----------------------------------------------------------------------------- per stage
@pytest.mark.parametrize("precision", ["f32", "bf16", "tf32"])
def test_stages_individually(precision):
    """di_debug_stage: each stage against the oracle on the GPU's own stage input."""
    import torch
    case = Case(40, 64, 300, 4, precision)
    ctx = make_ctx(case)
    dt = ctx.storage_dtype
    n1, n2, B = case.n1, case.n2, case.batch
    y = y_device(case, ctx)
    xt = torch.empty((B, n1, n2), dtype=dt, device="cuda")
    h1 = torch.empty((B, n1, n2, 64), dtype=dt, device="cuda")
    h2 = torch.empty((B, n1, n2, 32), dtype=dt, device="cuda")
    xh = torch.empty((B, n1, n2), dtype=torch.float32, device="cuda")
    ctx.debug_stage(0, y, xt, B)
    ctx.debug_stage(1, xt, h1, B)
    ctx.debug_stage(2, h1, h2, B)
    ctx.debug_stage(3, h2, xh, B)
    torch.cuda.synchronize()
    tol = 1e-5 if precision == "f32" else 8e-3   # bf16 stage outputs are rounded to bf16 (2^-9); tf32 products
    f = lambda t: t.float().cpu().numpy().astype(np.float64)
    ref0 = oracle.proxy(case.phi, case.y).reshape(B, n1, n2)
    assert oracle.rel_l2(f(xt), ref0) <= tol
    p = case.params
    for b in range(B):
        r1 = oracle.conv_layer(f(xt)[b][None], p.w[0], p.b[0], relu=True)
        assert oracle.rel_l2(f(h1)[b].transpose(2, 0, 1), r1) <= tol
        r2 = oracle.conv_layer(f(h1)[b].transpose(2, 0, 1), p.w[1], p.b[1], relu=True)
        assert oracle.rel_l2(f(h2)[b].transpose(2, 0, 1), r2) <= tol
        r3 = oracle.conv_layer(f(h2)[b].transpose(2, 0, 1), p.w[2], p.b[2], relu=False)
        # stage 3 reads exact stage-2 values: fp32 FFMA ~1e-6; bf16 operands are exact, fp32 accumulation ~1e-6;
        # TF32 truncates the fp32 h2 and weights to 10-bit mantissas (2^-11 per product)
        tol3 = {"f32": 1e-5, "bf16": 1e-4, "tf32": 2e-3}[precision]
        assert oracle.rel_l2(f(xh)[b], r3[0]) <= tol3


# ----------------------------------------------------------------------------- degenerate shapes
@pytest.mark.parametrize("precision", ["f32", "bf16", "tf32"])
@pytest.mark.parametrize("n1,n2,m,batch", [
    (1, 1, 1, 2),        # N = 1, M = 1: every tap but the centre reads the zero padding
    (1, 64, 16, 3),      # one-row images (strip mostly padding)
    (64, 1, 16, 3),      # one-column images
    (8, 8, 64, 5),       # M = N (square Phi)
    (5, 8, 1, 4),        # a single measurement
    (16, 4, 30, 3),      # n2 = 4: smallest width with an fp32 TMA row (TF32 conv1 strip)
    (3, 200, 50, 2),     # n2 > 64 with a ragged last column segment, fewer rows than a unit
])
def test_degenerate_shapes(precision, n1, n2, m, batch):
    case = Case(n1, n2, m, batch, precision, 3, 2)
    ctx = make_ctx(case)
    out = run(case, ctx)
    assert np.all(np.isfinite(out))
    ref = case.oracle(np.arange(batch))
    rel, _, _ = compare(out, ref, case.x, precision)      # includes the element-wise bound
    assert rel <= TOL_REL_L2[precision], rel


def test_batch_zero_and_oversize_are_argument_errors():
    import torch
    from paper_1701_03891_b200 import DiError, di_recover
    case = Case(16, 16, 64, 2, "bf16")
    ctx = make_ctx(case, max_batch=2)
    y = torch.zeros((2, 64), dtype=torch.bfloat16, device="cuda")
    out = torch.empty((2, 16, 16), device="cuda")
    for b in (0, -1, 3):
        with pytest.raises(DiError) as e:
            di_recover(ctx.ctx, y, 64, b, out)
        assert e.value.status == 1


# ----------------------------------------------------------------------------- learned lifting (NEXT-3)
@pytest.mark.parametrize("precision", ["f32", "bf16", "tf32"])
def test_learned_lifting_matrix(precision):
    """A learned lifting L [N][M] replaces Phi^T in the first layer; Phi still senses (di_measure)."""
    import torch
    from paper_1701_03891_b200 import DeepInverse
    case = Case(24, 40, 200, 5, precision, 4, 2)
    r = np.random.default_rng(99)
    lift = (r.standard_normal((case.n1 * case.n2, case.m)) / np.sqrt(case.m)).astype(np.float32)
    if precision == "bf16":
        lift = synth.round_bf16(lift)
    ctx = DeepInverse(case.phi, case.params, case.n1, case.n2, precision, max_batch=case.batch, lift=lift)
    out = run(case, ctx)
    ref = oracle.forward(case.y, lift.T, case.params, case.n1, case.n2)   # x_tilde = (L^T)^T y = L y
    assert max(oracle.rel_l2(g, r_) for g, r_ in zip(out, ref)) <= TOL_REL_L2[precision]
    xs = synth.round_bf16(case.x) if precision == "bf16" else case.x
    y = ctx.measure(torch.from_numpy(case.x).cuda()).float().cpu().numpy()
    ym = oracle.measure(case.phi, xs)
    assert max(oracle.rel_l2(a, b) for a, b in zip(y, ym)) <= (1e-5 if precision == "f32" else 1e-2)


def test_inference_time_flat_across_measurement_rate():
    """PAPER.md Table 1 (§5): DeepInverse's recovery time does not depend on M/N -- the lifting GEMM is a small
    share next to the convolutions.  bf16, 64x64, batch 1024, M/N from 0.01 to 0.5: the slowest and fastest
    median di_recover times stay within 15 %."""
    import torch
    from paper_1701_03891_b200 import DeepInverse
    n, B = 64, 1024
    times = {}
    for m in (41, 410, 1229, 2048):
        phi = synth.make_phi(m, n * n, "bf16")
        ctx = DeepInverse(phi, synth.make_params().rounded("bf16"), n, n, "bf16", max_batch=B)
        y = torch.randn((B, m), device="cuda").to(torch.bfloat16)
        out = torch.empty((B, n, n), device="cuda")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(2):
            ctx.recover(y, out)
        ts = []
        for _ in range(5):
            ev[0].record()
            ctx.recover(y, out)
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        times[m] = float(np.median(ts))
        ctx.close()
    assert max(times.values()) <= 1.15 * min(times.values()), times


@pytest.mark.parametrize("n,m,batch", [(128, 4096, 512), (96, 2000, 300), (64, 410, 256)])
def test_proxy_on_cta_pairs(monkeypatch, n, m, batch):
    """The lifting GEMM on CTA pairs (k_proxy_pair: cta_group::2, M = 256 images over two SMs, two BN-pixel
    accumulators per CTA) against the oracle's x_tilde = Phi^T y element by element (stage 0 hook,
    bound from the arithmetic as in test_gpu_elementwise.py) and against the one-CTA kernel.  Ragged batch (300 = one
    full and one partial 256-image pair tile) and an N that is not a multiple of the pair's 2 x BN pixels."""
    import torch
    case = Case(n, n, m, batch, "bf16", 6, 3)
    monkeypatch.setenv("DI_EXP_PROXY_PAIR", "1")
    ctx = make_ctx(case)
    monkeypatch.setenv("DI_EXP_PROXY_PAIR", "0")
    ref_ctx = make_ctx(case)
    monkeypatch.delenv("DI_EXP_PROXY_PAIR")
    y = y_device(case, ctx)
    outs = []
    for c in (ctx, ref_ctx):
        xt = torch.empty((batch, n, n), dtype=torch.bfloat16, device="cuda")
        c.debug_stage(0, y, xt, batch)
        torch.cuda.synchronize()
        outs.append(xt.float().cpu().numpy().astype(np.float64))
    rows = sample_rows(batch, 6)
    ref = oracle.proxy(case.phi, case.y[rows]).reshape(len(rows), n, n)
    S = oracle.proxy(np.abs(case.phi), np.abs(case.y[rows])).reshape(len(rows), n, n)
    err = np.abs(outs[0][rows] - ref)
    assert np.all(err <= 2.0 ** -8 * np.abs(ref) + 2.0 ** -14 * S), float(err.max())
    assert np.array_equal(outs[0], outs[1]), "pair kernel differs from the one-CTA kernel"


def test_c_example_on_gpu(tmp_path):
    """The C ABI from plain C (examples/recover.c, host buffers through di_recover_host): y = 0 -> 0 and x_hat(2y) =
    2 x_hat(y) bitwise, synchronous argument errors."""
    import json
    import subprocess
    from test_abi import _build_c_example
    r = subprocess.run([_build_c_example(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout)
    assert d["homogeneity_and_zero_mismatches"] == 0 and d["arg_errors_ok"] == 1 and d["norm"] > 0
