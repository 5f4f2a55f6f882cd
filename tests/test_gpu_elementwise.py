"""Element-wise GPU parity, stage by stage, at shapes that put outputs on every tile tail and segment seam.

Per-image rel-L2 (the north_star statistic, tests/test_gpu_parity.py) cannot see one wrong pixel: at the 2e-2 bar a
completely wrong output costs 1/64 = 1.6 % at 64x64.  Here every output element of every stage is held to a bound
derived from the arithmetic of that element (forward error analysis), with
    S = sum over the element's terms of |w| |x|     (the oracle's conv / proxy applied to |W| and |X|)
  * bf16 storage (x_tilde, h1, h2 of the BF16 path): RNE to bf16 of an fp32 accumulation of exact bf16 products:
        |gpu - ref| <= 2^-8 |ref| + 2^-14 S
  * TF32 products (both operands truncated / rounded to a 10-bit mantissa) accumulated in fp32:
        |gpu - ref| <= 1.1 * 2^-9 S
  * fp32 FFMA accumulation, and the BF16 path's fp32 x_hat from exact bf16 products:
        |gpu - ref| <= 2^-14 S
ReLU is 1-Lipschitz, so the bounds pass through it.  A dropped tap, a wrong column shift of one TMEM quadrant or a
stale chunk costs a whole term (|w x| ~ S / n_terms ... S) and fails.  The oracle runs on the GPU's own input of each
stage (di_debug_stage), so each stage is checked alone.

Impulse probes: with one unit input at (image, row, column, channel) and zero biases, every output of a layer is ONE
product w * 1 -- exact in every precision -- so the response must equal the flipped 11x11 tap window of that channel
exactly (bf16: bitwise; TF32: the tf32 value of the tap), and must be zero everywhere else.  The impulses sit where
the responses land on conv2's tile tails (the balanced split 205 / 237 of a unit, chunk c0 = 240 of a 256-column
TMEM tile and the 253-output overlap), the boundary between 7- and 6-row blocks, the 64-column segment seams (pitch
74), the last partial row block, the image corners, and the 11-row units of conv3.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import Case, make_ctx, y_device

pytestmark = pytest.mark.gpu

C = (1, 64, 32, 1)
C2_ROWS, WSEG, NT, OUT_PER_TILE = 6, 64, 256, 253   # conv2 unit geometry: probes aim at its tiles


def _bound(ref, S, precision, stored_bf16):
    if precision == "tf32":
        return 1.1 * 2.0 ** -9 * S
    if stored_bf16:
        return 2.0 ** -8 * np.abs(ref) + 2.0 ** -14 * S
    return 2.0 ** -14 * S


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _run_stages(ctx, case):
    import torch
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
    return [_f64(xt)[:, None], _f64(h1).transpose(0, 3, 1, 2), _f64(h2).transpose(0, 3, 1, 2), _f64(xh)[:, None]]


SEAM_SHAPES = [(64, 64),     # the bench geometry: P = 69, 4 blocks of 7 rows (tiles 237 + 241), 6 of 6 (205 + 204)
               (61, 128),    # two 64-column segments (P = 74), a 1-row last row block
               (13, 130),    # three segments, the last 2 columns wide; 2 row blocks, the last 1 row
               (61, 65),     # a 1-column last segment
               (40, 72),     # ragged second segment, 4-row last block
               (61, 64),     # mixed row-block heights: 7 blocks of 7 rows, 2 of 6
               (20, 48),     # one segment narrower than 64 columns with n2 % 8 == 0 (conv1's TMA strip, P = 53)
               (9, 13)]      # one small unit: a single partial tile


@pytest.mark.parametrize("precision", ["bf16", "tf32", "f32"])
@pytest.mark.parametrize("n1,n2", SEAM_SHAPES)
def test_every_element_of_every_stage(precision, n1, n2):
    case = Case(n1, n2, max(1, (n1 * n2) // 10), 2, precision, 6, 3)
    ctx = make_ctx(case)
    outs = _run_stages(ctx, case)
    p = case.params
    bf = precision == "bf16"

    def stage_ref(s, b):
        if s == 0:
            ref = oracle.proxy(case.phi, case.y[b:b + 1]).reshape(1, n1, n2)
            S = oracle.proxy(np.abs(case.phi), np.abs(case.y[b:b + 1])).reshape(1, n1, n2)
            return ref, S
        x = outs[s - 1][b]
        ref = oracle.conv_layer(x, p.w[s - 1], None, relu=(s < 3))
        S = oracle.conv_layer(np.abs(x), np.abs(np.asarray(p.w[s - 1], np.float64)), None, relu=False)
        return ref, S

    jobs = [(s, b) for s in range(4) for b in range(case.batch)]
    with ThreadPoolExecutor(8) as ex:               # ctypes releases the GIL: the oracle calls run in parallel
        refs = list(ex.map(lambda sb: stage_ref(*sb), jobs))
    for (s, b), (ref, S) in zip(jobs, refs):
        got = outs[s][b]
        assert got.shape == ref.shape, (s, got.shape, ref.shape)
        tol = _bound(ref, S, precision, stored_bf16=bf and s < 3)
        err = np.abs(got - ref)
        bad = np.argwhere(err > tol)
        assert bad.size == 0, (f"stage {s} image {b}: {len(bad)} elements out of bound, first (ch, r, c) = "
                               f"{bad[:5].tolist()}, err {err[tuple(bad[0])]:.3g} > tol {tol[tuple(bad[0])]:.3g}")


# ------------------------------------------------------------------------------------------------ impulse probes
def _ntiles(L):
    return (L + OUT_PER_TILE - 1) // OUT_PER_TILE


def _row_blocks(n1, n2):
    """conv2's row blocks (r0, rows): 6-row blocks and a short last one, or -- one column segment, when it needs
    fewer tiles and every block runs the same number -- ntall 7-row blocks then 6-row ones (mixed heights, DESIGN.md
    §6).  An independent restatement of the kernel's rule, used only to aim the probes."""
    wseg = min(n2, WSEG)
    P = n2 + 5 if n2 <= WSEG else WSEG + 10
    uniform = [(r0, min(C2_ROWS, n1 - r0)) for r0 in range(0, n1, C2_ROWS)]
    nrb = (n1 + C2_ROWS) // (C2_ROWS + 1)
    ntall = n1 - C2_ROWS * nrb
    if n2 > WSEG or not 0 < ntall <= nrb or _ntiles(C2_ROWS * P + wseg) != _ntiles((C2_ROWS - 1) * P + wseg):
        return uniform
    mixed, r0 = [], 0
    for rb in range(nrb):
        rows = C2_ROWS + (rb < ntall)
        mixed.append((r0, rows))
        r0 += rows
    tiles = lambda blocks: sum(_ntiles((r - 1) * P + wseg) for _, r in blocks)
    return mixed if tiles(mixed) < tiles(uniform) else uniform


def _conv2_tile_positions(n1, n2):
    """Image positions (r, c) of conv2 outputs at tile tails: positions 237 / 240 / 252 / 253 of a unit's strip
    (the first tile of a 7-row unit ends at 237, chunk c0 = 240, the last of 253 complete outputs, the first of the
    next tile) and the unit's last position, for the first, a middle and the last row block (and the last 7-row
    block when heights are mixed) and every column segment."""
    wseg = min(n2, WSEG)
    P = n2 + 5 if n2 <= WSEG else WSEG + 10
    blocks = _row_blocks(n1, n2)
    pick = {0, len(blocks) // 2, len(blocks) - 1}
    pick |= {i for i in range(1, len(blocks)) if blocks[i][1] != blocks[i - 1][1]} | \
        {i - 1 for i in range(1, len(blocks)) if blocks[i][1] != blocks[i - 1][1]}
    out = []
    for i in sorted(pick):
        r0, rows = blocks[i]
        L = (rows - 1) * P + wseg
        for seg in range((n2 + wseg - 1) // wseg):
            c0 = seg * wseg
            for o in (204, 205, 236, 237, 240, 252, 253, L - 1):
                if o >= L:
                    continue
                rr, cc = divmod(o, P)
                if cc < wseg and c0 + cc < n2:
                    out.append((r0 + rr, c0 + cc))
    return out


def _probe_positions(n1, n2):
    pos = [(0, 0), (0, n2 - 1), (n1 - 1, 0), (n1 - 1, n2 - 1), (n1 // 2, n2 // 2)]
    pos += _conv2_tile_positions(n1, n2)
    for seam in range(WSEG, n2, WSEG):                       # segment seams: the last / first column of a segment
        pos += [(n1 // 2, seam - 1), (n1 // 2, seam), (n1 - 1, seam - 1), (0, seam)]
    for r in range(10, n1, 11):                              # conv3's 11-row units: last row, first of the next
        pos += [(r, min(n2 - 1, 33)), (min(n1 - 1, r + 1), min(n2 - 1, 40))]
    return sorted(set(pos))


def _impulse_case(n1, n2, precision, stage, positions):
    """One impulse per image (no two responses overlap), the channel varying with the image."""
    import torch
    cin = C[stage - 1]
    B = len(positions)
    x = np.zeros((B, n1, n2, cin), np.float32)
    chans = [(7 * i + 3) % cin for i in range(B)]
    for i, ((r, c), ch) in enumerate(zip(positions, chans)):
        x[i, r, c, ch] = 1.0
    dt = torch.bfloat16 if precision == "bf16" else torch.float32
    t = torch.from_numpy(x if cin > 1 else x[..., 0]).to(device="cuda", dtype=dt)
    return t, chans


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
@pytest.mark.parametrize("stage", [1, 2, 3])
@pytest.mark.parametrize("n1,n2", [(64, 64), (61, 128), (13, 130), (40, 72)])
def test_impulse_response_is_the_tap_window(precision, stage, n1, n2):
    import torch
    positions = _probe_positions(n1, n2)
    case = Case(n1, n2, 8, len(positions), precision, 1, 0)
    ctx = make_ctx(case)
    xin, chans = _impulse_case(n1, n2, precision, stage, positions)
    B = len(positions)
    cout = C[stage]
    dt = ctx.storage_dtype if stage < 3 else torch.float32
    shape = (B, n1, n2, cout) if cout > 1 else (B, n1, n2)
    out = torch.empty(shape, dtype=dt, device="cuda")
    ctx.debug_stage(stage, xin, out, B)
    torch.cuda.synchronize()
    got = _f64(out)
    if cout == 1:
        got = got[..., None]
    w = np.asarray(case.params.w[stage - 1], np.float64)
    for i, ((r, c), ch) in enumerate(zip(positions, chans)):
        one = np.zeros((1, n1, n2))
        one[0, r, c] = 1.0
        ref = oracle.conv_layer(one, w[:, ch:ch + 1], None, relu=(stage < 3))      # zero channels add exact zeros
        ref = ref.transpose(1, 2, 0)
        g = got[i]
        assert np.all((g != 0) <= (ref != 0)), f"image {i} impulse at {(r, c)}: output outside the tap window"
        if precision == "bf16":
            assert np.array_equal(g, ref), (f"image {i} impulse at {(r, c)} ch {ch}: "
                                            f"{np.argwhere(g != ref)[:5].tolist()}")
        else:   # TF32: the product is the tap's tf32 value (10-bit mantissa)
            np.testing.assert_allclose(g, ref, rtol=2.0 ** -10, atol=0, err_msg=f"impulse at {(r, c)}")
