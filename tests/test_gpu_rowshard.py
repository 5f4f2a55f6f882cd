"""Row-sharded Phi on one GPU: each "rank" is a context over a row block of Phi
(rowshard.row_range); its fp32 partial proxy (di_proxy_partial) is checked against the oracle's proxy of that row
block, the partials are summed on the device (a stand-in for the reduce-scatter; the collective itself is
covered by tests/test_multiproc.py over gloo) and the convolutions on each batch block (di_recover_from_proxy)
are checked against the oracle's forward pass over the FULL Phi -- x_tilde = sum_g Phi_g^T y_g."""
import numpy as np
import pytest

import oracle
from gpu_helpers import TOL_REL_L2, Case, compare

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision,n,m,batch,world", [("bf16", 16, 64, 4, 2), ("bf16", 64, 410, 6, 3),
                                                        ("tf32", 32, 256, 4, 2), ("f32", 16, 100, 4, 4),
                                                        ("bf16", 40, 333, 4, 2)])
def test_row_sharded_recovery_matches_full_phi(precision, n, m, batch, world):
    import torch
    from paper_1701_03891_b200 import DeepInverse, batch_range, row_range
    case = Case(n, n, m, batch, precision, bias="channel")
    ctxs, parts = [], []
    for g in range(world):
        lo, hi = row_range(m, world, g)
        ctx = DeepInverse(np.ascontiguousarray(case.phi[lo:hi]), case.params, n, n, precision, max_batch=batch)
        y = torch.from_numpy(np.ascontiguousarray(case.y[:, lo:hi])).to("cuda", ctx.storage_dtype)
        part = ctx.proxy_partial(y)
        torch.cuda.synchronize()
        ref = oracle.proxy(case.phi[lo:hi], case.y[:, lo:hi])
        tol = 1e-5 if precision != "tf32" else 4e-3     # fp32 accumulation of exact (bf16/fp32) products
        assert max(oracle.rel_l2(a, r) for a, r in zip(part.cpu().numpy(), ref.reshape(batch, -1))) <= tol
        ctxs.append(ctx), parts.append(part)
    total = torch.stack(parts).sum(0)                   # the reduce-scatter's sum
    ref = case.oracle(np.arange(batch))
    for g in range(world if batch % world == 0 else 1):
        lo, hi = batch_range(batch, world, g) if batch % world == 0 else (0, batch)
        out = ctxs[g].recover_from_proxy(total[lo:hi].contiguous())
        torch.cuda.synchronize()
        rel, dps, _ = compare(out.cpu().numpy(), ref[lo:hi], case.x[lo:hi], precision)
        assert rel <= TOL_REL_L2[precision], rel
    for c in ctxs:
        c.close()


def test_single_shard_equals_replicated_recover():
    """world = 1: di_proxy_partial + di_recover_from_proxy reproduces di_recover (fp32 path bit for bit)."""
    import torch
    from paper_1701_03891_b200 import DeepInverse
    case = Case(16, 16, 64, 4, "f32", bias="channel")
    ctx = DeepInverse(case.phi, case.params, 16, 16, "f32", max_batch=4)
    y = torch.from_numpy(case.y).cuda()
    a = ctx.recover(y).cpu().numpy()
    b = ctx.recover_from_proxy(ctx.proxy_partial(y)).cpu().numpy()
    assert np.array_equal(a, b)
    ctx.close()


def test_recover_from_proxy_argument_errors():
    import torch
    from paper_1701_03891_b200 import DeepInverse, DiError
    case = Case(16, 16, 64, 2, "bf16")
    ctx = DeepInverse(case.phi, case.params, 16, 16, "bf16", max_batch=2)
    with pytest.raises(DiError):
        ctx.recover_from_proxy(torch.zeros((3, 256), device="cuda"))   # batch > max_batch
    with pytest.raises(TypeError):
        ctx.recover_from_proxy(torch.zeros((2, 256), device="cuda", dtype=torch.bfloat16))
    ctx.close()


@pytest.mark.parametrize("precision,n,m,batch,world", [("bf16", 32, 256, 4, 2), ("bf16", 64, 410, 6, 3),
                                                        ("tf32", 16, 100, 4, 4), ("f32", 16, 100, 4, 2)])
def test_fused_scatter_matches_full_phi_and_the_unfused_form(precision, n, m, batch, world):
    """di_proxy_scatter (the lifting GEMM's epilogue storing each image's partial rows into the owner's slot) and
    di_recover_from_slots (the owner's rank-order slot sum + convolutions), with `world` virtual ranks on one GPU:
    each rank's GEMM runs to completion before the next (no kernel waits on another), writing into the owners'
    staging buffers through plain device pointers -- on G GPUs the same pointers are CUDA-IPC peer mappings.  Equal
    bit for bit to di_recover_from_proxy on the same rank-order sum, and to the full-Phi oracle within tolerance."""
    import torch
    from paper_1701_03891_b200 import DeepInverse, batch_range, row_range
    case = Case(n, n, m, batch, precision, bias="channel")
    N, nb = n * n, batch // world
    staging = [torch.zeros((world, nb, N), dtype=torch.float32, device="cuda") for _ in range(world)]
    ctxs, parts = [], []
    for g in range(world):
        lo, hi = row_range(m, world, g)
        ctx = DeepInverse(np.ascontiguousarray(case.phi[lo:hi]), case.params, n, n, precision, max_batch=batch)
        y = torch.from_numpy(np.ascontiguousarray(case.y[:, lo:hi])).to("cuda", ctx.storage_dtype)
        ctx.proxy_scatter(y, [s.data_ptr() for s in staging], world, g)
        parts.append(ctx.proxy_partial(y))
        ctxs.append(ctx)
    torch.cuda.synchronize()
    ref = case.oracle(np.arange(batch))
    for r in range(world):
        lo, hi = batch_range(batch, world, r)
        for g in range(world):   # slot g of owner r holds rank g's partial rows of r's block
            assert torch.equal(staging[r][g], parts[g][lo:hi])
        out = ctxs[r].recover_from_slots(staging[r], world).cpu().numpy()
        total = parts[0][lo:hi].clone()
        for g in range(1, world):
            total += parts[g][lo:hi]
        ref_unfused = ctxs[r].recover_from_proxy(total.contiguous()).cpu().numpy()
        assert np.array_equal(out, ref_unfused)
        rel, _, _ = compare(out, ref[lo:hi], case.x[lo:hi], precision)
        assert rel <= TOL_REL_L2[precision], rel
    for c in ctxs:
        c.close()


def test_fused_single_rank_recover():
    """RowShardedDeepInverse.recover(fused=True) without a process group (world = 1) equals the replicated path."""
    import torch
    from paper_1701_03891_b200 import RowShardedDeepInverse
    case = Case(32, 32, 256, 4, "bf16", bias="channel")
    rs = RowShardedDeepInverse(case.phi, case.params, 32, 32, "bf16", max_batch=4)
    y = torch.from_numpy(case.y).to("cuda", torch.bfloat16)
    a = rs.recover(y, fused=True).cpu().numpy()
    b = rs.ctx.recover(y).cpu().numpy()
    rel = max(oracle.rel_l2(u, v) for u, v in zip(a, b))
    assert rel <= 1e-6, rel   # the bf16 rounding of an fp32 proxy vs the GEMM's own bf16 epilogue
    rs.close()


def test_proxy_scatter_argument_errors():
    import torch
    from paper_1701_03891_b200 import DeepInverse, DiError
    case = Case(16, 16, 64, 4, "bf16")
    ctx = DeepInverse(case.phi, case.params, 16, 16, "bf16", max_batch=4)
    y = torch.from_numpy(case.y).to("cuda", torch.bfloat16)
    buf = torch.zeros((3, 1, 256), device="cuda")
    with pytest.raises(DiError):
        ctx.proxy_scatter(y, [buf.data_ptr()] * 3, 3, 0)      # batch 4 not a multiple of 3
    with pytest.raises(DiError):
        ctx.proxy_scatter(y, [buf.data_ptr()] * 2, 2, 2)      # rank outside [0, world)
    ctx.close()
