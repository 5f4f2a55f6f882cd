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
