"""Multi-process host logic of the batch-sharded path (bench.py), world_size 2 over gloo on CPU.

The GPU path shards images across ranks with no data-path collective; what the ranks
share is the sharding rule, the max-over-ranks timing and the seeded inputs, which must be identical
however the batch is split.
"""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

import bench
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = bench.dist_env()
        per = 3
        lo, hi = bench.shard(r, per)
        c = synth.CONFIGS["tiny"]
        x = synth.make_images(c.n, lo, hi - lo, c.n_blobs, c.n_rects)
        # max over ranks of a per-rank "device time"
        t = bench.max_over_ranks(1.0 + r)
        bench.barrier()
        # gather the shards to rank 0 (checking only, as in the GPU harness)
        xt = torch.from_numpy(x)
        parts = [torch.empty_like(xt) for _ in range(w)]
        dist.all_gather(parts, xt)
        if r == 0:
            q.put((lo, hi, t, bench.aggregate(per, w, t), torch.cat(parts).numpy()))
        else:
            q.put((lo, hi, t, None, None))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_timing_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = sorted((a, b) for a, b, *_ in res)
    assert ranges == [(0, 3), (3, 6)], "contiguous blocks of global image indices"
    assert all(t == 2.0 for _, _, t, _, _ in res), "max over ranks"
    agg, gathered = next((a, g) for *_, a, g in res if a is not None)
    assert agg == 6 / 2.0, "whole-job throughput = all ranks' units / slowest rank"
    c = synth.CONFIGS["tiny"]
    whole = synth.make_images(c.n, 0, 6, c.n_blobs, c.n_rects)
    assert np.array_equal(gathered, whole), "sharded inputs identical to the unsharded batch"


def test_single_process_defaults():
    assert bench.dist_env()[1] >= 1
    assert bench.shard(0, 4096) == (0, 4096)
    assert bench.max_over_ranks(3.5) == 3.5


def _train_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        phi, p, y, x, n1, n2 = _train_case()
        per = y.shape[0] // world
        sl = slice(rank * per, (rank + 1) * per)
        loss, dws, dbs = oracle.train_grad(y[sl], x[sl], phi, p, n1, n2, scale=1.0 / y.shape[0], threads=1)
        flat = torch.from_numpy(np.concatenate([g.ravel() for g in dws + dbs] + [np.array([loss])]))
        dist.all_reduce(flat)          # the one collective of data-parallel training (tools/train_dp.py)
        if rank == 0:
            q.put(flat.numpy())
    finally:
        dist.destroy_process_group()


def _train_case():
    r = np.random.default_rng(7)
    n1, n2, m, b = 6, 6, 20, 4
    phi = r.standard_normal((m, n1 * n2)) / np.sqrt(m)
    widths = (1, 3, 2, 1)
    ws = [r.standard_normal((widths[l + 1], widths[l], 3, 3)) * 0.5 for l in range(3)]
    bs = [r.uniform(-0.1, 0.1, widths[l + 1]) for l in range(3)]
    return phi, synth.Params(ws, bs), r.standard_normal((b, m)), r.uniform(0, 1, (b, n1, n2)), n1, n2


def test_two_rank_gradient_allreduce_equals_full_batch_gradient():
    """Data-parallel training: shard gradients with scale 1/global batch, summed by all_reduce, equal the
    full-batch gradient (the decomposition tools/train_dp.py relies on)."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = q.get(timeout=120)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    phi, p, y, x, n1, n2 = _train_case()
    loss, dws, dbs = oracle.train_grad(y, x, phi, p, n1, n2, scale=1.0 / y.shape[0], threads=1)
    ref = np.concatenate([g.ravel() for g in dws + dbs] + [np.array([loss])])
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-15)


def _rowshard_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1701_03891_b200.rowshard import batch_range, row_range, sum_scatter
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        phi, y = _rowshard_case()
        lo, hi = row_range(phi.shape[0], world, rank)
        part = torch.from_numpy(oracle.proxy(phi[lo:hi], y[:, lo:hi]).reshape(y.shape[0], -1))
        mine = sum_scatter(part)                       # the one collective of the row-sharded path
        q.put((rank, (lo, hi), batch_range(y.shape[0], world, rank), mine.numpy()))
    finally:
        dist.destroy_process_group()


def _rowshard_case():
    r = np.random.default_rng(11)
    m, n, b = 37, 8, 4
    return r.standard_normal((m, n * n)) / np.sqrt(m), r.standard_normal((b, m))


def test_two_rank_row_sharded_proxy_reduce_scatter():
    """NEXT-4 host logic: the row blocks tile Phi's rows, and the reduce-scatter of the per-rank partial proxies
    leaves each rank the full-Phi proxy of its batch block (x_tilde = sum_g Phi_g^T y_g)."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rowshard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    phi, y = _rowshard_case()
    assert [r[1] for r in res] == [(0, 19), (19, 37)]
    full = oracle.proxy(phi, y).reshape(y.shape[0], -1)
    for _, _, (lo, hi), mine in res:
        assert np.allclose(mine, full[lo:hi], rtol=1e-12, atol=1e-12)


def test_row_and_batch_ranges():
    from paper_1701_03891_b200.rowshard import batch_range, row_range
    for m in (1, 7, 410, 16384):
        for w in (1, 2, 3, 8):
            if w > m:
                continue
            spans = [row_range(m, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    assert batch_range(8, 4, 3) == (6, 8)
    import pytest
    with pytest.raises(ValueError):
        batch_range(6, 4, 0)
    with pytest.raises(ValueError):
        row_range(2, 3, 0)


class _OracleCtx:
    """Stands in for DeepInverse in the CPU test of bench.output_check: recover() runs the oracle (test-only)."""
    storage_dtype = None

    def __init__(self, c, corrupt=False):
        import torch
        self.c, self.corrupt = c, corrupt
        self.storage_dtype = torch.float32

    def recover(self, yd):
        import torch
        import oracle
        phi, _, _, params = bench.make_inputs(self.c, "f32", 0, 1)
        out = oracle.forward(yd.numpy(), phi, params, self.c.n, self.c.n).astype(np.float32)
        return torch.from_numpy(out)


def _gather_worker(rank, world, port, corrupt, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = synth.CONFIGS["tiny"]
        B = c.batch
        lo, hi = bench.shard(rank, B)
        _, _, y, _ = bench.make_inputs(c, "f32", lo, B)
        xhat = _OracleCtx(c).recover(torch.from_numpy(y))
        if corrupt and rank == 1:
            xhat[2, 7, 9] += 0.5                         # one wrong pixel on rank 1
        parts = bench.gather_to_all(xhat, world)
        if rank == 0:
            q.put(bench.output_check(_OracleCtx(c), c, "f32", B, world, parts, "cpu"))
    finally:
        dist.destroy_process_group()


def _run_gather(corrupt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, corrupt, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = q.get(timeout=180)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    return res


def test_two_rank_output_gather_check():
    """bench.py's output check over 2 gloo ranks: x_hat gathered to rank 0 equals rank 0's own recovery of the same
    global images bitwise and the oracle within tolerance; one corrupted pixel on rank 1 fails both."""
    good = _run_gather(False)
    assert good["pass"] and good["bitwise_vs_rank0_recovery"] and good["ranks"] == 2 and good["oracle_images"] == 8
    bad = _run_gather(True)
    assert not bad["pass"] and not bad["bitwise_vs_rank0_recovery"]
    assert bad["oracle_max_pixel_err_over_max"] > bad["tol"]


def test_bench_launcher_and_world_check():
    """`python bench.py --gpus N` without torchrun re-executes under torchrun with N ranks on a loopback rendezvous;
    under torchrun a WORLD_SIZE different from --gpus is refused."""
    cmd = bench.launcher_cmd(["--gpus", "4", "--steps", "3"], 4, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")
    old = dict(os.environ)
    try:
        os.environ.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
        assert bench.main(["--gpus", "4"]) == 2
        assert bench.main(["--gpus", "0"]) == 2
    finally:
        os.environ.clear()
        os.environ.update(old)


def test_make_inputs_rows_matches_contiguous_generation():
    c = synth.CONFIGS["tiny"]
    _, x, y, _ = bench.make_inputs(c, "bf16", 0, 8)
    _, x2, y2, _ = bench.make_inputs_rows(c, "bf16", [0, 1, 5, 6, 7])
    assert np.array_equal(x2, x[[0, 1, 5, 6, 7]]) and np.array_equal(y2, y[[0, 1, 5, 6, 7]])
    assert bench.check_rows(4096)[:2] == [0, 1] and bench.check_rows(4096)[-1] == 4095 and len(bench.check_rows(4096)) == 64
