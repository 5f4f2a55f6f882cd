"""Row-sharded recovery on real ranks: run under torchrun with G ranks (one per GPU).

Every rank holds rows row_range(M, G, rank) of Phi and recovers the GLOBAL batch's images of its batch block, both
with the NCCL reduce-scatter (RowShardedDeepInverse.recover) and with the fused form (the lifting GEMM's epilogue
writing into the owners' peer-mapped staging buffers over NVLink, recover(fused=True)).  Rank 0 gathers the blocks
and checks them against the fp64 oracle with the full Phi.  Prints one JSON line; exit code 1 on a failed check.

  python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 tools/rowshard_check.py [n] [M] [B]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import synth
from paper_1701_03891_b200 import RowShardedDeepInverse, batch_range, row_range

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
B = int(sys.argv[3]) if len(sys.argv) > 3 else 8 * world
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
phi = synth.make_phi(M, n * n, "bf16")
x = synth.make_images(n, 0, B, 8, 4)
y = synth.measure(phi, x, "bf16")
params = synth.make_params().rounded("bf16")
lo, hi = row_range(M, world, rank)
rs = RowShardedDeepInverse(phi[lo:hi], params, n, n, "bf16", device=local, max_batch=B)
yr = torch.from_numpy(np.ascontiguousarray(y[:, lo:hi])).to(device=dev, dtype=torch.bfloat16)
out = {}
for fused in (False, True):
    xh = rs.recover(yr, fused=fused)
    torch.cuda.synchronize()
    parts = [torch.empty_like(xh) for _ in range(world)] if world > 1 else [xh]
    if world > 1:
        dist.all_gather(parts, xh)
    out[fused] = torch.cat(parts).cpu().numpy()
ok = True
line = {"world": world, "n": n, "M": M, "global_batch": B}
if rank == 0:
    import oracle
    ref = oracle.forward(y, phi, params, n, n)
    for fused in (False, True):
        rel = max(oracle.rel_l2(g, r) for g, r in zip(out[fused], ref))
        pix = max(float(np.max(np.abs(g - r)) / np.max(np.abs(r))) for g, r in zip(out[fused], ref))
        line["fused" if fused else "reduce_scatter"] = {"max_rel_l2": rel, "max_pixel_err_over_max": pix}
        ok &= rel <= 2e-2 and pix <= 2e-2
    line["pass"] = bool(ok)
    print(json.dumps(line), flush=True)
rs.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
sys.exit(0 if ok else 1)
