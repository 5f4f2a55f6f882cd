"""Data-parallel training step: every rank computes the gradient of its shard with
scale = 1/global_batch (di_train_grad), the gradients are summed across ranks with one NCCL all-reduce (the only
collective of the method), and every rank applies the same SGD step (di_sgd_step).  Prints per-step device times.

  python tools/train_dp.py [steps] [batch_per_rank] [config] [f32|tf32|bf16]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/train_dp.py ..."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import torch.distributed as dist
import synth
from paper_1701_03891_b200 import DeepInverse

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = sys.argv[3] if len(sys.argv) > 3 else "paper"
prec = sys.argv[4] if len(sys.argv) > 4 else "f32"
rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
c = synth.CONFIGS[cfg]
st = "bf16" if prec == "bf16" else "f32"
phi = synth.make_phi(c.m, c.N, st)
x = synth.make_images(c.n, rank * B, B, c.n_blobs, c.n_rects, c.texture_var)
y = synth.measure(phi, x, st)
ctx = DeepInverse(phi, synth.make_params(bias="channel").rounded(st), c.n, c.n, prec, device=local, max_batch=B)
yd, xd = torch.from_numpy(y).to(dev).to(ctx.storage_dtype), torch.from_numpy(x).to(dev)
scale = 1.0 / (B * world)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
times, losses, lr = [], [], None
for s in range(steps + 2):
    ev[0].record()
    loss, g = ctx.train_grad(yd, xd, scale)
    ev[1].record()
    if world > 1:
        dist.all_reduce(g)                      # sum of the shard gradients = the global-batch gradient
        dist.all_reduce(loss)
    ev[2].record()
    if lr is None:
        lr = 0.05 * float(loss.item()) / float((g.double() ** 2).sum())
    ctx.sgd_step(g, lr, 0.9)
    ev[3].record()
    torch.cuda.synchronize()
    losses.append(float(loss.item()))
    if s >= 2:
        times.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
t = np.mean(times, axis=0)
if rank == 0:
    print(json.dumps({"cfg": cfg, "precision": prec, "world": world, "batch_per_rank": B, "ms": {"grad": t[0], "allreduce": t[1],
                      "sgd": t[2]}, "images_per_s": B * world / (t.sum() / 1e3), "loss_first_last": [losses[0], losses[-1]]}))
if world > 1:
    dist.destroy_process_group()
