"""One rank's share of a row-sharded recovery, timed on one GPU.

With Phi [M][N] split over G ranks by rows, rank g lifts ALL B images over its M/G rows (di_proxy_partial: a
bf16 tcgen05 GEMM that streams its Phi block from HBM once), the partials are reduce-scattered (B*N*4 bytes per
rank over NVLink/NVSwitch -- reported, not timed: one GPU here), and the rank runs the convolutions on its B/G
images (di_recover_from_proxy).  Prints one JSON line with the device times (CUDA events, median of --reps).

  python tools/rowshard_bench.py [--n 512] [--ratio 0.25] [--world 8] [--batch 64] [--reps 10]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse, row_range

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--ratio", type=float, default=0.25)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
N = a.n * a.n
M = int(round(a.ratio * N))
lo, hi = row_range(M, a.world, 0)
t0 = time.time()
phi_g = synth.make_phi(M, N, "bf16", rows=(lo, hi))
gen_s = time.time() - t0
ctx = DeepInverse(phi_g, synth.make_params(), a.n, a.n, "bf16", max_batch=a.batch)
del phi_g
g = torch.Generator(device="cuda").manual_seed(1701)
y = (torch.randn((a.batch, hi - lo), generator=g, device="cuda") / np.sqrt(M) * np.sqrt(N) * 0.3).to(torch.bfloat16)
per = a.batch // a.world
part = torch.empty((a.batch, N), device="cuda")
xhat = torch.empty((per, a.n, a.n), device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tp, tc = [], []
for r in range(a.reps + 3):
    ev[0].record()
    ctx.proxy_partial(y, out=part)
    ev[1].record()
    ctx.recover_from_proxy(part[:per], xhat=xhat)   # stand-in for this rank's reduce-scattered block
    ev[2].record()
    torch.cuda.synchronize()
    if r >= 3:
        tp.append(ev[0].elapsed_time(ev[1])), tc.append(ev[1].elapsed_time(ev[2]))
tp, tc = float(np.median(tp)), float(np.median(tc))
phi_bytes = (hi - lo) * N * 2
flops = 2.0 * a.batch * (hi - lo) * N
print(json.dumps({
    "n": a.n, "M": M, "world": a.world, "rows_per_rank": hi - lo, "global_batch": a.batch,
    "phi_block_GB": phi_bytes / 1e9, "proxy_partial_ms": tp, "proxy_GBps": phi_bytes / tp / 1e6,
    "proxy_TFLOPs": flops / tp / 1e9, "convs_ms_per_rank": tc, "reduce_scatter_bytes_per_rank": a.batch * N * 4,
    "images_per_s_per_job_excl_collective": a.batch / ((tp + tc) / 1e3), "host_phi_gen_s": gen_s}))
