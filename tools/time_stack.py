"""Timing of a custom layer stack through the C ABI: python tools/time_stack.py
<prec> <batch> <n> <m> <w1,w2,...> -- e.g. bf16 4096 64 410 1,64,64,32,1 (CUDA events, device-resident y)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
prec, B, n, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
widths = [int(v) for v in sys.argv[5].split(",")]
r = np.random.default_rng(5)
ws = [(r.standard_normal((co, ci, 11, 11)) * np.sqrt(2.0 / (ci * 121))).astype(np.float32)
      for ci, co in zip(widths[:-1], widths[1:])]
bs = [r.uniform(-0.1, 0.1, co).astype(np.float32) for co in widths[1:]]
st = "bf16" if prec == "bf16" else "f32"
params = synth.Params(ws, bs).rounded(st)
phi = synth.make_phi(m, n * n, st)
y = np.random.default_rng(1).standard_normal((B, m)).astype(np.float32)
ctx = DeepInverse(phi, params, n, n, prec, max_batch=B)
yd = torch.from_numpy(y).to(device="cuda", dtype=ctx.storage_dtype)
out = torch.empty((B, n, n), device="cuda")
for _ in range(3): ctx.recover(yd, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ctx.recover(yd, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
flop = 2 * B * n * n * sum(ci * co * 121 for ci, co in zip(widths[:-1], widths[1:]))
print(json.dumps({"prec": prec, "widths": widths, "batch": B, "n": n, "ms": round(ms, 3),
                  "images_per_s": round(B / ms * 1e3), "conv_tflops": round(flop / ms / 1e9, 1)}))
