"""How much do the library's per-stage CUDA events (di_set_profiling: an event between consecutive kernels, which
keeps a programmatic dependent launch from starting early) cost the step?  20 recoveries timed by two outer events,
profiling on / off alternating, 6 rounds, lowrate."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
c = synth.CONFIGS["lowrate"]
phi = synth.make_phi(c.m, c.N, "bf16")
B = c.batch
x = np.random.default_rng(0).random((B, c.n, c.n), dtype=np.float32)
y = (x.reshape(B, -1) @ phi.T).astype(np.float32)
ctx = DeepInverse(phi, synth.make_params().rounded("bf16"), c.n, c.n, "bf16", max_batch=B)
yd = torch.from_numpy(y).to(device="cuda", dtype=ctx.storage_dtype)
out = torch.empty((B, c.n, c.n), device="cuda")
for _ in range(5): ctx.recover(yd, out)
torch.cuda.synchronize()
res = {"on": [], "off": []}
for rnd in range(6):
    for mode in ("on", "off"):
        ctx.set_profiling(mode == "on"); ctx.stage_times(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20): ctx.recover(yd, out)
        e1.record(); torch.cuda.synchronize()
        res[mode].append(round(e0.elapsed_time(e1) / 20, 4))
ctx.set_profiling(False)
print(json.dumps({"ms_per_step": res, "median_on": float(np.median(res["on"])), "median_off": float(np.median(res["off"]))}))
