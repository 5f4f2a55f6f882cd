"""One library (DI_LIB), one process: the lowrate recovery as the bench times it (5 warm-up, 20 timed steps, per-stage
CUDA events) and then sustained (back to back for 2 s); one JSON line.  Driven by ab_lib_sustained.sh."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
c = synth.CONFIGS["lowrate"]
B = c.batch
phi = synth.make_phi(c.m, c.N, "bf16")
params = synth.make_params().rounded("bf16")
x = synth.make_images(c.n, 0, B, c.n_blobs, c.n_rects, c.texture_var)
y = synth.measure(phi, x, "bf16")
ctx = DeepInverse(phi, params, c.n, c.n, "bf16", max_batch=B)
yd = torch.from_numpy(y).to(device="cuda", dtype=torch.bfloat16)
xd = torch.empty((B, c.n, c.n), device="cuda")
time.sleep(1.0)
for _ in range(5): ctx.recover(yd, xd)
torch.cuda.synchronize()
ctx.set_profiling(True); ctx.stage_times(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): ctx.recover(yd, xd)
e1.record(); torch.cuda.synchronize()
burst = e0.elapsed_time(e1) / 20
ms, calls = ctx.stage_times(reset=True)
ctx.set_profiling(False)
n, t0 = 0, time.time()
e0.record()
while time.time() - t0 < 2.0:
    for _ in range(10): ctx.recover(yd, xd)
    n += 10
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / n
print(json.dumps({"lib": os.path.basename(os.environ.get("DI_LIB", "libdeepinverse.so")), "burst_ms": round(burst, 4),
                  "burst_images_s": round(B / burst * 1e3), "sustained_images_s": round(B / sus * 1e3),
                  "stages_ms": [round(m / calls, 4) for m in ms], "xhat_sum": float(xd.double().sum())}), flush=True)
