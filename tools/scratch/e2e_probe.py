"""Where the end-to-end (di_recover_host) step loses time against the device-resident step: timings + a torch
profiler timeline of two e2e steps (kernels and copies), summarised as busy / idle intervals of the GPU."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
c = synth.CONFIGS["lowrate"]
B = c.batch
phi = synth.make_phi(c.m, c.N, "bf16")
ctx = DeepInverse(phi, synth.make_params().rounded("bf16"), c.n, c.n, "bf16", max_batch=B)
y = np.random.default_rng(0).standard_normal((B, c.m)).astype(np.float32)
yd = torch.from_numpy(y).to(device="cuda", dtype=torch.bfloat16)
yh = yd.cpu().pin_memory()
xh = torch.empty((B, c.n, c.n), dtype=torch.float32).pin_memory()
xd = torch.empty((B, c.n, c.n), device="cuda")
def tm(fn, k=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
out = {}
out["device_ms"] = tm(lambda: ctx.recover(yd, xd))
out["e2e_ms"] = tm(lambda: ctx.recover_host(yh, xh.numpy()))
out["h2d_y_ms"] = tm(lambda: yd.copy_(yh, non_blocking=True))
out["d2h_x_ms"] = tm(lambda: xh.copy_(xd, non_blocking=True))
xn = xh.numpy()
t0 = time.perf_counter()
for _ in range(20): ctx.recover_host(yh, xn)
out["e2e_wall_ms"] = (time.perf_counter() - t0) / 20 * 1e3
print(json.dumps(out))
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3): ctx.recover_host(yh, xn)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
if iv:
    t_start = iv[0][0]
    rows = []
    for s, e, n in iv:
        rows.append((round((s - t_start) / 1e3, 3), round((e - s) / 1e3, 3), n[:40]))
    for r in rows[:200]: print(r)
