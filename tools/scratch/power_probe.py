"""Power / clock trace while the lowrate recovery runs back to back for ~3 s (nvml sampled every 5 ms from a
separate process): is the step power-capped, and at what draw?"""
import os, sys, json, subprocess, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
LOOP = r"""
import sys, time, pynvml as nv
nv.nvmlInit(); h = nv.nvmlDeviceGetHandleByIndex(0)
t_end = time.time() + float(sys.argv[1])
while time.time() < t_end:
    t = time.time()
    p = nv.nvmlDeviceGetPowerUsage(h) / 1e3
    try:
        pi = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
        pin = pi.value.uiVal / 1e3 if pi.nvmlReturn == 0 else -1
    except Exception:
        pin = -1
    c = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
    print(f"{t:.4f} {p:.1f} {pin:.1f} {c} {r}", flush=True)
    time.sleep(0.005)
"""
c = synth.CONFIGS["lowrate"]
B = c.batch
phi = synth.make_phi(c.m, c.N, "bf16")
params = synth.make_params().rounded("bf16")
x = synth.make_images(c.n, 0, B, c.n_blobs, c.n_rects, c.texture_var)
y = synth.measure(phi, x, "bf16")
ctx = DeepInverse(phi, params, c.n, c.n, "bf16", max_batch=B)
yd = torch.from_numpy(y).to(device="cuda", dtype=torch.bfloat16)
xd = torch.empty((B, c.n, c.n), device="cuda")
for _ in range(5): ctx.recover(yd, xd)
torch.cuda.synchronize()
time.sleep(2.0)
pr = subprocess.Popen([sys.executable, "-c", LOOP, "6"], stdout=subprocess.PIPE, text=True)
time.sleep(1.0)
t0 = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(20): ctx.recover(yd, xd)
    n += 20
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
t1 = time.time()
out = pr.communicate()[0]
ms = e0.elapsed_time(e1) / n
rows = [l.split() for l in out.splitlines() if l.strip()]
inside = [r for r in rows if t0 + 0.2 < float(r[0]) < t1]
idle = [r for r in rows if float(r[0]) < t0]
pw = np.array([float(r[1]) for r in inside]); pin = np.array([float(r[2]) for r in inside])
clk = np.array([float(r[3]) for r in inside])
print(json.dumps({"steps": n, "ms_per_step": ms, "images_s": B / ms * 1e3,
                  "power_avg_w": {"median": float(np.median(pw)), "max": float(pw.max())},
                  "power_instant_w": {"median": float(np.median(pin)), "max": float(pin.max()), "p10": float(np.percentile(pin, 10))},
                  "sm_mhz": {"median": float(np.median(clk)), "min": float(clk.min()), "max": float(clk.max())},
                  "reasons": sorted(set(r[4] for r in inside)), "idle_power_w": float(np.median([float(r[1]) for r in idle])) if idle else None,
                  "samples": len(inside)}))
