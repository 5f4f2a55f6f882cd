"""A/B of di_recover_host chunk plans (DI_EXP_E2E_RATIO read at di_create): contexts with ratio 2 (r01 halving
plan), 3, 4, 6 in one process, e2e and device steps timed alternately (CUDA events, 20 steps each, 5 rounds)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
c = synth.CONFIGS["lowrate"]
B = c.batch
phi = synth.make_phi(c.m, c.N, "bf16")
params = synth.make_params().rounded("bf16")
ratios = [int(r) for r in (sys.argv[1:] or ["2", "3", "4", "6"])]
ctxs = {}
for r in ratios:
    os.environ["DI_EXP_E2E_RATIO"] = str(r)
    ctxs[r] = DeepInverse(phi, params, c.n, c.n, "bf16", max_batch=B)
y = np.random.default_rng(0).standard_normal((B, c.m)).astype(np.float32)
yd = torch.from_numpy(y).to(device="cuda", dtype=torch.bfloat16)
yh = yd.cpu().pin_memory()
xh = torch.empty((B, c.n, c.n), dtype=torch.float32).pin_memory()
xd = torch.empty((B, c.n, c.n), device="cuda")
xn = xh.numpy()
def tm(fn, k=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
ref = None
for rnd in range(5):
    for r, ctx in ctxs.items():
        d = tm(lambda: ctx.recover(yd, xd))
        e = tm(lambda: ctx.recover_host(yh, xn))
        if ref is None: ref = xn.copy()
        same = bool(np.array_equal(ref, xn))
        print(json.dumps({"round": rnd, "ratio": r, "device_ms": round(d, 4), "e2e_ms": round(e, 4),
                          "e2e_images_s": round(B / e * 1e3), "gap": round(e / d - 1, 4), "bitwise": same}), flush=True)
