"""Sustained (power-capped) A/B of experiment switches read at di_create: each variant's context runs the lowrate
recovery back to back for ~1.5 s per turn, variants alternating, 4 rounds; images/s from CUDA events over the turn.
  python tools/scratch/ab_sustained.py 'DI_EXP_C2_CLUSTER=2' 'DI_EXP_C2_CLUSTER=4' ..."""
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
yd = torch.from_numpy(y).to(device="cuda", dtype=torch.bfloat16)
variants = sys.argv[1:] or ["DI_EXP_C2_CLUSTER=2", "DI_EXP_C2_CLUSTER=4"]
ctxs = {}
for v in variants:
    saved = dict(os.environ)
    for kv in v.split(","):
        if "=" in kv:
            k, val = kv.split("=", 1)
            os.environ[k] = val
    ctxs[v] = (DeepInverse(phi, params, c.n, c.n, "bf16", max_batch=B), torch.empty((B, c.n, c.n), device="cuda"))
    os.environ.clear(); os.environ.update(saved)
ref = None
res = {v: [] for v in variants}
for rnd in range(4):
    for v, (ctx, xd) in ctxs.items():
        for _ in range(3): ctx.recover(yd, xd)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n, t0 = 0, time.time()
        e0.record()
        while time.time() - t0 < 1.5:
            for _ in range(10): ctx.recover(yd, xd)
            n += 10
            torch.cuda.synchronize()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        if ref is None: ref = xd.clone()
        res[v].append(B / ms * 1e3)
        print(json.dumps({"round": rnd, "variant": v, "ms": round(ms, 4), "images_s": round(B / ms * 1e3),
                          "bitwise_vs_first": bool(torch.equal(ref, xd))}), flush=True)
print(json.dumps({v: {"median": float(np.median(r)), "all": [round(a) for a in r]} for v, r in res.items()}))
