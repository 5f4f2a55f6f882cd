"""A/B of di_recover_host settings read at di_create (env assignments, e.g. DI_EXP_E2E_WAVES=0): one context per
variant in one process, e2e and device steps timed alternately (CUDA events, 20 steps, 5 rounds)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
c = synth.CONFIGS["lowrate"]
B = c.batch
phi = synth.make_phi(c.m, c.N, "bf16")
params = synth.make_params().rounded("bf16")
variants = sys.argv[1:] or ["DI_EXP_E2E_WAVES=1", "DI_EXP_E2E_WAVES=0"]
ctxs = {}
for v in variants:
    saved = dict(os.environ)
    for kv in v.split(","):
        k, val = kv.split("=", 1)
        os.environ[k] = val
    ctxs[v] = DeepInverse(phi, params, c.n, c.n, "bf16", max_batch=B)
    os.environ.clear(); os.environ.update(saved)
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
res = {v: [] for v in variants}
for rnd in range(6):
    for v, ctx in ctxs.items():
        d = tm(lambda: ctx.recover(yd, xd))
        e = tm(lambda: ctx.recover_host(yh, xn))
        if ref is None: ref = xn.copy()
        res[v].append((round(e / d - 1, 4), round(B / e * 1e3)))
        assert np.array_equal(ref, xn)
print(json.dumps({v: {"gap": [a for a, _ in r], "e2e": [b for _, b in r], "median_gap": float(np.median([a for a, _ in r]))}
                  for v, r in res.items()}))
