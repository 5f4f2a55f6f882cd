"""Quick per-stage timing of the bf16 path on the bench workload (CUDA events inside the library)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
cfg = sys.argv[1] if len(sys.argv) > 1 else "lowrate"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = synth.CONFIGS[cfg]
prec = sys.argv[3] if len(sys.argv) > 3 else ("tf32" if cfg == "paper" else "bf16")
st = "bf16" if prec == "bf16" else "f32"
t0 = time.time()
phi = synth.make_phi(c.m, c.N, st)
B = int(sys.argv[4]) if len(sys.argv) > 4 else c.batch
x = np.random.default_rng(0).random((B, c.n, c.n), dtype=np.float32)
y = (x.reshape(B, -1) @ phi.T).astype(np.float32)
gen_s = time.time() - t0
ctx = DeepInverse(phi, synth.make_params().rounded(st), c.n, c.n, prec, max_batch=B)
yd = torch.from_numpy(y).to(device="cuda", dtype=ctx.storage_dtype)
out = torch.empty((B, c.n, c.n), device="cuda")
for _ in range(3): ctx.recover(yd, out)
torch.cuda.synchronize()
ctx.set_profiling(True); ctx.stage_times(reset=True)
for _ in range(reps): ctx.recover(yd, out)
ms, calls = ctx.stage_times(reset=True)
tot = sum(ms) / calls
print(json.dumps({"cfg": cfg, "prec": prec, "batch": B, "stages_ms": [round(m / calls, 4) for m in ms],
                  "total_ms": round(tot, 4), "images_per_s": round(B / (tot / 1e3)),
                  "proxy_tflops": round(2 * c.m * c.N * B / (ms[0] / calls / 1e3) / 1e12, 1),
                  "conv2_tflops": round(2*32*64*121*B*c.N / (ms[2]/calls/1e3) / 1e12, 1), "gen_s": round(gen_s, 1)}))
