"""Quick per-stage timing of the bf16 path on the bench workload (CUDA events inside the library)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse
cfg = sys.argv[1] if len(sys.argv) > 1 else "lowrate"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
c = synth.CONFIGS[cfg]
phi = synth.make_phi(c.m, c.N, "bf16")
B = c.batch
x = np.random.default_rng(0).random((B, c.n, c.n), dtype=np.float32)
y = (x.reshape(B, -1) @ phi.T).astype(np.float32)
ctx = DeepInverse(phi, synth.make_params().rounded("bf16"), c.n, c.n, "bf16", max_batch=B)
yd = torch.from_numpy(y).to(device="cuda", dtype=torch.bfloat16)
out = torch.empty((B, c.n, c.n), device="cuda")
for _ in range(3): ctx.recover(yd, out)
torch.cuda.synchronize()
ctx.set_profiling(True); ctx.stage_times(reset=True)
for _ in range(reps): ctx.recover(yd, out)
ms, calls = ctx.stage_times(reset=True)
print(json.dumps({"variant": os.environ.get("DI_CONV2_VARIANT", "0"), "cfg": cfg,
                  "stages_ms": [round(m / calls, 4) for m in ms],
                  "conv2_tflops": round(2*32*64*121*B*c.N / (ms[2]/calls/1e3) / 1e12, 1)}))
