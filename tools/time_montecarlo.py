"""Monte-Carlo recovery loop on the GPU (§5 protocol, synthetic images): x (device) -> y = Phi x ->
+ noise at an SNR -> x_hat = M(y) -> per-image PSNR / NMSE / success.  Prints per-stage device times."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1701_03891_b200 import DeepInverse

cfg = sys.argv[1] if len(sys.argv) > 1 else "lowrate"
snr = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
c = synth.CONFIGS[cfg]
prec = "bf16"
phi = synth.make_phi(c.m, c.N, prec)
B = c.batch
x = torch.from_numpy(synth.make_images(c.n, 0, B, c.n_blobs, c.n_rects, c.texture_var)).cuda()
ctx = DeepInverse(phi, synth.make_params().rounded(prec), c.n, c.n, prec, max_batch=B)
y = torch.empty((B, c.m), dtype=torch.bfloat16, device="cuda")
xh = torch.empty((B, c.n, c.n), device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
tot = np.zeros(4)
for r in range(reps + 3):
    ev[0].record(); ctx.measure(x, y); ev[1].record(); ctx.add_noise(y, snr, 1701 + r); ev[2].record()
    ctx.recover(y, xh); ev[3].record(); m = ctx.metrics(xh, x); ev[4].record()
    torch.cuda.synchronize()
    if r >= 3:
        tot += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
tot /= reps
print(json.dumps({"cfg": cfg, "snr_db": snr, "batch": B, "ms": {"measure": tot[0], "noise": tot[1], "recover": tot[2],
                  "metrics+d2h": tot[3]}, "images_per_s": B / (tot.sum() / 1e3),
                  "mean_psnr_db": float(np.mean(m[0])), "success_rate": float(np.mean(m[2]))}))
