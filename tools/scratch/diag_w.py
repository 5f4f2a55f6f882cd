"""Per-stage element-wise check of conv2 (stage 2) and conv3 (stage 3) on selected images of a large batch."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np, torch
import oracle
from gpu_helpers import Case, make_ctx, y_device
n, B = int(sys.argv[1]), int(sys.argv[2])
imgs = [int(v) for v in sys.argv[3].split(",")]
case = Case(n, n, 410 if n == 64 else n * n // 10, B, "bf16", 8, 4)
ctx = make_ctx(case)
y = y_device(case, ctx)
dt = ctx.storage_dtype
xt = torch.empty((B, n, n), dtype=dt, device="cuda"); h1 = torch.empty((B, n, n, 64), dtype=dt, device="cuda")
h2 = torch.empty((B, n, n, 32), dtype=dt, device="cuda"); xh = torch.empty((B, n, n), dtype=torch.float32, device="cuda")
ctx.debug_stage(0, y, xt, B); ctx.debug_stage(1, xt, h1, B); ctx.debug_stage(2, h1, h2, B); ctx.debug_stage(3, h2, xh, B)
torch.cuda.synchronize()
p = case.params
for b in imgs:
    a1 = h1[b].float().cpu().numpy().astype(np.float64).transpose(2, 0, 1)
    r2 = oracle.conv_layer(a1, p.w[1], None, relu=True)
    g2 = h2[b].float().cpu().numpy().astype(np.float64).transpose(2, 0, 1)
    e2 = np.abs(g2 - r2).max(axis=0) / max(np.abs(r2).max(), 1e-30)
    a2 = g2
    r3 = oracle.conv_layer(a2, p.w[2], None, relu=False)[0]
    g3 = xh[b].cpu().numpy().astype(np.float64)
    e3 = np.abs(g3 - r3) / max(np.abs(r3).max(), 1e-30)
    bad2 = np.argwhere(e2 > 1.5e-2); bad3 = np.argwhere(e3 > 1e-3)
    print(f"img {b}: conv2 max {e2.max():.3g} bad {len(bad2)} rows {sorted(set(bad2[:, 0].tolist()))[:20]} | "
          f"conv3 max {e3.max():.3g} bad {len(bad3)} rows {sorted(set(bad3[:, 0].tolist()))[:20]} cols {sorted(set(bad3[:, 1].tolist()))[:12]}")
