import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_helpers import Case, make_ctx, y_device
case = Case(64, 64, 410, 20, "bf16")
ctx = make_ctx(case, max_batch=20)
B, n1, n2 = 20, 64, 64
y = y_device(case, ctx)
def stages():
    xt = torch.empty((B, n1, n2), dtype=torch.bfloat16, device="cuda")
    h1 = torch.empty((B, n1, n2, 64), dtype=torch.bfloat16, device="cuda")
    h2 = torch.empty((B, n1, n2, 32), dtype=torch.bfloat16, device="cuda")
    xh = torch.empty((B, n1, n2), dtype=torch.float32, device="cuda")
    ctx.debug_stage(0, y, xt, B); ctx.debug_stage(1, xt, h1, B); ctx.debug_stage(2, h1, h2, B); ctx.debug_stage(3, h2, xh, B)
    torch.cuda.synchronize()
    return xt, h1, h2, xh
r1 = stages(); r2 = stages()
for i, (a, b) in enumerate(zip(r1, r2)):
    a = a.float().cpu().numpy(); b = b.float().cpu().numpy()
    d = a != b
    print("stage", i, "ndiff", int(d.sum()), "of", d.size, "maxabs", float(np.abs(a-b).max()))
    if d.any():
        idx = np.argwhere(d)
        print("  first diffs", idx[:10].tolist())
        print("  imgs with diffs", np.unique(idx[:,0]).tolist())
# stage 2 repeated on identical input
xt, h1, h2, xh = r1
outs = []
for k in range(4):
    o = torch.empty_like(h2); ctx.debug_stage(2, h1, o, B); torch.cuda.synchronize(); outs.append(o.float().cpu().numpy())
for k in range(1, 4):
    d = outs[k] != outs[0]
    print("conv2 rerun", k, "ndiff", int(d.sum()), "rows", np.unique(np.argwhere(d)[:,1]).tolist()[:20] if d.any() else [])
