import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from gpu_helpers import Case, make_ctx, y_device
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
case = Case(64, 64, 410, 20, prec)
ctx = make_ctx(case, max_batch=20)
y = y_device(case, ctx)
outs = [ctx.recover(y).cpu().numpy() for _ in range(4)]
for k in range(1, 4):
    d = outs[k] != outs[0]
    print("rerun", k, "ndiff", int(d.sum()), "maxabs", float(np.abs(outs[k]-outs[0]).max()))
    if d.any():
        idx = np.argwhere(d); print("  imgs", np.unique(idx[:,0]).tolist(), "rows", np.unique(idx[:,1]).tolist()[:30])
one = ctx.recover(y[7:8].contiguous()).cpu().numpy()
print("batch-invariance ndiff", int((one[0] != outs[0][7]).sum()))
