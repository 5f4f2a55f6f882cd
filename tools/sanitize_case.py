"""Small run of every kernel (bf16, tf32, fp32; recover, stages, sensing, metrics) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from gpu_helpers import Case, make_ctx
for prec in ("bf16", "tf32", "f32"):
    for (n1, n2, m, b) in [(16, 16, 64, 4), (40, 72, 300, 5), (64, 64, 410, 3)]:
        case = Case(n1, n2, m, b, prec, 4, 2)
        ctx = make_ctx(case)
        y = torch.from_numpy(case.y).cuda().to(ctx.storage_dtype)
        xh = ctx.recover(y)
        x = torch.from_numpy(case.x).cuda()
        ym = ctx.measure(x)
        ctx.add_noise(ym, 20.0, 1)
        ctx.metrics(xh, x)
        torch.cuda.synchronize()
        print(prec, n1, n2, "ok", float(xh.abs().max()))
        ctx.close()
